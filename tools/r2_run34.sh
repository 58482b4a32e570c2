set -x
O=gpurun_out/r2_34
mkdir -p $O
for ns in 0 4 5 7; do SPC_NSPLIT=$ns timeout 600 python bench.py --no-cpu-baseline --steps 8 > $O/bench_c2_ns$ns.json 2> /dev/null; done
for ns in 0 8; do SPC_NSPLIT=$ns timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4s_ns$ns.json 2> /dev/null; done
