# r2 pass 3: VCOOP value path (GQA): GPU suite with fp32 output parity, bench-geometry parity, A/B vs r1 K2
set -x
O=gpurun_out/r2_03
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
for c in c3 c4 c3b2 c2; do timeout 600 python tools/ab_k2.py --config $c --libs ab/lib_base.so ab/lib_vcoop.so --rounds 2 > $O/ab_$c.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
