# r3 final pass 4 (final build: split-model changes): default bench (C2 + ctx_128k C3), C4 rank share, launch list at C2
set -x
O=gpurun_out/r3_final4
mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ctx128k > $O/ncu_launch_c2.log 2>&1
