# r2 pass 28: combine rewrite: parity + bench + launch list
set -x
O=gpurun_out/r2_28
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_launch3.log 2>&1
