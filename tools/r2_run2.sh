# r2 pass 2: advisor regressions, launcher, bench-geometry parity, suite, bench lines
set -x
O=gpurun_out/r2_02
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 2400 python -m pytest tests/test_regressions_gpu.py tests/test_bench_gpu.py tests/test_bench_geometry_gpu.py -q -x > $O/pytest_new.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
