set -x
O=gpurun_out/r2_33
mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
