# bench --graph at C1 (device and e2e through step graphs), eager C1 for comparison; graph tests
set -x
O=gpurun_out/r2_39
mkdir -p $O
timeout 900 python -m pytest tests/test_graph_gpu.py tests/test_bench_gpu.py -m gpu -q -x > $O/tests.log 2>&1
for r in 1 2; do
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 > $O/bench_c1_eager_$r.json 2> $O/bench_c1_eager_$r.err
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 --graph > $O/bench_c1_graph_$r.json 2> $O/bench_c1_graph_$r.err
done
