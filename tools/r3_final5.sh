# r3 final pass 5 (MHA split tie-break): GPU suite, smoke, default bench (C2 + ctx_128k C3), C4 rank share
set -x
O=gpurun_out/r3_final5
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
tail -2 $O/pytest_gpu.log
