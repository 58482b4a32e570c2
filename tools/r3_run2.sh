# r3: GPU suite + smoke + default bench (C2 line with the C3 128k companion) after the K2 uniform-warp / elect refill change
set -x
O=gpurun_out/r3_run2
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
tail -3 $O/pytest_gpu.log
