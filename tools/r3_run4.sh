# r3 pass 4: transposed scores for the 8-row GQA K2 (TSC) + warp-uniform issue at all row counts:
# GPU suite, smoke, default bench (C2 + ctx_128k C3), C4 rank share, ncu of K2 at C3 (+ lines)
set -x
O=gpurun_out/r3_run4
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
tail -3 $O/pytest_gpu.log
