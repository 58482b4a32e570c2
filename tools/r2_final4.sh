# r2 final pass 4 (after step graphs and the K1 row change): GPU suite, smoke, default bench line, reference arm
set -x
O=gpurun_out/r2_final4
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
