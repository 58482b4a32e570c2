# r2 checkpoint 2: GPU suite, smoke, bench lines, reference arm, full decoder, launch list
set -x
O=gpurun_out/r2_23
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 600 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --full-decoder > $O/fulldecoder_c2.json 2> $O/fulldecoder_c2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
