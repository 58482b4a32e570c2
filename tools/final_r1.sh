# final r1 measurement pass (one box): smoke, bench lines, GPU suite, launch list, ncu captures
set -x
mkdir -p gpurun_out/fin2
O=gpurun_out/fin2
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c3 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c4 > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py --full-decoder > $O/fulldecoder_c2.json 2> $O/fulldecoder_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
