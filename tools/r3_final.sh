# r3 final pass (after TSC, uniform issue, spill stores): GPU suite, smoke, default bench (C2 + ctx_128k C3),
# C4 rank share, C1 eager/graph, full decoder, reference arm, launch list at C2, ncu of K2 at C2 and C3
set -x
O=gpurun_out/r3_final
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 --graph > $O/bench_c1_graph.json 2> $O/bench_c1_graph.err
timeout 600 python bench.py --full-decoder > $O/fulldecoder_c2.json 2> $O/fulldecoder_c2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ctx128k > $O/ncu_launch_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c2 python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
tail -3 $O/pytest_gpu.log
