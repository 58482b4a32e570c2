# r2 final pass 3 (accumulator fold as its own instantiation; K1 without float64 divisions by powers of two or 1/s):
# GPU suite, smoke, bench lines, full decoder, launch lists (C2, C1), ncu of K2 (C2, C3, C4 share), K1 metrics, sanitizer
set -x
O=gpurun_out/r2_final3
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 600 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --full-decoder > $O/fulldecoder_c2.json 2> $O/fulldecoder_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c2 python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c4s python tools/profile_layer.py --config c4 --heads 1 --batch 32 --steps 4 > $O/ncu_c4s.log 2>&1
for c in c2 c3; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_quantize --csv --log-file $O/k1_$c.csv python tools/profile_layer.py --config $c --steps 1 > $O/ncu_k1_$c.log 2>&1
done
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python -m pytest tests/test_decode_gpu.py -m gpu -q -k "gqa_batch or c1_geometry_vs_oracle" > $O/memcheck.log 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python -m pytest tests/test_decode_gpu.py -m gpu -q -k "gqa_batch_vs_oracle" > $O/racecheck.log 2>&1
# the folding instantiation under the sanitizers: 32k, one split = 128 blocks per warp
SPC_NSPLIT=1 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tests/precision_child.py --b 1 --H 1 --Hq 4 --n0 32768 > $O/memcheck_fold.log 2>&1
SPC_NSPLIT=1 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tests/precision_child.py --b 1 --H 1 --Hq 4 --n0 32768 > $O/racecheck_fold.log 2>&1
SPC_NSPLIT=1 timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tests/precision_child.py --b 1 --H 2 --Hq 2 --bits 2 --n0 32768 > $O/memcheck_fold_pg.log 2>&1
