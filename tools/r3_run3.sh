# r3 pass 3 (after the warp-uniform K2 issue path): sanitizers over the MHA (NR=2) refill path,
# C4 rank-share / C1 / C1 --graph / full-decoder bench lines, launch list at C2, ncu of K2 at C2
set -x
O=gpurun_out/r3_run3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
for tool in memcheck racecheck synccheck; do
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool python -m pytest tests/test_decode_gpu.py -m gpu -q -k "c1_geometry_vs_oracle or kv_head_scope_mha_2bit or gqa_batch_vs_oracle" > $O/$tool.log 2>&1
done
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 200 --graph > $O/bench_c1_graph.json 2> $O/bench_c1_graph.err
timeout 600 python bench.py --full-decoder > $O/fulldecoder_c2.json 2> $O/fulldecoder_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ctx128k > $O/ncu_launch_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c2 python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_c2.log 2>&1
grep -h "ERROR SUMMARY\|passed\|failed" $O/*check.log
