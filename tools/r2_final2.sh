# r2 final pass 2 (after the accumulator fold): GPU suite, smoke, bench lines, full decoder, launch list, ncu of K2, sanitizer
set -x
O=gpurun_out/r2_final2
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
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c2 python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python -m pytest tests/test_decode_gpu.py -m gpu -q -k "gqa_batch or c1_geometry_vs_oracle" > $O/memcheck.log 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python -m pytest tests/test_decode_gpu.py -m gpu -q -k "gqa_batch_vs_oracle" > $O/racecheck.log 2>&1
timeout 900 python tools/ab_k2.py --config c2 --libs abl/lib_fold0.so abl/lib_new.so --rounds 2 > $O/ab_c2.json 2> $O/ab_c2.err
timeout 900 python tools/ab_k2.py --config c3 --libs abl/lib_fold0.so abl/lib_new.so --rounds 2 > $O/ab_c3.json 2> $O/ab_c3.err
SPC_NSPLIT=8 timeout 300 python tools/split_precision.py --case c4_share8 > $O/sp_c4_s8.json 2> $O/sp.err
