# fold as a per-launch instantiation: tests, A/B vs no fold, bench lines; host-row size probe for the slow-tier layout
set -x
O=gpurun_out/r2_36
mkdir -p $O
timeout 900 python -m pytest tests/test_fold_gpu.py tests/test_bench_geometry_gpu.py -m gpu -q > $O/tests.log 2>&1
for c in "4 4 1" "1 4 1"; do set -- $c
  SPC_LIB_PATH=abl/lib_fold0.so SPC_NSPLIT=4 timeout 300 python tests/precision_child.py --b 2 --H $1 --Hq $2 --bits $3 --seqs 1 > $O/nofold_H$1_Hq$2_b$3.json 2>> $O/child.err
  SPC_NSPLIT=4 timeout 300 python tests/precision_child.py --b 2 --H $1 --Hq $2 --bits $3 --seqs 1 > $O/fold_H$1_Hq$2_b$3.json 2>> $O/child.err
done
timeout 900 python tools/ab_k2.py --config c2 --libs abl/lib_fold0.so abl/lib_new2.so --rounds 2 > $O/ab_c2.json 2> $O/ab_c2.err
timeout 900 python tools/ab_k2.py --config c3 --libs abl/lib_fold0.so abl/lib_new2.so --rounds 2 > $O/ab_c3.json 2> $O/ab_c3.err
timeout 900 python tools/ab_k2.py --config c4 --heads 1 --batch 32 --libs abl/lib_fold0.so abl/lib_new2.so --rounds 2 > $O/ab_c4s.json 2> $O/ab_c4s.err
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
# zero-copy gather rate vs host row size, 2 GiB slab (C4 share: 256 B K and V rows today; 512 B interleaved)
timeout 300 tools/h2d_probe 256 11520 8388608 > $O/h2d_rows.jsonl 2>&1
timeout 300 tools/h2d_probe 512 5760 4194304 >> $O/h2d_rows.jsonl 2>&1
timeout 300 tools/h2d_probe 2048 1600 1048576 >> $O/h2d_rows.jsonl 2>&1
timeout 300 tools/h2d_probe 4096 800 524288 >> $O/h2d_rows.jsonl 2>&1
timeout 300 tools/h2d_probe 8192 1504 262144 >> $O/h2d_rows.jsonl 2>&1
timeout 300 tools/h2d_probe 16384 752 131072 >> $O/h2d_rows.jsonl 2>&1
