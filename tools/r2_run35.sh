# accumulator fold: precision vs split count and K2 time, fold F = 0 (off) / 4 / 8 (default) / 16
set -x
O=gpurun_out/r2_35
mkdir -p $O
for F in 0 4 8 16; do
  for s in 8 32; do
    SPC_LIB_PATH=abl/lib_fold$F.so SPC_NSPLIT=$s timeout 300 python tools/split_precision.py --case c4_share8 > $O/sp_c4_f${F}_s$s.json 2>> $O/sp.err
  done
  SPC_LIB_PATH=abl/lib_fold$F.so timeout 300 python tools/split_precision.py --case c3 --seqs 0,7 > $O/sp_c3_f${F}.json 2>> $O/sp.err
done
timeout 900 python tools/ab_k2.py --config c3 --libs abl/lib_fold0.so abl/lib_fold4.so abl/lib_fold8.so abl/lib_fold16.so --rounds 2 > $O/ab_c3.json 2> $O/ab_c3.err
timeout 900 python tools/ab_k2.py --config c4 --heads 1 --batch 32 --libs abl/lib_fold0.so abl/lib_fold4.so abl/lib_fold8.so abl/lib_fold16.so --rounds 2 > $O/ab_c4s.json 2> $O/ab_c4s.err
timeout 900 python tools/ab_k2.py --config c2 --libs abl/lib_fold0.so abl/lib_fold8.so --rounds 2 > $O/ab_c2.json 2> $O/ab_c2.err
SPC_PARITY_LOG=$O/parity.json timeout 1500 python -m pytest tests/test_bench_geometry_gpu.py -m gpu -q > $O/geom.log 2>&1
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4_share8.json 2> $O/bench_c4_share8.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
