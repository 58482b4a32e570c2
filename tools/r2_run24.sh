# r2 pass 24: full decoder regression check (prefetch depth fix) vs the r1 library on one box
set -x
O=gpurun_out/r2_24
mkdir -p $O
timeout 600 python bench.py --full-decoder > $O/fulldecoder_c2_fix.json 2> $O/fulldecoder_c2_fix.err
SPC_LIB_PATH=ab/lib_base.so timeout 600 python bench.py --full-decoder > $O/fulldecoder_c2_r1lib.json 2> $O/fulldecoder_c2_r1lib.err
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4share.json 2> $O/bench_c4share.err
timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/bench_c2.json 2> $O/bench_c2.err
