# r2 pass 17: copy-stream priority at the C4 rank share
set -x
O=gpurun_out/r2_17
mkdir -p $O
SPC_COPY_PRIO=low timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4share_low.json 2> $O/bench_c4share_low.err
SPC_COPY_PRIO=high timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4share_high.json 2> $O/bench_c4share_high.err
SPC_LIB_PATH=ab/lib_side128.so SPC_COPY_PRIO=low timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4share_side128_low.json 2> $O/bench_c4share_side128_low.err
