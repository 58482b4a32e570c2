# r2 pass 18: PCIe gather with shared-memory staged (slot, pos) lists: depth 1 vs 4 on the small-row path
set -x
O=gpurun_out/r2_18
mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_quant_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
for lib in ab/lib_pf1.so ab/lib_pf4.so; do
  n=$(basename $lib .so)
  SPC_LIB_PATH=$lib timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4share_$n.json 2> $O/bench_c4share_$n.err
done
SPC_LIB_PATH=ab/lib_pf1.so timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 6 > $O/bench_c3_pf1.json 2> $O/bench_c3_pf1.err
SPC_LIB_PATH=ab/lib_pf1.so timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 6 > $O/bench_c2_pf1.json 2> $O/bench_c2_pf1.err
