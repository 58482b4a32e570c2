# r2 pass 12: side kernels beside K2 (K2 GQA at 120 regs, 128-thread K3b/K5) A/B in the 32-layer bench; top-k ncu
set -x
O=gpurun_out/r2_12
mkdir -p $O
for lib in ab/lib_topk3.so ab/lib_side128.so; do
  n=$(basename $lib .so)
  SPC_LIB_PATH=$lib timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4share_$n.json 2> $O/bench_c4share_$n.err
  SPC_LIB_PATH=$lib timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_$n.json 2> $O/bench_c3_$n.err
done
for lib in ab/lib_topk3.so ab/lib_side128.so; do
  n=$(basename $lib .so)
  SPC_LIB_PATH=$lib timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline > $O/bench_c4share_${n}_2.json 2> /dev/null
  SPC_LIB_PATH=$lib timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3_${n}_2.json 2> /dev/null
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_topk -s 2 -c 1 -o $O/topk_c4share python tools/profile_layer.py --config c4 --heads 1 --batch 32 --steps 4 > $O/ncu_topk.log 2>&1
