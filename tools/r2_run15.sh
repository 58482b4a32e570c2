# r2 pass 15: price each side kernel's interference with K2 in the 32-layer loop (SPC_DEBUG_SKIP; timing only)
set -x
O=gpurun_out/r2_15
mkdir -p $O
for sk in 0 1 2 4 6 7; do
  SPC_DEBUG_SKIP=$sk timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4share_skip$sk.json 2> $O/bench_c4share_skip$sk.err
done
for sk in 0 7; do
  SPC_DEBUG_SKIP=$sk timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 6 > $O/bench_c3_skip$sk.json 2> $O/bench_c3_skip$sk.err
  SPC_DEBUG_SKIP=$sk timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 6 > $O/bench_c2_skip$sk.json 2> $O/bench_c2_skip$sk.err
done
