# r2 pass 14: PCIe gather in-flight budget vs K2 at the C4 rank share (256 B rows)
set -x
O=gpurun_out/r2_14
mkdir -p $O
for b in 32768 65536 131072 262144 524288; do
  timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --pf-inflight $b --steps 6 > $O/bench_c4share_pf$b.json 2> $O/bench_c4share_pf$b.err
done
for b in 65536 131072; do
  timeout 600 python bench.py --config c3 --no-cpu-baseline --pf-inflight $b --steps 6 > $O/bench_c3_pf$b.json 2> $O/bench_c3_pf$b.err
done
