# r2 pass 16: K3b aggregate interference at the C4 rank share: compute-stream priority, aggregate CTA budget
set -x
O=gpurun_out/r2_16
mkdir -p $O
timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 --compute-priority -1 > $O/bench_c4share_prio.json 2> $O/bench_c4share_prio.err
for n in 148 296 592 4096; do
  SPC_AGG_CTAS=$n timeout 600 python bench.py --config c4 --share 8 --no-cpu-baseline --steps 6 > $O/bench_c4share_agg$n.json 2> $O/bench_c4share_agg$n.err
done
timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 6 --compute-priority -1 > $O/bench_c3_prio.json 2> $O/bench_c3_prio.err
timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 6 --compute-priority -1 > $O/bench_c2_prio.json 2> $O/bench_c2_prio.err
