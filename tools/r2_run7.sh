# r2 pass 7: C4 rank-share K2 (1 kv head x 32 seqs), split sweep; spill price (NOSPILL A/B)
set -x
O=gpurun_out/r2_07
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4share.csv python tools/profile_layer.py --config c4 --heads 1 --batch 32 --steps 4 > $O/ncu_launch.log 2>&1
for ns in 0 8 12 17 24 34 48; do echo "nsplit $ns"; SPC_NSPLIT=$ns timeout 600 python tools/ab_k2.py --config c4 --heads 1 --batch 32 --libs ab/lib_cur.so --rounds 1; done > $O/split_sweep_c4share.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c4share python tools/profile_layer.py --config c4 --heads 1 --batch 32 --steps 4 > $O/ncu_c4.log 2>&1
for c in c3 c2; do timeout 900 python tools/ab_k2.py --config $c --libs ab/lib_cur.so ab/lib_nospill.so --rounds 2 > $O/ab_nospill_$c.txt 2>&1; done
