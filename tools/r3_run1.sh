# fresh K2 ncu captures (source-level) at C3 and C2 for per-phase instruction attribution
set -x
O=gpurun_out/r3_run1
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c2 python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_c2.log 2>&1
ls -la $O
