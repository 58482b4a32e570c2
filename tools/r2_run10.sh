# r2 pass 10: ncu of the top-k kernel (where its 130-180 us go)
set -x
O=gpurun_out/r2_10
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_topk -s 2 -c 1 -o $O/topk_c4share python tools/profile_layer.py --config c4 --heads 1 --batch 32 --steps 4 > $O/ncu_topk.log 2>&1
