set -x
O=gpurun_out/r2_29
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_combine -s 4 -c 1 -o $O/combine_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu.log 2>&1
