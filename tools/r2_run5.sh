# r2 pass 5: VCOOP z-MMA A layout + row-major P pairs; A/B vs r1 and the first VCOOP; mma.sync probe
set -x
O=gpurun_out/r2_05
mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py -m gpu -q -x > $O/pytest_decode.log 2>&1
./tools/mma_probe > $O/mma_probe.json 2>&1
for c in c3 c4; do timeout 900 python tools/ab_k2.py --config $c --libs ab/lib_base.so ab/lib_vcoop.so ab/lib_vco2.so --rounds 2 > $O/ab_$c.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
