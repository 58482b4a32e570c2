# r2 pass 27: split-count sweep of the current K2 (one-layer harness)
set -x
O=gpurun_out/r2_27
mkdir -p $O
for ns in 0 3 4 5 6 7 8; do echo "nsplit $ns"; SPC_NSPLIT=$ns timeout 600 python tools/ab_k2.py --config c2 --libs ab/lib_cur.so --rounds 1; done > $O/split_c2.txt 2>&1
for ns in 0 12 14 16 18 20 24; do echo "nsplit $ns"; SPC_NSPLIT=$ns timeout 600 python tools/ab_k2.py --config c3 --libs ab/lib_cur.so --rounds 1; done > $O/split_c3.txt 2>&1
