# r2 pass 13: hot-path timeline: what overlaps K2 in the 32-layer loop (C4 share, C3)
set -x
O=gpurun_out/r2_13
mkdir -p $O
timeout 900 python tools/timeline_hotpath.py --config c4 --heads 1 --batch 32 > $O/timeline_c4share.txt 2>&1
timeout 900 python tools/timeline_hotpath.py --config c3 > $O/timeline_c3.txt 2>&1
mv gpurun_out/timeline_*.json $O/ 2>/dev/null
rm -f gpurun_out/trace_*.json
