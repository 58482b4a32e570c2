# r2 pass 26: compute-sanitizer over the round-2 kernels (K1 v2, VCOOP K2, top-k, gather, K3r, debug output)
set -x
O=gpurun_out/r2_26
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
T1="tests/test_quant_gpu.py -k (tie_heavy or b2_d128 or b1_d128) "
timeout 1200 $CS --tool memcheck python -m pytest tests/test_quant_gpu.py -m gpu -q -k "tie_heavy or b2_d128 or b1_d128" > $O/memcheck_k1.log 2>&1
timeout 1200 $CS --tool racecheck python -m pytest tests/test_quant_gpu.py -m gpu -q -k "tie_heavy or b2_d128-prefill or b1_d128-prefill" > $O/racecheck_k1.log 2>&1
timeout 1500 $CS --tool memcheck python -m pytest tests/test_decode_gpu.py -m gpu -q -k "gqa_batch or agg_recompute or kv_head_scope_vs or select_topk or odd_topk" > $O/memcheck_decode.log 2>&1
timeout 1500 $CS --tool racecheck python -m pytest tests/test_decode_gpu.py -m gpu -q -k "gqa_batch_vs_oracle or select_topk_kats" > $O/racecheck_decode.log 2>&1
timeout 900 $CS --tool synccheck python -m pytest tests/test_decode_gpu.py -m gpu -q -k "gqa_batch_vs_oracle" > $O/synccheck_decode.log 2>&1
for f in $O/*.log; do echo "== $f"; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK SUMMARY" $f | tail -3; done > $O/summary.txt
