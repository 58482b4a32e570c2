# K1: conflict-free value-parameter reads and packing loads (42-byte code rows); bit-exactness + ncu
set -x
O=gpurun_out/r2_40
mkdir -p $O
timeout 900 python -m pytest tests/test_quant_gpu.py tests/test_regressions_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
for c in c2 c3; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_quantize --csv --log-file $O/k1_$c.csv python tools/profile_layer.py --config $c --steps 1 > $O/ncu_$c.log 2>&1
done
