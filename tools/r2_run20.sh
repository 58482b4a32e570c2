# r2 pass 20: K1 v2 with the cheaper fast code: tests, timing
set -x
O=gpurun_out/r2_20
mkdir -p $O
timeout 900 python -m pytest tests/test_quant_gpu.py tests/test_regressions_gpu.py tests/test_decode_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
for c in c2 c3; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_quantize --csv --log-file $O/k1_v2_$c.csv python tools/profile_layer.py --config $c --steps 1 > $O/ncu_$c.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quantize_fast2 -c 1 -o $O/k1_v2_c2 python tools/profile_layer.py --config c2 --steps 1 > $O/ncu_full.log 2>&1
