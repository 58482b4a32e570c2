# r2 pass 19: K1 v2 quantizer: bit-exact tests, timing vs v1, ncu
set -x
O=gpurun_out/r2_19
mkdir -p $O
timeout 900 python -m pytest tests/test_quant_gpu.py tests/test_regressions_gpu.py tests/test_decode_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:k_quantize --csv --log-file $O/k1_v2_c2.csv python tools/profile_layer.py --config c2 --steps 1 > $O/ncu_v2.log 2>&1
SPC_K1_V1=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:k_quantize --csv --log-file $O/k1_v1_c2.csv python tools/profile_layer.py --config c2 --steps 1 > $O/ncu_v1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:k_quantize --csv --log-file $O/k1_v2_c3.csv python tools/profile_layer.py --config c3 --steps 1 > $O/ncu_v2c3.log 2>&1
SPC_K1_V1=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:k_quantize --csv --log-file $O/k1_v1_c3.csv python tools/profile_layer.py --config c3 --steps 1 > $O/ncu_v1c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quantize_fast2 -c 1 -o $O/k1_v2_c2 python tools/profile_layer.py --config c2 --steps 1 > $O/ncu_full.log 2>&1
