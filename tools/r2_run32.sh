set -x
O=gpurun_out/r2_32
mkdir -p $O
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_shard_gpu.py tests/test_decoder_gpu.py tests/test_adapter_gpu.py tests/test_regressions_gpu.py tests/test_quant_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_launch3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_launch2.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
