# r2 pass 25: aggregate recompute option (K3r): parity + bench vs spill
set -x
O=gpurun_out/r2_25
mkdir -p $O
timeout 1200 python -m pytest tests/test_decode_gpu.py tests/test_regressions_gpu.py -m gpu -q > $O/pytest.log 2>&1
for c in c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 6 > $O/bench_${c}_spill.json 2> $O/bench_${c}_spill.err
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 6 --agg-mode recompute > $O/bench_${c}_recompute.json 2> $O/bench_${c}_recompute.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_agg --csv --log-file $O/agg_kernels_c2.csv python tools/profile_layer.py --config c2 --steps 3 > $O/ncu_agg.log 2>&1
