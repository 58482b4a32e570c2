# r2 first measurement pass: GPU suite, C2/C3 bench lines, ncu --set full (with source) of K2 at C3 and C2
set -x
O=gpurun_out/r2_01
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
lscpu > $O/lscpu.txt; nproc >> $O/lscpu.txt; free -g >> $O/lscpu.txt
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c2 python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_c2.log 2>&1
