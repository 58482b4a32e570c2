# r2 pass 4: VCOOP + C-MMA + merge factors; fp32-output parity; bench-geometry parity; A/B; ncu
set -x
O=gpurun_out/r2_04
mkdir -p $O
export SPC_PARITY_LOG=$O/parity_bench_geometry.json
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
for c in c3 c2; do timeout 900 python tools/ab_k2.py --config $c --libs ab/lib_base.so ab/lib_vcoop.so ab/lib_cmma.so --rounds 2 > $O/ab_$c.txt 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c3 python tools/profile_layer.py --config c3 --steps 4 > $O/ncu_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attend_fast -s 2 -c 1 -o $O/k2_c2 python tools/profile_layer.py --config c2 --steps 4 > $O/ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,pcie__throughput.avg.pct_of_peak_sustained_elapsed,syslts__t_sectors_aperture_sysmem.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_prefetch -s 4 -c 8 --csv --log-file $O/ncu_k5_c2.csv python tools/profile_layer.py --config c2 --steps 8 > $O/ncu_k5.log 2>&1
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
