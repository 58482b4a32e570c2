# K1 variants A (rot 2j, 42-byte rows), B (rot j, 42), C (rot 2j, 34), O (r2 final: rot j, 34): ncu time/instructions/conflicts
set -x
O=gpurun_out/r2_41
mkdir -p $O
for V in O A B C; do for c in c2 c3; do
SPC_LIB_PATH=abl/lib_k1$V.so timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:k_quantize --csv --log-file $O/k1_${V}_$c.csv python tools/profile_layer.py --config $c --steps 1 > $O/ncu_${V}_$c.log 2>&1
done; done
