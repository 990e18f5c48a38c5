set -x
MODE=search ROUNDS=2 REPS=5 timeout 1200 python scripts/variant_time.py scratch/sp_base scratch/sp_skew scratch/sp_l2pf scratch/sp_both > gpurun_out/r2c_sp_variants.jsonl 2>&1; echo sweep rc=$?
WORKLOAD=c4 REPS=2 timeout 300 python scripts/gen_once.py > gpurun_out/gen_plain.log 2>&1 && \
WORKLOAD=c4 REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:generate_kernel -s 1 -c 1 -o gpurun_out/r2c_gen_c4 python scripts/gen_once.py > gpurun_out/ncu_gen.log 2>&1; echo ncu_gen rc=$?
