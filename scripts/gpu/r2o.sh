set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1500 python scripts/variant_time.py scratch/g_head scratch/g_base scratch/g_rs > gpurun_out/r2o_gen_variants.jsonl 2>&1; echo sweep rc=$?
MODE=search ROUNDS=2 REPS=5 timeout 1200 python scripts/variant_time.py scratch/sp_base scratch/sp_2m > gpurun_out/r2o_sp_variants.jsonl 2>&1; echo sweep rc=$?
