set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1500 python scripts/variant_time.py scratch/g_base scratch/g_nopf scratch/g_triaos_nopf > gpurun_out/r2w_gen_variants.jsonl 2>&1; echo sweep rc=$?
cat gpurun_out/r2w_gen_variants.jsonl
