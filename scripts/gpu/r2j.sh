set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1200 python scripts/variant_time.py scratch/g_b4 scratch/g_b3 scratch/g_pq3 > gpurun_out/r2j_gen_variants.jsonl 2>&1; echo sweep rc=$?
