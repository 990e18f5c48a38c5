set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1500 python scripts/variant_time.py scratch/g_b3 scratch/g_pq3 scratch/g_b2 scratch/g_pq2 scratch/g_k4 scratch/g_k4pq > gpurun_out/r2k_gen_variants.jsonl 2>&1; echo sweep rc=$?
