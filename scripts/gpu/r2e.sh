set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1200 python scripts/variant_time.py scratch/g_s1 scratch/g_p1 scratch/g_p1b4 scratch/g_s1b4 > gpurun_out/r2e_gen_variants.jsonl 2>&1; echo sweep rc=$?
