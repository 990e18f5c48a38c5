set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1500 python scripts/variant_time.py scratch/g_vp_fb scratch/g_vfe > gpurun_out/r2aa_gen_variants.jsonl 2>&1; echo sweep rc=$?
cat gpurun_out/r2aa_gen_variants.jsonl
