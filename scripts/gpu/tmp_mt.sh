MODE=search ROUNDS=3 REPS=5 timeout 1200 python scripts/variant_time.py scratch/sp_base scratch/sp_mt > gpurun_out/r2au_sp_variants.jsonl 2>&1; cat gpurun_out/r2au_sp_variants.jsonl
