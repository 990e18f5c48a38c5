for nt in 1 2; do RICI_SP_NT=$nt MODE=search RANK_MODE=1 ROUNDS=1 REPS=5 timeout 600 python scripts/variant_time.py . ; done > gpurun_out/r2al_rank_nt.jsonl 2>&1
for m in 8 12 4; do RICI_RANK_PREFIXES_SP=$m MODE=search RANK_MODE=1 ROUNDS=1 REPS=5 timeout 600 python scripts/variant_time.py . ; done >> gpurun_out/r2al_rank_nt.jsonl 2>&1
cat gpurun_out/r2al_rank_nt.jsonl
