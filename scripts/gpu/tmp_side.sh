for f in -1 0.04 0.055 0.065 0.09; do RICI_SP_SIDE_FRAC=$f MODE=search ROUNDS=1 REPS=5 timeout 600 python scripts/variant_time.py . ; done > gpurun_out/r2an_side.jsonl 2>&1
cat gpurun_out/r2an_side.jsonl
