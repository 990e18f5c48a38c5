for p in 2 1; do RICI_SP_PAIRS=$p MODE=search ROUNDS=1 REPS=5 timeout 600 python scripts/variant_time.py . ; done > gpurun_out/r2ax_pairs.jsonl 2>&1; cat gpurun_out/r2ax_pairs.jsonl
RICI_SP_PAIRS=1 WORKLOAD=c4 timeout 600 python scripts/timeline.py > gpurun_out/r2ax_timeline_pairs1.txt 2>&1; grep -E "crss|span" gpurun_out/r2ax_timeline_pairs1.txt | cut -c1-110
