MODE=search ROUNDS=2 REPS=5 timeout 1200 python scripts/variant_time.py scratch/sp_head scratch/sp_feat > gpurun_out/r2ap_sp_variants.jsonl 2>&1; cat gpurun_out/r2ap_sp_variants.jsonl
WORKLOAD=c4 timeout 600 python scripts/timeline.py > gpurun_out/r2ap_timeline_c4.txt 2>&1; grep -E "features|span" gpurun_out/r2ap_timeline_c4.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2ap_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/r2ap_pytest.log
