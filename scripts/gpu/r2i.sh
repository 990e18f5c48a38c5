set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest.log 2>&1; echo pytest rc=$?
MODE=search ROUNDS=1 REPS=5 timeout 600 python scripts/variant_time.py . > gpurun_out/r2i_search.jsonl 2>&1; echo search rc=$?
timeout 300 python scripts/c4_search_once.py > gpurun_out/r2i_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv python scripts/c4_search_once.py > gpurun_out/r2i_ncu.log 2>&1; echo ncu rc=$?
