set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1200 python scripts/variant_time.py scratch/g_r0 scratch/g_r1 > gpurun_out/r2h_gen_variants.jsonl 2>&1; echo sweep rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_clutterbox.py -m gpu -x -q > gpurun_out/r2h_pytest.log 2>&1; echo pytest rc=$?
WORKLOAD=c3 timeout 600 python scripts/gen_stats.py > gpurun_out/r2h_stats_c3.json 2>&1; echo stats rc=$?
