set -x
MODE=gen ROUNDS=2 REPS=3 WORKLOADS=c2,c3,c4 timeout 1200 python scripts/variant_time.py scratch/gen_base scratch/gen_s0 scratch/gen_s1 > gpurun_out/r2d_gen_variants.jsonl 2>&1; echo sweep rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_pytest.log 2>&1; echo pytest rc=$?
