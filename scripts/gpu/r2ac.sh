set -x
MODE=search ROUNDS=2 REPS=5 timeout 1200 python scripts/variant_time.py scratch/sp_base scratch/sp_tail > gpurun_out/r2ac_sp_variants.jsonl 2>&1; echo sweep rc=$?
cat gpurun_out/r2ac_sp_variants.jsonl
timeout 600 python scripts/sp_prof.py > gpurun_out/r2ac_sp_prof_tail.json 2>&1; echo prof rc=$?
cat gpurun_out/r2ac_sp_prof_tail.json
