set -x
MODE=search ROUNDS=2 REPS=5 timeout 1200 python scripts/variant_time.py scratch/sp_base scratch/sp_epi > gpurun_out/r2s_sp_variants.jsonl 2>&1; echo sweep rc=$?
cat gpurun_out/r2s_sp_variants.jsonl
rm -rf scratch/sp_prof_keep; mv scratch/sp_prof scratch/sp_prof_keep; cp -r scratch/sp_prof_epi scratch/sp_prof
timeout 600 python scripts/sp_prof.py > gpurun_out/r2s_sp_prof_epi.json 2>&1; echo prof rc=$?
cat gpurun_out/r2s_sp_prof_epi.json
