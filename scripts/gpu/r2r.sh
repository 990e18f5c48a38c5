set -x
timeout 600 python scripts/sp_prof.py > gpurun_out/r2r_sp_prof.json 2>&1; echo prof rc=$?
cat gpurun_out/r2r_sp_prof.json
