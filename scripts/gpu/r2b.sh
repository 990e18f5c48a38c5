set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
WORKLOAD=c4 REPS=1 timeout 300 python scripts/gen_once.py > gpurun_out/gen_plain.log 2>&1 && \
WORKLOAD=c4 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:generate_kernel -s 1 -c 1 -o gpurun_out/r2b_gen_c4 python scripts/gen_once.py > gpurun_out/ncu_gen.log 2>&1; echo ncu_gen rc=$?
timeout 300 python scripts/c4_search_once.py > gpurun_out/search_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:crss_mma_sp_kernel -c 2 -o gpurun_out/r2b_sp_c4 python scripts/c4_search_once.py > gpurun_out/ncu_sp.log 2>&1; echo ncu_sp rc=$?
