set -x
timeout 900 python -m paper_2007_02306_b200.clutterbox --scenes 50 --levels 1-20 --grid 100,100 --out gpurun_out/r2q_c5_sweep_50x20.json > gpurun_out/r2q_c5.log 2>&1; echo c5 rc=$?
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/r2q_ncu_launch.log 2>&1; echo launches rc=$?
timeout 300 python scripts/c4_search_once.py > gpurun_out/search_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:crss_mma_sp_kernel -c 1 -o gpurun_out/r2q_sp_c4 python scripts/c4_search_once.py > gpurun_out/r2q_ncu_sp.log 2>&1; echo ncu_sp rc=$?
WORKLOAD=c4 REPS=2 timeout 300 python scripts/gen_once.py > gpurun_out/gen_plain.log 2>&1 && \
WORKLOAD=c4 REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:generate_kernel -s 1 -c 1 -o gpurun_out/r2q_gen_c4 python scripts/gen_once.py > gpurun_out/r2q_ncu_gen.log 2>&1; echo ncu_gen rc=$?
