set -x
timeout 300 python scripts/c4_search_once.py > gpurun_out/search_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:crss_mma_sp_kernel -c 1 -o gpurun_out/r2am_sp_c4 python scripts/c4_search_once.py > gpurun_out/r2am_ncu_sp.log 2>&1; echo ncu_sp rc=$?
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2am_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/r2am_ncu_launch.log 2>&1; echo launches rc=$?
