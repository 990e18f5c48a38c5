set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2l_pytest.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo bench rc=$?
WORKLOAD=c4 REPS=2 timeout 300 python scripts/gen_once.py > gpurun_out/gen_plain.log 2>&1 && \
WORKLOAD=c4 REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:generate_kernel -s 1 -c 1 -o gpurun_out/r2l_gen_c4 python scripts/gen_once.py > gpurun_out/ncu_gen.log 2>&1; echo ncu_gen rc=$?
