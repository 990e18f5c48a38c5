set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2ab_pytest.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/r2ab_bench.json 2> gpurun_out/r2ab_bench.err; echo bench rc=$?
