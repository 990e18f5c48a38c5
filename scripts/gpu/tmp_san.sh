timeout 300 python scripts/sanitize_case.py > gpurun_out/r2ar_plain.log 2>&1; echo plain rc=$?; tail -1 gpurun_out/r2ar_plain.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/r2ar_memcheck.log 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/r2ar_memcheck.log
