set -x
for w in c2 c3 c4; do WORKLOAD=$w timeout 600 python scripts/gen_stats.py > gpurun_out/r2g_stats_$w.json 2>&1; echo stats $w rc=$?; done
