WORKLOAD=c4 timeout 600 python scripts/timeline.py > gpurun_out/r2ao_timeline_c4.txt 2>&1; grep -v "^HOST" gpurun_out/r2ao_timeline_c4.txt | awk '$2 != "us" || 1' | sort -t+ -k2 -n -r | head -30
