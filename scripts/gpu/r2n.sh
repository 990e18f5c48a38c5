timeout 600 python scripts/img_compare.py scratch/g_head scratch/g_base scratch/g_rs > gpurun_out/r2n_cmp.txt 2>&1
WORKLOAD=c3 timeout 600 python scripts/img_compare.py scratch/g_head scratch/g_base scratch/g_rs >> gpurun_out/r2n_cmp.txt 2>&1
cat gpurun_out/r2n_cmp.txt
