timeout 900 python -m paper_2007_02306_b200.clutterbox --scenes 50 --levels 1-20 --grid 100,100 --out gpurun_out/r2aw_c5_sweep_50x20.json > gpurun_out/r2aw_c5.log 2>&1; echo c5 rc=$?
python -c "import json; d=json.load(open('gpurun_out/r2aw_c5_sweep_50x20.json')); print(d['wall_s'], d['images_generated'], d['comparisons'])"
