#!/bin/bash
# compare the 4-stage library (in tree) with a 3-stage build (scripts/librici_s3.so)
set -e
python bench.py --steps 5 --warmup 3 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stages4', d['crss']['ms'])"
cp paper_2007_02306_b200/librici.so /tmp/l4.so
cp scripts/librici_s3.so paper_2007_02306_b200/librici.so
python bench.py --steps 5 --warmup 3 --no-cpu-baseline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stages3', d['crss']['ms'])"
cp /tmp/l4.so paper_2007_02306_b200/librici.so
