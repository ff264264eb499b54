#!/bin/bash
# top-k scan timing (C2 cache, B = 4,096 and 32, top-1/4/16) + an ncu capture of the top-16 scan
TAG=${1:-r03k}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python scripts/sweep.py --n 100000 --latents 1 --batches 32,4096 --scorers tc --topks 1,4,16 > gpurun_out/${TAG}_sweep.log 2>&1; echo "sweep=$?"
grep '^{' gpurun_out/${TAG}_sweep.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k: d[k] for k in d if k in ('b','topk','scorer','score_ms','step_ms','kernel_ms')})"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_score_tc2 --launch-skip 3 --launch-count 1 -o gpurun_out/${TAG}_top16 python scripts/sweep.py --n 100000 --latents 0 --batches 4096 --scorers tc --topks 16 --steps 3 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu=$?"
