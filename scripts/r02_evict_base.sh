#!/bin/bash
# eviction baseline: 12.5M-entry 1% eviction (wall) + launch list, C2 bench maintenance line
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
EVICT_REPS=3 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/${1:-r02b}_evict.log 2>&1; echo "evict=$?"; tail -1 gpurun_out/${1:-r02b}_evict.log
EVICT_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${1:-r02b}_evict_launches.csv python scripts/evict_scale.py 12500000 > /dev/null 2>&1; echo "ncu=$?"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${1:-r02b}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${1:-r02b}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('maintenance'))"
