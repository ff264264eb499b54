#!/bin/bash
# ncu --set full with source of one k_evict_select launch (12.5M entries, 1% LCBFU eviction)
TAG=${1:-r03n}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
ARGS=${ARGS:-"12500000 0 0 1"}
EVICT_REPS=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_evict_select --launch-skip 2 --launch-count 1 \
  -o gpurun_out/${TAG}_evict python scripts/evict_scale.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu=$?"
tail -3 gpurun_out/${TAG}_ncu.log
