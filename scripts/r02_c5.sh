#!/bin/bash
# C5 at N = 1 (100M entries, 161 GB, Zipf queries, 1% LCBFU eviction + re-insertion per round) and C3
TAG=${1:-r02c5}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/${TAG}_c5.log 2>&1; echo "c5=$?"; tail -1 gpurun_out/${TAG}_c5.log | cut -c1-1500
timeout 900 python bench.py --config c3 --steps 20 --warmup 5 > gpurun_out/${TAG}_c3.log 2>&1; echo "c3=$?"; tail -1 gpurun_out/${TAG}_c3.log | cut -c1-600
