#!/bin/bash
# C4 (the default bench workload) at N = 1: launch list of the timed command and one ncu --set
# full capture of the dominant kernel (the CTA-pair tcgen05 scan over the 10M-entry shard)
TAG=${1:-r02c4}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu_list=$?"
timeout 900 ncu --set full --import-source on -k regex:k_score_tc2 -c 1 --clock-control none -o gpurun_out/${TAG}_score python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu_full=$?"
