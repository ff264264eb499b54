#!/bin/bash
# C4 scan: entry tiles per unit (L2 reuse of the entry chunks across the 64 query-tile pairs)
TAG=${1:-r02q}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest -q tests/test_gpu_host_api.py > gpurun_out/${TAG}_pytest_host.log 2>&1; echo "host_api=$? $(tail -1 gpurun_out/${TAG}_pytest_host.log)"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-maintenance > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['e2e'])[:400])"
for nc in 0 8 16 32; do
  if [ $nc = 0 ]; then unset NIRVANA_TC_CHUNK; else export NIRVANA_TC_CHUNK=$nc; fi
  timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_c4_nc$nc.log 2>&1; echo "nc=$nc rc=$?"; tail -1 gpurun_out/${TAG}_c4_nc$nc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks'], d['roofline']['frac'])"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:k_score_tc2 -c 1 --clock-control none --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{print $(NF-2), $NF}'
done
