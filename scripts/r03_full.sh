#!/bin/bash
# end-of-round validation: full GPU suite, smoke, default bench (C4), C2 (with maintenance), C5 at
# N = 1, the eviction kernel's ncu capture at 12.5M entries (normal build) and its launch list
TAG=${1:-r03full}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1500 python -m pytest -q tests -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$? $(tail -1 gpurun_out/${TAG}_smoke.log | cut -c1-200)"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.log 2>&1; echo "bench_c4=$?"; tail -1 gpurun_out/${TAG}_bench_c4.log | cut -c1-300
timeout 600 python bench.py --config c2 > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d.get('maintenance',{}).get('evict_ms_rounds'))"
EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_evict.log 2>&1; echo "evict=$?"; tail -1 gpurun_out/${TAG}_evict.log | cut -c1-600
EVICT_REPS=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_evict_launches.csv python scripts/evict_scale.py 12500000 > /dev/null 2>&1; echo "ncu_list=$?"
EVICT_REPS=3 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_evict_select --launch-skip 2 --launch-count 1 -o gpurun_out/${TAG}_evict python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_evict_ncu.log 2>&1; echo "ncu_full=$?"
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c5.log 2>&1; echo "c5=$?"; tail -1 gpurun_out/${TAG}_bench_c5.log | cut -c1-400
