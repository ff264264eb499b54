#!/bin/bash
# full GPU suite + eviction trace / launch list / ncu capture of the fused select kernel
TAG=${1:-r02f}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1200 python -m pytest -q tests -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | head -20
NIRVANA_EVICT_TRACE=1 EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_evict.log 2>&1; echo "evict=$?"; grep -E "evict_trace|entries" gpurun_out/${TAG}_evict.log | tail -5
NIRVANA_EVICT_TRACE=1 EVICT_REPS=3 timeout 600 python scripts/evict_scale.py 12500000 0 1 > gpurun_out/${TAG}_evict_entry.log 2>&1; echo "evict_entry=$?"; grep -E "evict_trace|entries" gpurun_out/${TAG}_evict_entry.log | tail -4
EVICT_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum -k regex:"k_evict|k_sort" --clock-control none --csv --log-file gpurun_out/${TAG}_evict_launches.csv python scripts/evict_scale.py 12500000 > /dev/null 2>&1; echo "ncu_list=$?"
EVICT_REPS=1 timeout 600 ncu --set full --import-source on -k regex:k_evict_select -c 1 --clock-control none -o gpurun_out/${TAG}_evict_select python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu_full=$?"
NIRVANA_EVICT_TRACE=1 timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.log 2>gpurun_out/${TAG}_bench_c2.err; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('maintenance'))"; grep evict_trace gpurun_out/${TAG}_bench_c2.err | tail -2
