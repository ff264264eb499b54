#!/bin/bash
# eviction cycle: fused-eviction tests + every eviction-touching GPU test, 12.5M-entry timing,
# launch list, C2 maintenance line
TAG=${1:-r02e}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest -q -x tests/test_gpu_evict_select.py tests/test_gpu_policies.py tests/test_gpu_sort.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_push.py > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "FAIL|Error|assert" gpurun_out/${TAG}_pytest.log | head -20
EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_evict.log 2>&1; echo "evict=$?"; tail -1 gpurun_out/${TAG}_evict.log
EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 0 1 > gpurun_out/${TAG}_evict_entry.log 2>&1; echo "evict_entry=$?"; tail -1 gpurun_out/${TAG}_evict_entry.log
EVICT_REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_evict_launches.csv python scripts/evict_scale.py 12500000 > /dev/null 2>&1; echo "ncu=$?"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('maintenance'))"
