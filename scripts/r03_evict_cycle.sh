#!/bin/bash
# eviction cycle: every eviction-touching GPU test on the normal build, then the phase trace
TAG=${1:-r03e}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest -q -x tests/test_gpu_evict_select.py tests/test_gpu_policies.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_push.py tests/test_gpu_serving.py > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED|^ERROR|Error" gpurun_out/${TAG}_pytest.log | head -20
for cfg in "12500000 0 0 1" "12500000 0 1 1" "100000 0 0 0"; do
  set -- $cfg
  EVICT_REPS=4 timeout 600 python scripts/evict_scale.py $cfg > gpurun_out/${TAG}_evict_$1_g$3_a$4.log 2>&1; echo "evict $cfg rc=$?"; tail -1 gpurun_out/${TAG}_evict_$1_g$3_a$4.log | cut -c1-700
done
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('maintenance'))"
bash scripts/r03_evict_trace.sh ${TAG}tr
