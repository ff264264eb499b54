#!/bin/bash
# checkpoint / resume tests + the eviction and host-API tests + smoke
TAG=${1:-r03c}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1200 python -m pytest -q tests/test_gpu_checkpoint.py tests/test_gpu_evict_select.py tests/test_gpu_host_api.py tests/test_gpu_serving.py tests/test_gpu_sharded.py > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED|^ERROR|Error" gpurun_out/${TAG}_pytest.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$? $(tail -1 gpurun_out/${TAG}_smoke.log | cut -c1-200)"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('maintenance',{}).get('evict_ms_rounds'))"
