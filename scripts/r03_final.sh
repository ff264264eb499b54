#!/bin/bash
# final validation at HEAD: full GPU suite, smoke, default bench (C4), C2, C3, reference arm
TAG=${1:-r03fin}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1500 python -m pytest -q tests -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$? $(tail -1 gpurun_out/${TAG}_smoke.log | cut -c1-200)"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.log 2>&1; echo "bench_c4=$?"; tail -1 gpurun_out/${TAG}_bench_c4.log | cut -c1-300
timeout 600 python bench.py --config c2 > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d.get('maintenance',{}).get('evict_ms_rounds'))"
timeout 900 python bench.py --config c3 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c3.log 2>&1; echo "bench_c3=$?"; tail -1 gpurun_out/${TAG}_bench_c3.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1; echo "ref=$?"; tail -1 gpurun_out/${TAG}_bench_ref.log | cut -c1-300
EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_evict.log 2>&1; echo "evict=$?"; tail -1 gpurun_out/${TAG}_evict.log | cut -c1-600
EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 0 1 > gpurun_out/${TAG}_evict_entry.log 2>&1; echo "evict_entry=$?"; tail -1 gpurun_out/${TAG}_evict_entry.log | cut -c1-600
