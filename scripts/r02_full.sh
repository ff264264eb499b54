#!/bin/bash
# full GPU suite, smoke, default bench (C4) + C2 bench, C4 launch list + ncu capture of the scan
TAG=${1:-r02full}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1500 python -m pytest -q tests -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/${TAG}_pytest.log | head -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$? $(tail -1 gpurun_out/${TAG}_smoke.log | cut -c1-200)"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.log 2>&1; echo "bench_c4=$?"; tail -1 gpurun_out/${TAG}_bench_c4.log | cut -c1-400
timeout 600 python bench.py --config c2 > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | cut -c1-300
bash scripts/r02_c4_profile.sh ${TAG}c4
