#!/bin/bash
# compute-sanitizer (memcheck + racecheck) over the fused eviction tests and the failure tests
TAG=${1:-r02s}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_evict_select.py -k "fused or view or saturation" > gpurun_out/${TAG}_memcheck_evict.log 2>&1; echo "memcheck=$? $(grep -c 'Invalid\|ERROR SUMMARY' gpurun_out/${TAG}_memcheck_evict.log) $(grep 'ERROR SUMMARY' gpurun_out/${TAG}_memcheck_evict.log | tail -1)"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_evict_select.py -k "fused_evict_paths and 0-0" > gpurun_out/${TAG}_racecheck_evict.log 2>&1; echo "racecheck=$? $(grep 'ERROR SUMMARY\|hazard' gpurun_out/${TAG}_racecheck_evict.log | tail -2)"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_failure.py -k virtual tests/test_gpu_serving.py -k "peek or virtual" > gpurun_out/${TAG}_memcheck_failure.log 2>&1; echo "memcheck_failure=$? $(grep 'ERROR SUMMARY' gpurun_out/${TAG}_memcheck_failure.log | tail -1)"
