#!/bin/bash
# compute-sanitizer over the single-sweep-window eviction, the candidate apply, the chunked ordered
# compaction and checkpoint / resume
TAG=${1:-r03s}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_evict_select.py -k "window or extremes or view or saturation or adversarial" > gpurun_out/${TAG}_memcheck_evict.log 2>&1; echo "memcheck=$? $(grep 'ERROR SUMMARY' gpurun_out/${TAG}_memcheck_evict.log | tail -1) $(tail -1 gpurun_out/${TAG}_memcheck_evict.log)"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_checkpoint.py > gpurun_out/${TAG}_memcheck_ckpt.log 2>&1; echo "memcheck_ckpt=$? $(grep 'ERROR SUMMARY' gpurun_out/${TAG}_memcheck_ckpt.log | tail -1) $(tail -1 gpurun_out/${TAG}_memcheck_ckpt.log)"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_evict_select.py -k "single_sweep_window and 1-0-0" > gpurun_out/${TAG}_racecheck_evict.log 2>&1; echo "racecheck=$? $(grep 'ERROR SUMMARY\|hazard' gpurun_out/${TAG}_racecheck_evict.log | tail -2) $(tail -1 gpurun_out/${TAG}_racecheck_evict.log)"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_evict_select.py -k "single_sweep_window and 3-0-0" > gpurun_out/${TAG}_synccheck_evict.log 2>&1; echo "synccheck=$? $(grep 'ERROR SUMMARY' gpurun_out/${TAG}_synccheck_evict.log | tail -1) $(tail -1 gpurun_out/${TAG}_synccheck_evict.log)"
