#!/bin/bash
# One GPU verification cycle (run under gpurun): tests, bench, launch list, ncu capture.
# usage: scripts/gpu_cycle.sh TAG [full|quick]
TAG=${1:-dev}; MODE=${2:-full}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x > gpurun_out/${TAG}_tc.log 2>&1; echo "tc_tests=$? $(tail -1 gpurun_out/${TAG}_tc.log)"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "gpu_tests=$? $(tail -1 gpurun_out/${TAG}_pytest_gpu.log)"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | cut -c1-2000
if [ "$MODE" = "full" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_normalise|k_score|k_finalize" --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launches=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_tc -s 3 -c 1 -o gpurun_out/${TAG}_prof_tc_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu_full=$?"
fi
