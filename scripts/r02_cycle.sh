#!/bin/bash
# usage: scripts/r02_cycle.sh TAG  -- GPU tests + default bench (C4) + C2 bench
TAG=${1:-r02}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "gpu_tests=$? $(tail -1 gpurun_out/${TAG}_pytest_gpu.log)"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c4.log 2>&1; echo "bench_c4=$?"; tail -1 gpurun_out/${TAG}_bench_c4.log | cut -c1-3000
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 gpurun_out/${TAG}_bench_c2.log | cut -c1-600
