#!/bin/bash
TAG=${1:-r02i}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest -q -x tests/test_gpu_evict_select.py tests/test_gpu_policies.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_push.py tests/test_gpu_serving.py > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
grep -E "^FAILED|^ERROR|Error" gpurun_out/${TAG}_pytest.log | head -10
for pol in 0 1; do
NIRVANA_EVICT_TRACE=1 EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 $pol > gpurun_out/${TAG}_evict_p$pol.log 2>&1; echo "evict p$pol=$?"; grep -E "evict_trace|entries" gpurun_out/${TAG}_evict_p$pol.log | tail -3 | cut -c1-400
done
EVICT_REPS=1 timeout 600 ncu --set full --import-source on -k regex:k_evict_select -c 1 --clock-control none -o gpurun_out/${TAG}_evict_select python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu_full=$?"
# variant: one 512-thread CTA per SM (128 registers)
NV_BUILD_EXTRA_FLAGS="-DNV_SEL_MINB=1" python -c "from paper_2312_04429_b200 import build; build.build(force=True)" > gpurun_out/${TAG}_build_minb1.log 2>&1
NIRVANA_EVICT_TRACE=1 EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_evict_minb1.log 2>&1; echo "evict minb1=$?"; grep -E "evict_trace" gpurun_out/${TAG}_evict_minb1.log | tail -2 | cut -c1-300
