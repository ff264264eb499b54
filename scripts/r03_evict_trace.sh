#!/bin/bash
# eviction phase trace: NV_SEL_TRACE=1 build, 1% evictions at 12.5M and 100K entries with the
# per-phase %globaltimer stamps of k_evict_select (earliest / latest CTA per stamp)
TAG=${1:-r03tr}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
NV_BUILD_EXTRA_FLAGS="-DNV_SEL_TRACE=1 ${EXTRA_FLAGS}" python -m paper_2312_04429_b200.build --force > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail -20 gpurun_out/${TAG}_build.log; exit 1; }
python -c "import oracle; oracle.build()"
for win in ${WINDOWS:--1 0}; do
for cfg in "12500000 0 0 1" "100000 0 0 0"; do
  set -- $cfg
  EVICT_WINDOW=$win NIRVANA_EVICT_TRACE=1 EVICT_REPS=4 timeout 600 python scripts/evict_scale.py $cfg > gpurun_out/${TAG}_evict_$1_a$4_w$win.log 2>&1; echo "evict $cfg window $win rc=$?"
  grep -E "sel_phases|evict_trace|sel_cta" gpurun_out/${TAG}_evict_$1_a$4_w$win.log | tail -3 | cut -c1-1200
  tail -1 gpurun_out/${TAG}_evict_$1_a$4_w$win.log | cut -c1-600
done
done
