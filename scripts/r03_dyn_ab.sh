#!/bin/bash
# A/B of the claimed-tail sweep (NV_SEL_DYN_PCT) with the phase trace, 12.5M entries, window on / off
TAG=${1:-r03d}
mkdir -p gpurun_out
export PYTHONPATH=$PWD:$PYTHONPATH
python -c "import oracle; oracle.build()" > /dev/null 2>&1
for pct in ${PCTS:-0 25 40 0}; do
  NV_BUILD_EXTRA_FLAGS="-DNV_SEL_TRACE=1 -DNV_SEL_DYN_PCT=$pct" python -m paper_2312_04429_b200.build --force > gpurun_out/${TAG}_build_$pct.log 2>&1 || { echo build failed; exit 1; }
  for win in -1 0; do
    EVICT_WINDOW=$win NIRVANA_EVICT_TRACE=1 EVICT_REPS=4 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/${TAG}_p${pct}_w$win.log 2>&1
    python - gpurun_out/${TAG}_p${pct}_w$win.log $pct $win <<'PY'
import json, sys
L = open(sys.argv[1]).read().splitlines()
tr = [json.loads(l)["evict_trace"] for l in L if l.startswith('{"evict_trace"')][1:]
ph = [json.loads(l)["sel_phases_us"] for l in L if l.startswith('{"sel_phases_us"')][1:]
ct = [json.loads(l) for l in L if l.startswith('{"sel_cta_grid"')][1:]
res = json.loads(L[-1])
print(f"pct={sys.argv[2]} window={sys.argv[3]} kernel_us={[t['select_kernel_us'] for t in tr]} "
      f"wall_ms={[round(res[f'evict{i}']['ms'],3) for i in range(1,4)]} end={[p[-1] for p in ph]}")
for c in ct[-1:]:
    print("   ", [(s['stamp'], s['median_us'], s['top'][0]) for s in c['slowest']])
PY
  done
done
