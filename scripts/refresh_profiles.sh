#!/bin/bash
# Regenerate the committed measurements (run under gpurun; outputs in gpurun_out/TAG_*, then
# copied into profiles/ by hand):  bench lines (C2 headline, reference arm, C3, C4 and C5 at
# N = 1), the C2 launch list, ncu --set full of the C2 scan and of the gather, eviction scale.
# usage: scripts/refresh_profiles.sh TAG [skip-c5]
TAG=${1:-final}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
o=gpurun_out/${TAG}
timeout 900 python -m pytest tests -m gpu -q > ${o}_pytest_gpu.log 2>&1; echo "gpu_tests=$? $(tail -1 ${o}_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1; echo "smoke=$? $(tail -1 ${o}_smoke.log | cut -c1-200)"
timeout 600 python bench.py > ${o}_bench_c2.log 2>&1; echo "bench_c2=$?"; tail -1 ${o}_bench_c2.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > ${o}_bench_reference.log 2>&1; echo "bench_ref=$?"
timeout 900 python bench.py --config c3 > ${o}_bench_c3.log 2>&1; echo "bench_c3=$?"
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > ${o}_bench_c4.log 2>&1; echo "bench_c4=$?"
if [ "$2" != "skip-c5" ]; then
  timeout 1500 python bench.py --config c5 --steps 4 --warmup 3 > ${o}_bench_c5.log 2>&1; echo "bench_c5=$?"
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_normalise|k_score|k_finalize" --csv \
  --log-file ${o}_c2_launches.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
  --no-maintenance > /dev/null 2>&1; echo "launches=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_tc -s 3 -c 1 -o ${o}_prof_tc_c2 \
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-maintenance > /dev/null 2>&1; echo "ncu_scan=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_finalize -s 3 -c 1 -o ${o}_prof_fin_c2 \
  python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-maintenance > /dev/null 2>&1; echo "ncu_fin=$?"
for gr in 0 1; do
  timeout 300 python scripts/evict_scale.py 12500000 0 $gr >> ${o}_evict_12p5m.jsonl 2>> ${o}_evict_err.log; echo "evict$gr=$?"
done
# memcheck of the newest paths (query slices with the side-stream finalizes; eviction without
# output lists; entry-mode pool-slot listing)
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_slices.py -q -x \
  -k "argument or without_lists or (1100 and 1-)" > ${o}_sanitizer_memcheck_slices.log 2>&1; echo "memcheck=$?"
