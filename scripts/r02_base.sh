mkdir -p gpurun_out
nproc > gpurun_out/r02a_host.txt; free -g >> gpurun_out/r02a_host.txt; nvidia-smi topo -m >> gpurun_out/r02a_host.txt 2>&1
( time timeout 600 python bench.py --config c4 --steps 5 --warmup 3 ) > gpurun_out/r02a_c4.log 2>&1; echo "c4=$?"
EVICT_REPS=3 timeout 600 python scripts/evict_scale.py 12500000 > gpurun_out/r02a_evict.log 2>&1; echo "evict=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a_evict_c2_launches.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu=$?"
