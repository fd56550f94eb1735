mkdir -p gpurun_out/s7
timeout 300 python tools/e2e_probe.py > gpurun_out/s7/e2e.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/s7/c4_a.json 2>&1
PSD_DEBUG_NOSTORE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/s7/c4_nostore.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/s7/c4_b.json 2>&1
