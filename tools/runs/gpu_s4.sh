mkdir -p gpurun_out/s4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4/admm_launches.csv python tools/admm_bench.py 4096 32 > gpurun_out/s4/admm_ncu.txt 2>&1
