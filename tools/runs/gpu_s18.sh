mkdir -p gpurun_out/s18
timeout 600 python bench.py --config c5 --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/s18/c5.json 2> gpurun_out/s18/c5.err
timeout 300 python bench.py --config c3 --no-e2e --no-cpu-baseline --steps 200 > gpurun_out/s18/c3.json 2>&1
timeout 300 python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 200 > gpurun_out/s18/c2.json 2>&1
timeout 300 python bench.py --config c2 --precision fp16 --no-e2e --no-cpu-baseline --steps 200 > gpurun_out/s18/c2_fp16.json 2>&1
timeout 600 python bench.py --precision fp16x3 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/s18/c4_fp16x3.json 2>&1
