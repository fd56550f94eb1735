mkdir -p gpurun_out/s5
timeout 120 python tools/small_stamps.py > gpurun_out/s5/small_stamps.txt 2>&1
timeout 200 python tools/admm_bench.py > gpurun_out/s5/admm_bench.txt 2>&1
timeout 300 python bench.py --config c2 --precision fp16 --no-e2e --no-cpu-baseline > gpurun_out/s5/c2_fp16.json 2>&1
