mkdir -p gpurun_out/s3
timeout 120 python tools/pair_stamps.py > gpurun_out/s3/pair_stamps.txt 2>&1
timeout 200 python tools/chain_stamps.py > gpurun_out/s3/chain_stamps.txt 2>&1
timeout 120 python tools/small_stamps.py > gpurun_out/s3/small_stamps.txt 2>&1
timeout 200 python tools/admm_bench.py > gpurun_out/s3/admm_bench.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err
timeout 600 python -m pytest tests/test_gpu_admm.py -m gpu -q > gpurun_out/s3/pytest_admm.txt 2>&1; echo "rc=$?" >> gpurun_out/s3/pytest_admm.txt
