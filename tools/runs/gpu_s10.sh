mkdir -p gpurun_out/s10
timeout 900 python -m pytest tests/test_distributed.py -m gpu -q > gpurun_out/s10/pytest_dist.txt 2>&1; echo "rc=$?" >> gpurun_out/s10/pytest_dist.txt
