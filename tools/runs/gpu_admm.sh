mkdir -p gpurun_out/admm
timeout 600 python -m pytest tests/test_gpu_admm.py -m gpu -q > gpurun_out/admm/pytest_admm.txt 2>&1; echo "rc=$?" >> gpurun_out/admm/pytest_admm.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/admm/pytest_all.txt 2>&1; echo "rc=$?" >> gpurun_out/admm/pytest_all.txt
