mkdir -p gpurun_out/s26
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_admm.py -m gpu -q -x -k "not c4_full and not c5_full" > gpurun_out/s26/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s26/pytest.txt
timeout 300 python tools/ab_c3.py > gpurun_out/s26/ab_c3.txt 2>&1
