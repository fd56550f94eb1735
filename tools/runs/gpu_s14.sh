mkdir -p gpurun_out/s14
free -g > gpurun_out/s14/mem.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c5_full_size" > gpurun_out/s14/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s14/pytest.txt
