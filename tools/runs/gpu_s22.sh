mkdir -p gpurun_out/s22
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split or pair_kernel" > gpurun_out/s22/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s22/pytest.txt
timeout 600 python tools/ab_probe.py PSD_NO_UPPER_ONLY fp16x3 > gpurun_out/s22/ab.txt 2>&1
