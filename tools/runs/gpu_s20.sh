mkdir -p gpurun_out/s20
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pair_kernel or c4_full or lower_triangle or sign_parity or split" > gpurun_out/s20/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s20/pytest.txt
timeout 500 python tools/ab_probe.py PSD_NO_UPPER_ONLY > gpurun_out/s20/ab.txt 2>&1
