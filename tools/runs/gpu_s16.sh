mkdir -p gpurun_out/s16
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "lower_triangle or project_host or zero_nan" > gpurun_out/s16/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s16/pytest.txt
timeout 300 python tools/e2e_probe.py > gpurun_out/s16/e2e.txt 2>&1
