mkdir -p gpurun_out/s28
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chain_kernel" > gpurun_out/s28/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s28/pytest.txt
timeout 300 python tools/ab_chain.py > gpurun_out/s28/ab_chain.txt 2>&1
