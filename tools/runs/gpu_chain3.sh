mkdir -p gpurun_out/ch3
timeout 200 python tools/chain_probe.py > gpurun_out/ch3/probe.txt 2>&1
timeout 100 python tools/chain_stamps2.py 1024 > gpurun_out/ch3/stamps.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/ch3/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/ch3/pytest.txt
