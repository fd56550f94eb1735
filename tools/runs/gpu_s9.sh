mkdir -p gpurun_out/s9
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "small_batch" > gpurun_out/s9/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s9/pytest.txt
timeout 300 python bench.py --config c2 --precision fp16 --no-e2e --no-cpu-baseline > gpurun_out/s9/c2_fp16.json 2>&1
timeout 300 python bench.py --config c2 --no-e2e --no-cpu-baseline > gpurun_out/s9/c2.json 2>&1
timeout 300 python tools/e2e_probe.py > gpurun_out/s9/e2e.txt 2>&1
