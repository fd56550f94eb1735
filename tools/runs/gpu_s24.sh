mkdir -p gpurun_out/s24
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_admm.py -m gpu -q -x -k "small or c1 or lower_triangle or admm or project_parity or zero_nan" > gpurun_out/s24/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s24/pytest.txt
timeout 300 python bench.py --config c2 --no-e2e --no-cpu-baseline --steps 200 > gpurun_out/s24/c2.json 2>&1
timeout 300 python bench.py --config c2 --precision fp16 --no-e2e --no-cpu-baseline --steps 200 > gpurun_out/s24/c2_fp16.json 2>&1
