mkdir -p gpurun_out/s13
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s13/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s13/pytest.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s13/c4.json 2> gpurun_out/s13/c4.err
timeout 300 python tools/admm_bench.py > gpurun_out/s13/admm.txt 2>&1
