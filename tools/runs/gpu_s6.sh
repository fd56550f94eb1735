mkdir -p gpurun_out/s6
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s6/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s6/pytest.txt
timeout 120 python tools/small_stamps.py > gpurun_out/s6/small_stamps.txt 2>&1
timeout 300 python bench.py --config c2 --no-e2e --no-cpu-baseline > gpurun_out/s6/c2.json 2>&1
timeout 300 python bench.py --config c2 --precision fp16 --no-e2e --no-cpu-baseline > gpurun_out/s6/c2_fp16.json 2>&1
timeout 300 python bench.py --config c3 --no-e2e --no-cpu-baseline > gpurun_out/s6/c3.json 2>&1
timeout 200 python tools/chain_stamps.py > gpurun_out/s6/chain_stamps.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s6/c4.json 2> gpurun_out/s6/c4.err
