timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "small or c2 or 64" > gpurun_out/abm_tests.txt 2>&1; tail -n 3 gpurun_out/abm_tests.txt
timeout 300 python tools/ab_small.py PSD_SMALL_MIRROR_SCALAR fp16 fp16x3
timeout 120 python tools/small_stamps.py 2>&1 | grep -i "small" | head -4
