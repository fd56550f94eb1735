mkdir -p gpurun_out/s12
timeout 500 python tools/ab_probe.py PSD_NO_COALESCE_LD > gpurun_out/s12/ab_ld.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s12/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s12/pytest.txt
