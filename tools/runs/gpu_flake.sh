mkdir -p gpurun_out/flake
for i in 1 2; do
  timeout 900 python -m pytest tests -m gpu -q > gpurun_out/flake/run$i.txt 2>&1; echo "rc=$?" >> gpurun_out/flake/run$i.txt
done
