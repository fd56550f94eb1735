mkdir -p gpurun_out/p1
(timeout 120 python tools/small_stamps.py > gpurun_out/p1/small_stamps.txt 2>&1)
(timeout 120 python tools/latency_probe2.py > gpurun_out/p1/lat.txt 2>&1)
(PSD_NO_GRAPH=1 timeout 120 python tools/latency_probe2.py >> gpurun_out/p1/lat.txt 2>&1)
(timeout 300 python bench.py --config c2 --no-e2e --no-cpu-baseline > gpurun_out/p1/c2.json 2>&1)
(timeout 300 python bench.py --config c3 --no-e2e --no-cpu-baseline > gpurun_out/p1/c3.json 2>&1)
(timeout 120 python tools/pair_stamps.py > gpurun_out/p1/pair_stamps.txt 2>&1)
(timeout 200 python tools/chain_stamps.py > gpurun_out/p1/chain_stamps.txt 2>&1)
(timeout 300 ncu --set full --clock-control none --import-source on -k regex:small_batch -c 1 -o gpurun_out/p1/prof_small -f python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p1/ncu_small.txt 2>&1)
