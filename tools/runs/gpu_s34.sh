mkdir -p gpurun_out/s34
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_batch -c 1 -o gpurun_out/s34/prof_c2 -f python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s34/ncu_c2.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sym_gemm_kernel -s 10 -c 1 -o gpurun_out/s34/prof_c3 -f python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s34/ncu_c3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s34/c2_launches.csv python bench.py --config c2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
