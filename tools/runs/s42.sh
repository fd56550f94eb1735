OUT=gpurun_out/s42; mkdir -p $OUT
timeout 300 python bench.py --config c3 --steps 100 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 300 python bench.py --config c2 --steps 100 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
