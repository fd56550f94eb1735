#!/bin/bash
# c2 small-n kernel: bench lines (fp16, fp16x3) + ncu --set full with source for the fp16 variant
OUT=gpurun_out/r2c2; mkdir -p $OUT
timeout 300 python bench.py --config c2 --precision fp16 --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c2_fp16.json 2> $OUT/bench_c2_fp16.err
timeout 300 python bench.py --config c2 --precision fp16x3 --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c2_fp16x3.json 2> $OUT/bench_c2_fp16x3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_batch -s 2 -c 1 \
    -o $OUT/prof_c2 -f python bench.py --config c2 --precision fp16 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/ncu.txt 2>&1
cat $OUT/bench_c2_fp16.json $OUT/bench_c2_fp16x3.json; tail -3 $OUT/ncu.txt
