#!/bin/bash
# small-n kernel v2 (128 threads/CTA, row per thread, 4 CTAs/SM): GPU suite, c2 bench lines, ncu
OUT=gpurun_out/r2sv2; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python bench.py --config c2 --precision fp16 --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c2_fp16.json 2> $OUT/bench_c2_fp16.err
timeout 300 python bench.py --config c2 --precision fp16x3 --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c2_fp16x3.json 2> $OUT/bench_c2_fp16x3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_batch -s 2 -c 1 \
    -o $OUT/prof_c2 -f python bench.py --config c2 --precision fp16 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/ncu.txt 2>&1
tail -15 $OUT/pytest_gpu.txt; cat $OUT/bench_c2_fp16.json $OUT/bench_c2_fp16x3.json; tail -3 $OUT/ncu.txt
