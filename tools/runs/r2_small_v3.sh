#!/bin/bash
# small-n kernel v3 (fragment-layout epilogue): small-n parity subset, c2 bench lines, ncu
OUT=gpurun_out/r2sv4; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "small or boundary or lower or sign or newton or degree1 or admm or c1 or stages" > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python bench.py --config c2 --precision fp16 --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c2_fp16.json 2> $OUT/bench_c2_fp16.err
timeout 300 python bench.py --config c2 --precision fp16x3 --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c2_fp16x3.json 2> $OUT/bench_c2_fp16x3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_batch -s 2 -c 1 \
    -o $OUT/prof_c2 -f python bench.py --config c2 --precision fp16 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/ncu.txt 2>&1
tail -15 $OUT/pytest_gpu.txt; cat $OUT/bench_c2_fp16.json $OUT/bench_c2_fp16x3.json | cut -c1-400; tail -3 $OUT/ncu.txt
