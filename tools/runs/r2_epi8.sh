#!/bin/bash
# 8-warp epilogue in the 1-CTA product kernel: c3 bench lines + the GPU suite
OUT=gpurun_out/${1:-epi8}; mkdir -p $OUT
for p in fp16 fp16x3 tf32x3; do
  timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c3_$p.json 2> $OUT/bench_c3_$p.err
done
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
tail -3 $OUT/pytest_gpu.txt; for f in $OUT/bench_*.json; do echo $f; cut -c1-200 $f; done
