#!/bin/bash
# session 3 baseline at HEAD: full GPU suite, smoke, default bench line, c2 lines
OUT=gpurun_out/${1:-r2s3base}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench_c4_fp16.json 2> $OUT/bench_c4_fp16.err
for p in fp16 fp16x3; do
  timeout 300 python bench.py --config c2 --precision $p --no-cpu-baseline --steps 100 > $OUT/bench_c2_$p.json 2> $OUT/bench_c2_$p.err
done
tail -3 $OUT/pytest_gpu.txt $OUT/smoke.txt; for f in $OUT/bench_*.json; do echo $f; cut -c1-300 $f; done
