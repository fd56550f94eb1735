#!/bin/bash
# full GPU suite + smoke + c3/c4 bench lines at the current code
OUT=gpurun_out/${1:-r2s3full}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
for p in fp16 bf16 fp16x3 tf32x3; do
  timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c3_$p.json 2> $OUT/bench_c3_$p.err
done
timeout 900 python bench.py > $OUT/bench_c4_fp16.json 2> $OUT/bench_c4_fp16.err
tail -3 $OUT/pytest_gpu.txt; tail -2 $OUT/smoke.txt; for f in $OUT/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(round(d['ms_per_step']*1000,1), 'us', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
