#!/bin/bash
# c3 bench lines (fp16, fp16x3, tf32x3) + the 1-CTA kernel's GPU tests
OUT=gpurun_out/${1:-r2s3c3}; mkdir -p $OUT
for p in fp16 fp16x3 tf32x3; do
  timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c3_$p.json 2> $OUT/bench_c3_$p.err
done
timeout 900 python -m pytest tests -m gpu -q -k "split_k or boundary or determinism or degree1 or newton or split_precision or sym_product or lower_triangle" > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
tail -2 $OUT/pytest.txt; for f in $OUT/bench_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
