#!/bin/bash
# cluster split-K for the split precisions on few-tile problems (+ upper-only operands with KS = 2)
OUT=gpurun_out/${1:-ks2}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split or c3 or determinism or lower_triangle or boundary or sym_product" > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for p in fp16 fp16x3 tf32x3; do
  timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 200 > $OUT/bench_c3_$p.json 2> $OUT/bench_c3_$p.err
done
tail -3 $OUT/pytest.txt; for f in $OUT/bench_*.json; do echo "$f $(python -c "import json;d=json.load(open('$f'));print(round(d['ms_per_step']*1000,1),'us', d['roofline']['frac'])")"; done
