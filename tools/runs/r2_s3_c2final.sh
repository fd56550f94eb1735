#!/bin/bash
# per-matrix commits in the small-n kernel by default: whole suite, c2 lines, stress (small), c4 line
OUT=gpurun_out/${1:-r2s3c2f}; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
for p in fp16 fp16x3; do
  timeout 300 python bench.py --config c2 --precision $p --no-cpu-baseline --steps 100 > $OUT/bench_c2_$p.json 2> $OUT/bench_c2_$p.err
done
timeout 600 python tools/stress.py 15 60 small > $OUT/stress_small.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c4_fp16.json 2> $OUT/bench_c4_fp16.err
tail -3 $OUT/pytest_gpu.txt; tail -2 $OUT/smoke.txt; tail -n1 $OUT/stress_small.txt
for f in $OUT/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); r=d.get('roofline') or {}; h=d.get('roofline_hbm') or {}; print(d['value'], round(d['ms_per_step'],4), r.get('frac'), h.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'))" 2>&1 | tail -1; done
