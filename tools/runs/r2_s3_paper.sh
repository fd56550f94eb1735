#!/bin/bash
# the paper's own B200 sizes (Tables 3-5): n = 5000 / 10000 / 20000, Lanczos bound in the time;
# fp16 (f~*_half) and the FP32-class split precisions (f~*_single); Lanczos cost at c5 / n = 10000
OUT=gpurun_out/${1:-r2s3paper}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/gpu.txt 2>&1
for c in p5k p10k p20k; do
  for p in fp16 fp16x3 tf32x3; do
    steps=10; [ $c = p20k ] && steps=5; [ $p != fp16 ] && [ $c = p20k ] && steps=3
    timeout 900 python bench.py --config $c --precision $p --no-cpu-baseline --steps $steps --warmup 3 > $OUT/bench_${c}_$p.json 2> $OUT/bench_${c}_$p.err
  done
done
timeout 600 python tools/lanczos_cost.py 16384 1 > $OUT/lz_cost_16384.txt 2>&1
timeout 600 python tools/lanczos_cost.py 10240 1 > $OUT/lz_cost_10240.txt 2>&1
for f in $OUT/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(round(d['ms_per_step'],2), 'ms', d['vs_baseline'], d['roofline']['frac'], d.get('e2e',{}).get('value'), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
cat $OUT/lz_cost_*.txt
