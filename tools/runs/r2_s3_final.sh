#!/bin/bash
# session-3 final: whole GPU suite, smoke, every config's bench line, reference arm, c4 launch list
OUT=gpurun_out/${1:-r2s3fin}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench_c4_fp16.json 2> $OUT/bench_c4_fp16.err
timeout 900 python bench.py --precision fp16x3 --no-cpu-baseline > $OUT/bench_c4_fp16x3.json 2> $OUT/bench_c4_fp16x3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --ref-seconds 60 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in c2 c3; do for p in fp16 fp16x3; do
  timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline --steps 100 > $OUT/bench_${c}_$p.json 2> $OUT/bench_${c}_$p.err
done; done
timeout 900 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_c5_fp16.json 2> $OUT/bench_c5_fp16.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.txt 2>&1
tail -3 $OUT/pytest_gpu.txt; tail -2 $OUT/smoke.txt
for f in $OUT/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); r=d.get('roofline') or {}; print(d['value'], round(d['ms_per_step'],4), r.get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'))" 2>&1 | tail -1; done
