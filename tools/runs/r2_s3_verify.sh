#!/bin/bash
# sanitizers over every kernel path (incl. the cluster split-K push reduction), stress sweeps, c3 bf16/tf32 lines
OUT=gpurun_out/${1:-r2s3ver}; mkdir -p $OUT
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > $OUT/san_memcheck.txt 2>&1; echo "rc=$?" >> $OUT/san_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py quick > $OUT/san_racecheck.txt 2>&1; echo "rc=$?" >> $OUT/san_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py quick > $OUT/san_synccheck.txt 2>&1; echo "rc=$?" >> $OUT/san_synccheck.txt
timeout 900 python tools/stress.py 9 50 > $OUT/stress.txt 2>&1
timeout 600 python tools/stress.py 10 50 small > $OUT/stress_small.txt 2>&1
for p in bf16 tf32; do
  timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c3_$p.json 2> $OUT/bench_c3_$p.err
done
for f in memcheck racecheck synccheck; do echo == $f; grep -c "^ok" $OUT/san_$f.txt; grep -i "error summary\|hazard\|rc=" $OUT/san_$f.txt | tail -3; done
tail -1 $OUT/stress.txt $OUT/stress_small.txt
for f in $OUT/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1; done
