#!/bin/bash
# round-2 bench refresh: every config's bench line, the default line with e2e + cpu baseline, the
# reference arm, the c4 launch list; plus the new determinism/in-place test
OUT=gpurun_out/${1:-r2fin}; mkdir -p $OUT
timeout 300 python -m pytest tests -m gpu -q -k "determinism" > $OUT/pytest_det.txt 2>&1; echo "rc=$?" >> $OUT/pytest_det.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c4_fp16.json 2> $OUT/bench_c4_fp16.err
timeout 900 python bench.py --precision fp16x3 --no-cpu-baseline > $OUT/bench_c4_fp16x3.json 2> $OUT/bench_c4_fp16x3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in c2 c3; do for p in fp16 fp16x3; do
  timeout 300 python bench.py --config $c --precision $p --no-cpu-baseline --steps 100 > $OUT/bench_${c}_$p.json 2> $OUT/bench_${c}_$p.err
done; done
timeout 900 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 5 > $OUT/bench_c5_fp16.json 2> $OUT/bench_c5_fp16.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.txt 2>&1
tail -2 $OUT/pytest_det.txt; for f in $OUT/bench_*.json; do echo $f; cut -c1-220 $f; done
