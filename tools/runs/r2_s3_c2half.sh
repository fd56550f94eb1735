#!/bin/bash
# 8-warp split path: independent halves (PSD_SMALL_SPLIT_COMMIT=2) vs per-matrix commits (1), debug A/B
OUT=gpurun_out/${1:-r2s3c2h}; mkdir -p $OUT
for v in 1 2 1 2; do
  PSD_LIB_VARIANT=debug PSD_SMALL_SPLIT_COMMIT=$v timeout 300 python bench.py --config c2 --precision fp16x3 --no-cpu-baseline --no-e2e --steps 100 > $OUT/dbg_v${v}.json 2>> $OUT/err.txt
  echo "v=$v fp16x3 $(python -c "import json; print(round(json.load(open('$OUT/dbg_v${v}.json'))['ms_per_step']*1000,1))") us" >> $OUT/ab.txt
done
PSD_LIB_VARIANT=debug PSD_SMALL_SPLIT_COMMIT=2 timeout 600 python -m pytest tests -m gpu -q -k "small or determinism or c2 or admm or split" > $OUT/pytest_v2.txt 2>&1; echo "rc=$?" >> $OUT/pytest_v2.txt
PSD_LIB_VARIANT=debug PSD_SMALL_SPLIT_COMMIT=2 timeout 600 python tools/stress.py 18 40 small > $OUT/stress_v2.txt 2>&1
cat $OUT/ab.txt; tail -2 $OUT/pytest_v2.txt; tail -n1 $OUT/stress_v2.txt
