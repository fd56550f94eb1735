#!/bin/bash
# small-n kernel: per-matrix commits (1) vs commits pipelined across steps (2), debug build A/B + parity subset
OUT=gpurun_out/${1:-r2s3c2p}; mkdir -p $OUT
for v in 1 2 1 2; do for p in fp16 fp16x3; do
  PSD_LIB_VARIANT=debug PSD_SMALL_SPLIT_COMMIT=$v timeout 300 python bench.py --config c2 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/dbg_v${v}_$p.json 2>> $OUT/err.txt
  echo "v=$v $p $(python -c "import json; print(round(json.load(open('$OUT/dbg_v${v}_$p.json'))['ms_per_step']*1000,1))") us" >> $OUT/ab.txt
done; done
PSD_LIB_VARIANT=debug PSD_SMALL_SPLIT_COMMIT=2 timeout 600 python -m pytest tests -m gpu -q -k "small or determinism or c2 or admm" > $OUT/pytest_v2.txt 2>&1; echo "rc=$?" >> $OUT/pytest_v2.txt
PSD_LIB_VARIANT=debug PSD_SMALL_SPLIT_COMMIT=2 timeout 600 python tools/stress.py 16 40 small > $OUT/stress_v2.txt 2>&1
cat $OUT/ab.txt; tail -2 $OUT/pytest_v2.txt; tail -n1 $OUT/stress_v2.txt
