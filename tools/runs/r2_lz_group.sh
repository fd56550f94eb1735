#!/bin/bash
# Lanczos bound: L2-resident groups of matrices (launch_lanczos_bound) -- cost at c4, group-size A/B
OUT=gpurun_out/${1:-r2lzg}; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -k "lanczos" > $OUT/pytest_lz.txt 2>&1; echo "rc=$?" >> $OUT/pytest_lz.txt
timeout 300 python tools/lanczos_cost.py > $OUT/cost_release.txt 2>&1
for g in 32 1 2 4 6; do
  echo "group $g" >> $OUT/cost_debug.txt
  PSD_LIB_VARIANT=debug PSD_LZ_GROUP=$g timeout 300 python tools/lanczos_cost.py >> $OUT/cost_debug.txt 2>&1
done
tail -2 $OUT/pytest_lz.txt; cat $OUT/cost_release.txt $OUT/cost_debug.txt
