#!/bin/bash
# c3 tile-shape / split-K A/B with the 8-warp epilogue (debug build switches)
OUT=gpurun_out/${1:-c3ab}; mkdir -p $OUT
run() { tag=$1; shift; env PSD_LIB_VARIANT=debug "$@" timeout 300 python bench.py --config c3 --precision ${P:-fp16} --no-cpu-baseline --no-e2e --steps 200 > $OUT/$tag.json 2> $OUT/$tag.err; echo "$tag $(python -c "import json;d=json.load(open('$OUT/$tag.json'));print(round(d['ms_per_step']*1000,1),'us')")"; }
for P in fp16 fp16x3; do
  export P
  run ${P}_default
  run ${P}_bn128 PSD_BN=128
  run ${P}_ks2 PSD_SPLITK=2
  run ${P}_ks2_bn128 PSD_SPLITK=2 PSD_BN=128
  run ${P}_ks4_bn128 PSD_SPLITK=4 PSD_BN=128
done 2>&1 | tee $OUT/summary.txt
