#!/bin/bash
# c3 single-pass fp16: KS = 2 with upper-only operands (debug switch) vs default
OUT=gpurun_out/${1:-c3ab2}; mkdir -p $OUT
run() { tag=$1; shift; env PSD_LIB_VARIANT=debug "$@" timeout 300 python bench.py --config c3 --precision ${P:-fp16} --no-cpu-baseline --no-e2e --steps 200 > $OUT/$tag.json 2> $OUT/$tag.err; echo "$tag $(python -c "import json;d=json.load(open('$OUT/$tag.json'));print(round(d['ms_per_step']*1000,1),'us')")"; }
for P in fp16 bf16; do export P; run ${P}_default; run ${P}_ks2 PSD_SPLITK=2; run ${P}_ks2_bn128 PSD_SPLITK=2 PSD_BN=128; done 2>&1 | tee $OUT/summary.txt
for P in fp16x3 tf32x3; do export P; run ${P}_default; run ${P}_ks2_bn128 PSD_SPLITK=2 PSD_BN=128; run ${P}_ks4_bn128 PSD_SPLITK=4 PSD_BN=128; done 2>&1 | tee -a $OUT/summary.txt
