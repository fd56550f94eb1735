#!/bin/bash
# cluster split-K: bulk (TMA) DSMEM push instead of per-thread st.async -- c3 lines, tests, timeline
OUT=gpurun_out/${1:-r2s3bulk}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -k "split_k or boundary or determinism or c3 or split_precision or polar or degree1 or newton" > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for p in fp16 fp16x3 tf32x3 bf16; do
  timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c3_$p.json 2> $OUT/bench_c3_$p.err
done
PSD_LIB_VARIANT=debug timeout 300 python tools/timeline_probe.py fp16 > $OUT/timeline_c3_fp16.txt 2>&1
PSD_LIB_VARIANT=debug timeout 300 python tools/timeline_probe.py fp16x3 > $OUT/timeline_c3_fp16x3.txt 2>&1
tail -2 $OUT/pytest.txt; tail -2 $OUT/timeline_c3_fp16.txt; tail -2 $OUT/timeline_c3_fp16x3.txt
for f in $OUT/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1; done
