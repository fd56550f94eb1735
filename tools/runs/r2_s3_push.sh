#!/bin/bash
# cluster split-K with the push reduction (st.async into the peer's receive buffer): c3 lines, tests,
# debug A/B of KS = 2 on the single-pass path, timeline
OUT=gpurun_out/${1:-r2s3push}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -k "split_k or boundary or determinism or degree1 or newton or split_precision or sym_product or lower_triangle or c3 or split_sign" > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for p in fp16 fp16x3 tf32x3; do
  timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/bench_c3_$p.json 2> $OUT/bench_c3_$p.err
done
for ks in 1 2; do for p in fp16 bf16; do
  PSD_LIB_VARIANT=debug PSD_SPLITK=$ks timeout 300 python bench.py --config c3 --precision $p --no-cpu-baseline --no-e2e --steps 100 > $OUT/dbg_ks${ks}_c3_$p.json 2> $OUT/dbg_ks${ks}_c3_$p.err
done; done
PSD_LIB_VARIANT=debug timeout 300 python tools/timeline_probe.py fp16x3 > $OUT/timeline_c3_fp16x3.txt 2>&1
tail -2 $OUT/pytest.txt; for f in $OUT/bench_*.json $OUT/dbg_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(round(d['ms_per_step']*1000,1), 'us', d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
tail -4 $OUT/timeline_c3_fp16x3.txt
