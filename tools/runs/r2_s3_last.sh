#!/bin/bash
# end-of-session check of the final tree: whole GPU suite, smoke, default bench line, stress sweeps
OUT=gpurun_out/${1:-r2s3last}; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench_c4_fp16.json 2> $OUT/bench_c4_fp16.err
timeout 900 python tools/stress.py 12 60 > $OUT/stress.txt 2>&1
timeout 600 python tools/stress.py 13 50 small > $OUT/stress_small.txt 2>&1
tail -3 $OUT/pytest_gpu.txt; tail -2 $OUT/smoke.txt; tail -1 $OUT/stress.txt $OUT/stress_small.txt
python -c "import json; d=json.load(open('$OUT/bench_c4_fp16.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
