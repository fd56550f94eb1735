#!/bin/bash
# round 2 verification: full GPU suite, smoke, compute-sanitizer over every kernel path, stress sweeps
OUT=gpurun_out/${1:-r2ver}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > $OUT/san_memcheck.txt 2>&1; echo "rc=$?" >> $OUT/san_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py quick > $OUT/san_racecheck.txt 2>&1; echo "rc=$?" >> $OUT/san_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py quick > $OUT/san_synccheck.txt 2>&1; echo "rc=$?" >> $OUT/san_synccheck.txt
timeout 900 python tools/stress.py 7 50 > $OUT/stress.txt 2>&1
timeout 600 python tools/stress.py 8 50 small > $OUT/stress_small.txt 2>&1
tail -3 $OUT/pytest_gpu.txt $OUT/smoke.txt; for f in memcheck racecheck synccheck; do tail -3 $OUT/san_$f.txt; done; tail -1 $OUT/stress.txt $OUT/stress_small.txt
