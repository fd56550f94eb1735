#!/bin/bash
# One GPU session: build check, GPU tests, smoke, bench, ncu launch list + one full capture.
# usage: tools/gpu_session.sh TAG [tests|bench|ncu|all] [extra bench args...]
TAG=${1:-run}; WHAT=${2:-all}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu_bench.txt 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sym_gemm -s 30 -c 1 \
      -o $OUT/prof_gemm -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu_full.txt 2>&1
fi
tail -3 $OUT/pytest_gpu.txt $OUT/smoke.txt 2>/dev/null; cat $OUT/bench.json 2>/dev/null; tail -2 $OUT/bench.err 2>/dev/null
