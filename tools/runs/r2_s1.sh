#!/bin/bash
# round 2 session 1: full GPU suite, smoke, bench lines (c4 fp16 default, c4 fp16x3/tf32x3 single filter), fold stamps, ncu
OUT=gpurun_out/r2s1; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
PSD_LIB_VARIANT=debug timeout 300 python tools/fold_probe.py > $OUT/fold.txt 2>&1
timeout 600 python bench.py > $OUT/bench_c4_fp16.json 2> $OUT/bench_c4_fp16.err
timeout 600 python bench.py --precision fp16x3 --no-cpu-baseline > $OUT/bench_c4_fp16x3.json 2> $OUT/bench_c4_fp16x3.err
timeout 600 python bench.py --precision tf32x3 --no-cpu-baseline --no-e2e > $OUT/bench_c4_tf32x3.json 2> $OUT/bench_c4_tf32x3.err
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches_x3.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --precision fp16x3 > $OUT/ncu_bench_x3.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sym_gemm_2cta -s 30 -c 1 \
    -o $OUT/prof_x3 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --precision fp16x3 > $OUT/ncu_full_x3.txt 2>&1
tail -3 $OUT/pytest_gpu.txt $OUT/smoke.txt; cat $OUT/bench_c4_fp16.json $OUT/bench_c4_fp16x3.json $OUT/bench_c4_tf32x3.json
