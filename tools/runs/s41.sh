# tests + smoke + c2/c3/c5 bench lines on the current code
OUT=gpurun_out/s41; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 300 python bench.py --config c2 --steps 100 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 300 python bench.py --config c2 --precision fp16 --steps 200 --no-cpu-baseline > $OUT/bench_c2_fp16.json 2> $OUT/bench_c2_fp16.err
timeout 300 python bench.py --config c3 --steps 100 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 python bench.py --config c5 --steps 5 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
