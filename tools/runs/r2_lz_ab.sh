#!/bin/bash
# Lanczos bound at c4: pipelined halves (default), serial, pipelined with big kernels for half B
echo "== release (pipelined)"; timeout 300 python tools/lanczos_cost.py 2>&1
for v in "PSD_LZ_SERIAL=1" "PSD_LZ_BIG_B=1" "PSD_NONE=1"; do
  echo "== debug lib $v"
  env $v PSD_LIB_VARIANT=debug timeout 300 python tools/lanczos_cost.py 2>&1
done
