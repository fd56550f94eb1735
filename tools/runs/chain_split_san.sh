PSD_CHAIN=1 PSD_CHAIN_SPLIT=1 PSD_NO_GRAPH=1 timeout 400 compute-sanitizer --print-limit 4 python tools/chain_crash.py 1024 fp16x3 2>&1 | grep -v "^=========     " | head -60
