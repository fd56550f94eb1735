timeout 300 python tools/ab_small.py PSD_SMALL_NOFOLD fp16 fp16x3
timeout 120 python tools/small_stamps.py 2>&1 | grep -i "small\|phase\|mma\|epilogue" | head -20
