"""Debug build only (PSD_LIB_VARIANT=debug PSD_DEBUG_STAMPS=1): the CTA-pair kernel's phase counters
for one split product per accumulation run length -- the MMA issuer's wait for a free accumulator is
the cost of folding K chunks (reading R23)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
assert os.environ.get("PSD_LIB_VARIANT") == "debug"
os.environ["PSD_DEBUG_STAMPS"] = "1"
import torch
from paper_2507_09165_b200 import Filter, filters
n, batch = 4096, 8
g = torch.Generator().manual_seed(0)
A = torch.randn(batch, n, n, generator=g)
X = ((A + A.transpose(1, 2)) / 2).cuda()
for prec in ["fp16x3", "tf32x3", "fp16"]:
    for kc in ([0, 256, 512, 1024] if prec != "fp16" else [0]):
        f = Filter(filters.half_filter(), precision=prec, accum_chunk=kc)
        for _ in range(2):
            f.sym_product(X, X)
        torch.cuda.synchronize()
        print(f"{prec} kchunk {kc}: see stderr line above", file=sys.stderr, flush=True)
