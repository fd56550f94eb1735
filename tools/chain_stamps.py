"""Per-product phase counters of the CTA-pair kernel inside the c4 chain (PSD_DEBUG_STAMPS=1,
graphs off)."""
import os, sys
os.environ["PSD_DEBUG_STAMPS"] = "1"
os.environ["PSD_NO_GRAPH"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_09165_b200 as pkg
n, batch = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 32)))
prec = sys.argv[3] if len(sys.argv) > 3 else "fp16"
A = torch.randn(batch, n, n, device="cuda")
f = pkg.Filter(pkg.filters.half_filter(), precision=prec)
f.project(A)
torch.cuda.synchronize()
