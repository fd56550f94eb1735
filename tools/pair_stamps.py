"""Phase counters of the CTA-pair product kernel at the c4 shape (PSD_DEBUG_STAMPS=1):
where the MMA issuer waits (tile id / accumulator / operand stages) and the epilogue cost."""
import os, sys
os.environ["PSD_DEBUG_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_09165_b200 as pkg
n, batch = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 32)))
prec = sys.argv[3] if len(sys.argv) > 3 else "fp16"
A = torch.randn(batch, n, n, device="cuda") / n ** 0.5
f = pkg.Filter(pkg.filters.half_filter(), precision=prec)
for _ in range(3):
    f.sym_product(A, A, None, alpha=1.0, beta=0.0)
torch.cuda.synchronize()
