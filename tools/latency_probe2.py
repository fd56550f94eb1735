"""Per-product latency: psd_sym_product back to back, and full projections, for small n."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_09165_b200 import Filter, filters
tag = " ".join(f"{k}={os.environ[k]}" for k in ["PSD_SPLITK", "PSD_NO_PDL", "PSD_NO_GRAPH"] if k in os.environ)
for n in [256, 1024]:
    X = torch.randn(n, n, device="cuda"); X = (X + X.T) / 2
    f = Filter(filters.remez_half_prefix(6))
    out = torch.empty_like(X)
    def t(fn, reps=50):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1000
    a = t(lambda: f.sym_product(X, X, out=out))
    b = t(lambda: f.project(X, out=out))
    print(f"n={n} [{tag}] sym_product (2 converts + 1 product) {a:.1f} us; project {b:.1f} us")
