"""e2e at c4: psd_project_host with several chunk counts, and the raw pinned H2D / D2H bandwidth."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_09165_b200 import Filter, filters
n, batch = 4096, 32
X = torch.randn(batch, n, n).pin_memory()
out = torch.empty_like(X).pin_memory()
d = torch.empty(batch, n, n, device="cuda")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
h2d = t(lambda: d.copy_(X, non_blocking=True)); d2h = t(lambda: out.copy_(d, non_blocking=True))
print(f"pinned H2D {X.numel() * 4 / h2d / 1e6:.1f} GB/s, D2H {X.numel() * 4 / d2h / 1e6:.1f} GB/s", flush=True)
f = Filter(filters.half_filter())
for chunks in [4, 8, 16]:
    ms = t(lambda: f.project_host(X, out, chunks=chunks))
    print(f"project_host chunks={chunks}: {ms:.1f} ms/step, {batch / ms * 1e3:.1f} matrices/s", flush=True)
