"""Latency probe for the few-tile path: time psd_project on one n x n matrix (CUDA events,
many repetitions) -- run under different PSD_SPLITK / PSD_NO_PDL environments."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_09165_b200 import Filter, filters
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = 50
X = torch.randn(n, n, device="cuda"); X = (X + X.T) / 2
f = Filter(filters.remez_half_prefix(6))
out = torch.empty_like(X)
for _ in range(5): f.project(X, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(reps): f.project(X, out=out)
e1.record(); torch.cuda.synchronize()
print(f"n={n} splitk={os.environ.get('PSD_SPLITK','auto')} pdl={'off' if os.environ.get('PSD_NO_PDL') else 'on'}: "
      f"{e0.elapsed_time(e1)/reps*1000:.1f} us per projection ({f.gemm_count()} products)")
