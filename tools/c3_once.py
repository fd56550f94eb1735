import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_09165_b200 import Filter, filters
X = torch.randn(1, 1024, 1024, device="cuda"); X = (X + X.transpose(1, 2)) / 2
f = Filter(filters.remez_half_prefix(6))
out = torch.empty_like(X)
for _ in range(4): f.project(X, out=out)
torch.cuda.synchronize()
