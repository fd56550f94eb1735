import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_09165_b200 import Filter, filters
n = int(sys.argv[1]); prec = sys.argv[2]
X = torch.randn(1, n, n, device="cuda"); X = (X + X.transpose(1, 2)) / 2
f = Filter(filters.remez_half_prefix(6), precision=prec)
f.project(X)
torch.cuda.synchronize()
print("ok", n, prec)
