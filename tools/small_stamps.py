import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PSD_DEBUG_STAMPS"] = "1"
os.environ["PSD_NO_GRAPH"] = "1"
import torch
from paper_2507_09165_b200 import Filter, filters
X = torch.randn(4096, 64, 64, device="cuda"); X = (X + X.transpose(1, 2)) / 2
for prec in ["fp16", "fp16x3"]:
    f = Filter(filters.c2_filter(), precision=prec)
    for _ in range(2): f.project(X)
    torch.cuda.synchronize()
