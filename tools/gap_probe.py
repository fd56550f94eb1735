"""Kernel span vs launch-to-launch time of the c4 product launches (debug build, PSD_DEBUG_STAMPS,
no graphs): each product's first-CTA-start to last-CTA-end span from the kernel's own stamps."""
import os, sys
os.environ["PSD_DEBUG_STAMPS"] = "1"
os.environ["PSD_NO_GRAPH"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_09165_b200 as pkg
n, batch = 4096, 32
X = torch.randn(batch, n, n, device="cuda")
X = (X + X.transpose(1, 2)) / 2
f = pkg.Filter(pkg.filters.half_filter())
f.project(X)
torch.cuda.synchronize()
