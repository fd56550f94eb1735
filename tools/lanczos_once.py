"""One Lanczos-bound projection at the c4 shape (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_09165_b200 as pkg
n, batch = 4096, 32
X = torch.randn(batch, n, n, device="cuda")
f = pkg.Filter(pkg.filters.half_filter(), bound="lanczos")
f.project(X)
torch.cuda.synchronize()
