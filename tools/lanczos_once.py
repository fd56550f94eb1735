"""One Lanczos-bound projection at the c4 shape with a product-free filter (for an ncu launch list
of the bound's kernels)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_09165_b200 as pkg
n, batch = 4096, 32
X = torch.randn(batch, n, n, device="cuda")
f = pkg.Filter([[1.0]], bound="lanczos")
f.project(X)
torch.cuda.synchronize()
