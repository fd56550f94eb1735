import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2507_09165_b200 as pkg
for n in (160, 128, 10):
    X = np.stack([np.eye(n), 2 * np.eye(n)])
    for prec in ("tf32", "fp16"):
        f = pkg.Filter(pkg.filters.half_filter(), precision=prec, bound="lanczos", lanczos_safety=1.0)
        lam = torch.zeros(2, dtype=torch.float64, device="cuda")
        f.project(torch.tensor(X, dtype=torch.float32, device="cuda"), lambda_out=lam)
        print(n, prec, lam.cpu().numpy(), f.status())
