"""Phase stamps (%globaltimer) of the 1-CTA product kernel via psd_sym_product (PSD_DEBUG_STAMPS=1)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PSD_DEBUG_STAMPS"] = "1"
import torch
from paper_2507_09165_b200 import Filter, filters
for n in [256, 1024, 1024]:
    X = torch.randn(n, n, device="cuda"); X = (X + X.T) / 2
    f = Filter(filters.remez_half_prefix(6))
    out = torch.empty_like(X)
    for _ in range(3): f.sym_product(X, X, X, out=out, beta=0.5)
    torch.cuda.synchronize()
