"""Phase stamps of the chain kernel (PSD_DEBUG_STAMPS=1, graphs off) at c3."""
import os, sys
os.environ["PSD_DEBUG_STAMPS"] = "1"
os.environ["PSD_NO_GRAPH"] = "1"
os.environ["PSD_CHAIN"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_09165_b200 as pkg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
X = torch.randn(1, n, n, device="cuda"); X = (X + X.transpose(1, 2)) / 2
f = pkg.Filter(pkg.filters.remez_half_prefix(6), precision="fp16")
for _ in range(2):
    f.project(X)
torch.cuda.synchronize()
