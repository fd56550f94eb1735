"""A few c3 projections (n = 1024, T = 6, fp16 unless argv[1]) for ncu captures of the 1-CTA kernel."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2507_09165_b200 import Filter, filters

prec = sys.argv[1] if len(sys.argv) > 1 else "fp16"
X = torch.tensor(synth.batch("goe", 1024, 1, 5), dtype=torch.float32, device="cuda")
f = Filter(filters.remez_half_prefix(6), precision=prec)
out = torch.empty_like(X)
for _ in range(3):
    f.project(X, out=out)
torch.cuda.synchronize()
print("ok")
