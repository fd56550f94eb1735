"""ADMM S/X update (psd_admm_update) vs the plain projection at the c4 shape (batch 32 x n=4096,
fp16, f~*_half+kappa): the cost of forming M on the fly and writing X_next in the epilogue."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
from paper_2507_09165_b200 import Filter, filters
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 32
C1, K1, y1 = synth.maxcut_admm(n, synth.SEED_BASE + 600)
C = torch.tensor(C1, dtype=torch.float32, device="cuda").expand(batch, n, n).contiguous()
K = torch.tensor(K1, dtype=torch.float32, device="cuda").expand(batch, n, n).contiguous()
y = torch.tensor(y1, dtype=torch.float32, device="cuda").expand(batch, n).contiguous()
f = Filter(filters.half_filter(), precision="fp16")
S, X = torch.empty_like(C), torch.empty_like(C)
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
# the same argument the fused update projects, formed in fp32 as the ABI does (R22):
# the projection's speed depends on the data (tensor-core power), so compare like with like
M = C - K * torch.tensor(1.0, dtype=torch.float32)
M.diagonal(dim1=1, dim2=2).sub_(y)
tp = t(lambda: f.project(M, out=S))
ta = t(lambda: f.admm_update(C, K, y, 1.0, S_out=S, X_out=X))
print(f"n={n} batch={batch}: project {tp:.2f} ms/step ({batch / tp * 1e3:.1f} matrices/s); "
      f"admm_update {ta:.2f} ms/step ({batch / ta * 1e3:.1f} updates/s); overhead {100 * (ta / tp - 1):.1f}%")
