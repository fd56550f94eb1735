"""Accumulation error of one tensor-core product: C = X X with X symmetric and exactly
representable in fp16 (so operand conversion is exact), vs the float64 product and vs a float32
CPU sgemm.  Separates the accumulator from operand rounding."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2507_09165_b200 import Filter, filters
rng = np.random.default_rng(5)
for n in [256, 512, 1024, 2048, 4096]:
    G = rng.standard_normal((n, n))
    X = ((G + G.T) / 2).astype(np.float16).astype(np.float64)      # symmetric, fp16-exact
    ref = X @ X
    c32 = (X.astype(np.float32) @ X.astype(np.float32)).astype(np.float64)
    t = torch.tensor(X[None], dtype=torch.float32, device="cuda")
    row = []
    for prec in ["fp16", "fp16x3", "tf32"]:
        f = Filter(filters.half_filter(), precision=prec)
        C = f.sym_product(t, t).double().cpu().numpy()[0]
        torch.cuda.synchronize()
        iu = np.triu_indices(n)
        e = np.linalg.norm((C - ref)[iu]) / np.linalg.norm(ref[iu])
        row.append(f"{prec} {e:.2e}")
    e32 = np.linalg.norm(c32 - ref) / np.linalg.norm(ref)
    print(f"n={n:5d} gpu: " + "  ".join(row) + f"   cpu sgemm {e32:.2e}   u32*sqrt(n) {2**-24 * np.sqrt(n):.1e}  u32*n {2**-24 * n:.1e}", flush=True)

# the same measurement through cuBLAS (library GEMMs, not on the product path): TF32 tensor-core
# sgemm and fp16 GEMM with fp32 output -- does the library's accumulation grow the same way?
torch.backends.cuda.matmul.allow_tf32 = True
rng = np.random.default_rng(5)
for n in [256, 1024, 4096]:
    G = rng.standard_normal((n, n))
    X = ((G + G.T) / 2).astype(np.float16).astype(np.float64)
    ref = X @ X
    t = torch.tensor(X, dtype=torch.float32, device="cuda")
    c_tf32 = (t @ t).double().cpu().numpy()
    h = t.half()
    c_h = torch.matmul(h, h, out=None).double().cpu().numpy() if False else None
    torch.backends.cuda.matmul.allow_tf32 = False
    c_f32 = (t @ t).double().cpu().numpy()
    torch.backends.cuda.matmul.allow_tf32 = True
    rel = lambda C: np.linalg.norm(C - ref) / np.linalg.norm(ref)
    print(f"n={n:5d} cuBLAS tf32 {rel(c_tf32):.2e}  cuBLAS fp32 (no TF32) {rel(c_f32):.2e}", flush=True)
