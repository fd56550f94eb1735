"""FP32-class split paths on the 'dominant' family (eigenvalues ~1e-3 in the filter's
transition region beside one dominant eigenvalue): relative error vs the float64 oracle with
the GPU's lambda~ for fp16x3 / bf16x3 / tf32x3 at several n."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
from oracle import chain, tables
from paper_2507_09165_b200 import Filter, filters
st_o = (tables.F_SINGLE_REFINED, tables.single_kappas(10))
for n in [512, 1024, 2048]:
    for fam in ["dominant", "goe"]:
        X = synth.batch(fam, n, 2, 900 + n)
        refs = None
        row = []
        for prec in ["fp16x3", "bf16x3", "tf32x3"]:
            f = Filter(filters.single_filter(), precision=prec)
            lam = torch.zeros(2, dtype=torch.float64, device="cuda")
            P = f.project(torch.tensor(X, dtype=torch.float32, device="cuda"), lambda_out=lam)
            torch.cuda.synchronize()
            P, lam = P.double().cpu().numpy(), lam.cpu().numpy()
            errs = []
            for b in range(2):
                ref, _ = chain.project(X[b], *st_o, lam=float(lam[b]))
                errs.append(np.linalg.norm(P[b] - ref) / np.linalg.norm(ref))
            row.append(f"{prec} {max(errs):.2e}")
        print(f"n={n:5d} {fam:9s} " + "  ".join(row), flush=True)
