"""Diagnostic 2: small-n kernel, single stages, sign output, vs oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
from oracle import chain
from paper_2507_09165_b200 import Filter

cases = {"ns1": [(1.5, -0.5)], "ns2": [(1.5, -0.5)] * 2, "d5": [(1.875, -1.25, 0.375)],
         "d5x2": [(1.875, -1.25, 0.375)] * 2, "lin3": [(0.0, 1.0)], "lin5": [(0.0, 0.0, 1.0)]}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
for name, st in cases.items():
    for prec in ["fp16", "fp16x3"]:
        for n_ in [n, 300]:
            X = synth.batch("goe", n_, 2, 99)
            f = Filter(st, precision=prec)
            Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
            lam = torch.zeros(2, dtype=torch.float64, device="cuda")
            S = f.sign(Xd, lambda_out=lam).double().cpu().numpy()
            errs = []
            for b in range(2):
                ref, _ = chain.sign(X[b], st, lam=float(lam[b]))
                errs.append(np.linalg.norm(S[b] - ref) / np.linalg.norm(ref))
                asym = np.abs(S[b] - S[b].T).max()
            print(f"{name:5s} {prec:6s} n={n_:3d} " + " ".join("%.2e" % e for e in errs) + f" asym={asym:.1e}", flush=True)
