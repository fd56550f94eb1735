"""Diagnostic: small-n kernel parity across (n, filter, precision, batch)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
from oracle import chain
from paper_2507_09165_b200 import Filter, filters

FILT = {"half": filters.half_filter(), "single": filters.single_filter(), "c2": filters.c2_filter(),
        "c1": filters.remez_half_prefix(3), "t4": filters.half_filter()[:4], "t5": filters.half_filter()[:5]}
for n in [int(a) for a in sys.argv[1].split(",")]:
    for fname in sys.argv[2].split(","):
        for prec in sys.argv[3].split(","):
            for batch in [int(a) for a in sys.argv[4].split(",")]:
                X = synth.batch("goe", n, batch, 1234 + n)
                st = FILT[fname]
                f = Filter(st, precision=prec)
                Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
                lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
                P = f.project(Xd, lambda_out=lam).double().cpu().numpy()
                errs = []
                for b in range(batch):
                    ref, _ = chain.project(X[b], st, lam=float(lam[b]))
                    errs.append(np.linalg.norm(P[b] - ref) / np.linalg.norm(ref))
                print(f"n={n:3d} filt={fname:6s} prec={prec:6s} batch={batch}: " + " ".join("%.1e" % e for e in errs), flush=True)
