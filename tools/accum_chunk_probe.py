"""K-chunked accumulation of the split (FP32-class) path (reading R23): error of one product and
of a whole projection, and the c4 step time, per accumulation run length kchunk (0 = one run).

    python tools/accum_chunk_probe.py            # on a B200 (gpurun)
"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
from oracle import chain, tables
from paper_2507_09165_b200 import Filter, filters

CHUNKS = [0, 256, 512, 1024, 2048]
rng = np.random.default_rng(5)
print("# one product C = X X, fp16-exact symmetric X (only the accumulation errs)")
for n in [1024, 2048, 4096]:
    G = rng.standard_normal((n, n))
    X = ((G + G.T) / 2).astype(np.float16).astype(np.float64)
    ref = X @ X
    iu = np.triu_indices(n)
    t = torch.tensor(X[None], dtype=torch.float32, device="cuda")
    row = []
    for prec in ["fp16x3", "tf32x3"]:
        for kc in CHUNKS:
            f = Filter(filters.half_filter(), precision=prec, accum_chunk=kc)
            C = f.sym_product(t, t).double().cpu().numpy()[0]
            e = np.linalg.norm((C - ref)[iu]) / np.linalg.norm(ref[iu])
            row.append(f"{prec}/{kc} {e:.2e}")
    print(f"n={n:5d} " + "  ".join(row), flush=True)

print("# projection parity, f~*_single + kappa, n = 2048 (batch 1: 1-CTA kernel; batch 3: pair kernel)")
for fam in ["dominant", "goe"]:
    for batch in [1, 3]:
        X = synth.batch(fam, 2048, batch, 2948 + 2048)
        refs = {}
        row = []
        for prec in ["fp16x3", "tf32x3"]:
            for kc in CHUNKS:
                f = Filter(filters.single_filter(), precision=prec, accum_chunk=kc)
                Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
                lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
                P = f.project(Xd, lambda_out=lam).double().cpu().numpy()
                if 0 not in refs:
                    refs[0], _ = chain.project(X[0], tables.F_SINGLE_REFINED, tables.single_kappas(10),
                                               lam=float(lam[0]))
                e = np.linalg.norm(P[0] - refs[0]) / np.linalg.norm(refs[0])
                row.append(f"{prec}/{kc} {e:.2e}")
        print(f"{fam:9s} batch {batch}: " + "  ".join(row), flush=True)

print("# c4 step time (32 x 4096, f~*_single + kappa, 31 products), ms per step")
X = torch.stack([torch.tensor(synth.make("sdp_shaped", 4096, synth.SEED_BASE + b), dtype=torch.float32)
                 for b in range(32)]).cuda()
out = torch.empty_like(X)
for prec in ["fp16x3", "tf32x3"]:
    row = []
    for kc in CHUNKS:
        f = Filter(filters.single_filter(), precision=prec, accum_chunk=kc)
        for _ in range(2):
            f.project(X, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f.project(X, out=out)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{kc}: {e0.elapsed_time(e1) / 5:.1f}")
        del f
    print(f"{prec}: " + "  ".join(row), flush=True)
