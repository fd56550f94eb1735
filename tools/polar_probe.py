"""psd_polar: parity against the float64 polar oracle per precision, and the time of one polar iterate
at n = 2048 / 4096 (CUDA events, warm) beside psd_sign at the same n."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from oracle import polar, tables
from paper_2507_09165_b200 import Filter, filters

HALF = (tables.F_HALF_REFINED, tables.half_kappas(7))
SINGLE = (tables.F_SINGLE_REFINED, tables.single_kappas(10))
for n, prec in [(300, "fp16"), (300, "bf16"), (300, "tf32"), (300, "fp16x3"), (300, "tf32x3"), (1024, "fp16"), (1024, "fp16x3")]:
    A = synth.ginibre(n, 11)[None]
    f = Filter(filters.single_filter() if prec.endswith("x3") else filters.half_filter(), precision=prec)
    lam = torch.zeros(1, dtype=torch.float64, device="cuda")
    U = f.polar(torch.tensor(A, dtype=torch.float32, device="cuda"), lambda_out=lam).double().cpu().numpy()
    ref, _ = polar.polar(A[0], *(SINGLE if prec.endswith("x3") else HALF), lam=float(lam[0]))
    print(f"parity n={n:5d} {prec:7s} rel err {np.linalg.norm(U[0] - ref) / np.linalg.norm(ref):.2e}", flush=True)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for n, batch in [(2048, 4), (4096, 4)]:
    A = torch.tensor(np.stack([synth.ginibre(n, b) for b in range(batch)]), dtype=torch.float32, device="cuda")
    X = torch.tensor(synth.batch("goe", n, batch, 3), dtype=torch.float32, device="cuda")
    f = Filter(filters.half_filter())
    out = torch.empty_like(A)
    tp = timed(lambda: f.polar(A, out=out))
    ts = timed(lambda: f.sign(X, out=out))
    print(f"time n={n} batch={batch} fp16: polar {tp:.2f} ms ({tp / batch:.2f} per matrix), sign {ts:.2f} ms "
          f"({ts / batch:.2f} per matrix), ratio {tp / ts:.1f}", flush=True)
