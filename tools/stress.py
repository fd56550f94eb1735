"""Randomised parity sweep (seeded): n, batch, precision, family, mode drawn at random, every case
vs the float64 oracle with the GPU's lambda~ -- beyond the fixed test matrix (odd paddings, the
1-CTA / CTA-pair switch, upper-only storage on both, split and tf32 paths, sign and ADMM)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
from oracle import admm, chain, polar, tables
from paper_2507_09165_b200 import Filter, filters

TOL = {"fp16": 5e-3, "bf16": 3e-2, "tf32": 5e-3, "fp16x3": 1e-5, "bf16x3": 1e-4}
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 2025)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
small = len(sys.argv) > 3 and sys.argv[3] == "small"     # n <= 64 sweep
t0 = time.time()
worst = {}
fails = 0
for c in range(cases):
    if small:   # the batched small-n kernel (n <= 64, fp16 / fp16x3) and its neighbours
        n = int(rng.choice([3, 8, 17, 31, 33, 48, 63, 64, 64]))
        batch = int(rng.integers(1, 600))
    else:
        n = int(rng.choice([65, 96, 130, 255, 257, 384, 511, 640, 777, 1000, 1024, 1100, 1280, 1536, 2048]))
        batch = int(rng.integers(1, 13 if n <= 1100 else 6))
    prec = str(rng.choice(["fp16", "fp16x3", "fp16", "fp16x3", "bf16", "tf32"] if small else
                          ["fp16", "fp16", "bf16", "tf32", "fp16x3", "bf16x3"]))
    fam = str(rng.choice(["goe", "haar", "sdp_shaped", "dominant"]))
    mode = str(rng.choice(["project", "project", "sign", "admm"] + ([] if small else ["polar"])))
    single = prec.endswith("x3")
    st_p = filters.single_filter() if single else filters.half_filter()
    st_o = (tables.F_SINGLE_REFINED, tables.single_kappas(10)) if single else (tables.F_HALF_REFINED, tables.half_kappas(7))
    f = Filter(st_p, precision=prec)
    b_check = sorted({0, batch - 1})
    if mode == "polar":
        # a general rows x cols input (psd_polar_rect): the block-restricted products on H = [[0,A],[A^T,0]]
        cols = int(rng.choice([n, max(1, n // 2), min(2048, n + 37)]))
        A = np.stack([np.asarray(synth.ginibre(max(n, cols), 1000 * c + b), dtype=np.float64)[:n, :cols]
                      for b in range(batch)])
        Ad = torch.tensor(A, dtype=torch.float32, device="cuda")
        lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
        U = f.polar(Ad, lambda_out=lam)
        torch.cuda.synchronize()
        U, lam = U.double().cpu().numpy(), lam.cpu().numpy()
        errs = []
        for b in b_check:
            ref, _ = polar.polar(A[b], *st_o, lam=float(lam[b]))
            errs.append(np.linalg.norm(U[b] - ref) / np.linalg.norm(ref))
        fam = f"{n}x{cols}"
    elif mode == "admm":
        Cs, Ks, ys = zip(*(synth.maxcut_admm(n, 1000 * c + b) for b in range(batch)))
        C, K, y = np.stack(Cs), np.stack(Ks), np.stack(ys)
        dev = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda").contiguous()
        S, Xn = f.admm_update(dev(C), dev(K), dev(y), 1.5)
        torch.cuda.synchronize()
        S = S.double().cpu().numpy()
        errs = []
        for b in b_check:
            M = admm.form_argument(C[b], K[b], y[b], 1.5)
            Sr, _, _ = admm.s_update(C[b], K[b], y[b], 1.5, *st_o, lam=chain.frobenius_bound(M))
            # R12: relative to ||reference||, floored at 1% of ||M|| (a nearly negative-definite input
            # has Pi(M) ~ 0 and its filter output is the method's residual: a relative error
            # against ~0 measures nothing)
            errs.append(np.linalg.norm(S[b] - Sr) / max(np.linalg.norm(Sr), 1e-2 * np.linalg.norm(M)))
    else:
        X = synth.batch(fam, n, batch, 1000 * c)
        Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
        lam = torch.zeros(batch, dtype=torch.float64, device="cuda")
        P = (f.sign if mode == "sign" else f.project)(Xd, lambda_out=lam)
        torch.cuda.synchronize()
        P, lam = P.double().cpu().numpy(), lam.cpu().numpy()
        errs = []
        for b in b_check:
            ref, _ = (chain.sign if mode == "sign" else chain.project)(X[b], *st_o, lam=float(lam[b]))
            # R12 floor, as above (projection of a nearly negative-definite X: ||Pi(X)|| ~ 0)
            errs.append(np.linalg.norm(P[b] - ref) / max(np.linalg.norm(ref), 1e-2 * np.linalg.norm(X[b])))
            assert np.array_equal(P[b], P[b].T)
    e = max(errs)
    # n < 64: the test suite's small-n bar (4x, TOL_SMALL_N: the fp16 rounding model of this
    # algorithm reaches 1.6e-2 on 8x8 inputs)
    bar = TOL[prec] * (10 if mode == "sign" and single else 1) * (2 if n < 96 else 1) * (4 if n < 64 else 1)
    if mode == "sign" and fam == "dominant" and not single:
        # the paper's failure family: eigenvalues ~1e-3 sit in the filter's transition
        # region, where S is ill-conditioned -- the bar is the rounding model: 3 x the change of the
        # float64 sign when only X_0 is rounded to the operand type
        b = b_check[-1]
        lamb = float(lam[b])
        X0 = torch.tensor(X[b] / lamb)
        X0r = (X0.to(torch.bfloat16) if prec == "bf16" else X0.to(torch.float16)).double().numpy()
        S64, _ = chain.sign(X[b], *st_o, lam=lamb)
        Sr, _ = chain.sign(X0r * lamb, *st_o, lam=lamb)
        bar = max(bar, 3 * np.linalg.norm(Sr - S64) / np.linalg.norm(S64))
    ok = e <= bar and f.status() == "PSD_OK"
    fails += not ok
    worst[prec] = max(worst.get(prec, 0.0), e / bar)
    print(f"{'ok  ' if ok else 'FAIL'} n={n:5d} batch={batch:2d} {prec:7s} {fam:10s} {mode:7s} err={e:.2e} bar={bar:.0e}", flush=True)
print(f"{cases - fails}/{cases} passed in {time.time() - t0:.0f} s; worst err/bar per precision: "
      + ", ".join(f"{k} {v:.2f}" for k, v in sorted(worst.items())))
