"""Rounding model of the split (FP32-class) and fp32 arithmetic of Algorithm 2.

Emulates, in numpy, the chain exactly as the planner lays it out (Y = Z Z; U = c_p Y Y + c_{p-1} Y;
U <- Y U + c_j Y; Z' = c_0 Z + Z U; P = 1/2 X + 1/2 lambda~ X_0 S; every product symmetrised from its
upper triangle, addends from the same rounded operand copy, reading R18) under three arithmetics:

  x3   fp16 hi + lo operands (per-buffer power-of-two scale), products hi*hi + hi*lo + lo*hi with
       round-to-nearest fp32 sums, fp32 epilogue  (the FP16X3 path after reading R23)
  x4   x3 plus the lo*lo term
  f32  fp32 operands, fp32 accumulation and epilogue  (what a true FP32 implementation does)

and returns the relative Frobenius error against the float64 oracle (oracle/chain.py).  This is
test / tolerance infrastructure: it derives the parity bars, it is not the product path.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
import numpy as np


def _split16(x, s):
    y = (x * s).astype(np.float32)
    hi = y.astype(np.float16).astype(np.float32)
    lo = (y - hi).astype(np.float16).astype(np.float32)
    return hi, lo


def emulate_project(X, stages, mode, lam, s=2.0 ** 10):
    """P of Algorithm 2 for the folded product-side `stages` under arithmetic `mode`."""
    X0 = X / lam
    sym = lambda M: np.triu(M) + np.triu(M, 1).T

    def store(v):
        if mode == "f64":
            return v
        v32 = v.astype(np.float32)
        if mode == "f32":
            return v32.astype(np.float64)
        hi, lo = _split16(v32, s)
        return (hi.astype(np.float64) + lo.astype(np.float64)) / s

    def prod(A, B):
        if mode == "f64":
            return A @ B
        if mode == "f32":
            return (A.astype(np.float32) @ B.astype(np.float32)).astype(np.float64)
        Ah, Al = _split16(A.astype(np.float32), s)
        Bh, Bl = _split16(B.astype(np.float32), s)
        f = lambda a, b: (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
        acc = f(Ah, Bh) + f(Ah, Bl) + f(Al, Bh)
        if mode == "x4":
            acc = acc + f(Al, Bl)
        return acc.astype(np.float64) / (s * s)

    def epi(alpha, acc, beta, D):
        if mode == "f64":
            return alpha * acc + beta * D
        return (np.float32(alpha) * acc.astype(np.float32) + np.float32(beta) * D.astype(np.float32)).astype(np.float64)

    Z = store(X0)
    for c in stages:
        p = len(c) - 1
        if p == 0:
            Z = store(c[0] * Z)
            continue
        Y = store(sym(prod(Z, Z)))
        if p == 1:
            Z = store(sym(epi(c[1], prod(Z, Y), c[0], Z)))
            continue
        U = store(sym(epi(c[p], prod(Y, Y), c[p - 1], Y)))
        for j in range(p - 2, 0, -1):
            U = store(sym(epi(1.0, prod(Y, U), c[j], Y)))
        Z = store(sym(epi(1.0, prod(Z, U), c[0], Z)))
    return sym(epi(0.5 * lam, prod(store(X0), Z), 0.5, X))


def model_errors(which, n, seeds, modes=("x3", "x4", "f32")):
    """{mode: [relative error vs the float64 oracle per seed]} on GOE inputs."""
    import synth
    from oracle import chain, tables
    from paper_2507_09165_b200 import filters
    prod_st, orc = {"c1": (filters.remez_half_prefix(3), (tables.F_HALF[:3], None)),
                    "c2": (filters.c2_filter(), (filters.c2_filter(), None)),
                    "half": (filters.half_filter(), (tables.F_HALF_REFINED, tables.half_kappas(7))),
                    "single": (filters.single_filter(), (tables.F_SINGLE_REFINED, tables.single_kappas(10)))}[which]
    out = {m: [] for m in modes}
    for seed in seeds:
        X = synth.goe(n, 1000 + seed)
        ref, lam = chain.project(X, *orc)
        for m in modes:
            P = emulate_project(X, prod_st, m, lam)
            out[m].append(float(np.linalg.norm(P - ref) / np.linalg.norm(ref)))
    return out


if __name__ == "__main__":
    for which, n in [("c1", 8), ("c2", 64), ("half", 64), ("single", 256)]:
        e = model_errors(which, n, range(12))
        print(which, n, {m: f"median {np.median(v):.2e} max {np.max(v):.2e}" for m, v in e.items()}, flush=True)
