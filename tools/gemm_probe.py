"""Probe: time the c4 chain (batch x n) under different CTA-pair tile orders.

    python tools/gemm_probe.py [--orders row,col,grouped4] [--n 4096] [--batch 32] [--steps 5]

Prints per order: ms per projection step, average product-kernel launch time, TFLOP/s.
Under ncu (--metrics dram__bytes_read.sum ...) run with --steps 1 --warmup 0.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", default="row,col,grouped2,grouped4")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--precision", default="fp16")
    args = ap.parse_args()
    import torch
    from paper_2507_09165_b200 import Filter, filters
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(args.batch, args.n, args.n, device="cuda", generator=g)
    X = (A + A.transpose(1, 2)) * 0.5
    del A
    out = torch.empty_like(X)
    n = args.n
    for order in args.orders.split(","):
        os.environ["PSD_TILE_ORDER"] = order
        f = Filter(filters.half_filter(), precision=args.precision)
        for _ in range(args.warmup):
            f.project(X, out=out)
        torch.cuda.synchronize()
        f.profile_read()
        f.profile(True)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(args.steps):
            f.project(X, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / max(args.steps, 1)
        pms, pl, kl = f.profile_read()
        avg = pms / max(pl, 1)
        tf = n * n * (n + 1) * args.batch / (avg / 1e3) / 1e12
        print(f"order={order:10s} ms/step={ms:8.3f} product_avg_ms={avg:7.3f} TFLOP/s(alg)={tf:7.1f}", flush=True)
        del f


if __name__ == "__main__":
    main()
