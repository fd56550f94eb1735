"""c3 latency: chain kernel vs per-product launches (PSD_NO_CHAIN), fp16 and fp16x3."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_09165_b200 import Filter, filters
for n, batch in [(1024, 1), (512, 1), (2048, 1), (384, 24)]:
    X = torch.randn(batch, n, n, device="cuda"); X = (X + X.transpose(1, 2)) / 2
    for prec in ["fp16", "fp16x3"]:
        for mode in ["chain", "nochain", "cs2"]:
            os.environ["PSD_CHAIN"] = "1"; os.environ.pop("PSD_NO_CHAIN", None); os.environ.pop("PSD_CHAIN_CS", None)
            if mode == "nochain": os.environ["PSD_NO_CHAIN"] = "1"
            if mode == "cs2": os.environ["PSD_CHAIN_CS"] = "2"
            f = Filter(filters.remez_half_prefix(6), precision=prec)
            out = torch.empty_like(X)
            for _ in range(5): f.project(X, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            reps = 50
            e0.record()
            for _ in range(reps): f.project(X, out=out)
            e1.record(); torch.cuda.synchronize()
            print(f"n={n} batch={batch} {prec} {mode}: {e0.elapsed_time(e1) / reps * 1000:.1f} us/projection", flush=True)
