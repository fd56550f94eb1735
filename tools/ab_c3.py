"""A/B of PSD_NO_UPPER_ONLY at config c3 (n = 1024, one matrix; graphs on: env read at capture, so
each mode gets its own Filter)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_09165_b200 import Filter, filters
X = torch.randn(1, 1024, 1024, device="cuda"); X = (X + X.transpose(1, 2)) / 2
outs = {}
for rnd in range(3):
    for mode in ["upper_only", "full"]:
        if mode == "full":
            os.environ["PSD_NO_UPPER_ONLY"] = "1"
        else:
            os.environ.pop("PSD_NO_UPPER_ONLY", None)
        f = Filter(filters.remez_half_prefix(6))
        out = torch.empty_like(X)
        for _ in range(5): f.project(X, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(200): f.project(X, out=out)
        b.record(); torch.cuda.synchronize()
        outs[mode] = out.clone()
        print(f"round {rnd} {mode}: {a.elapsed_time(b) / 200 * 1000:.1f} us/projection", flush=True)
print("bit-identical:", torch.equal(outs["upper_only"], outs["full"]))
