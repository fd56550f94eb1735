"""c3 (n = 1024, one matrix, fp16): default per-product launches vs the chain kernel, each with and
without upper-only storage; outputs compared bitwise."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_09165_b200 import Filter, filters
X = torch.randn(1, 1024, 1024, device="cuda"); X = (X + X.transpose(1, 2)) / 2
outs = {}
modes = {"launches+upper": {}, "launches+full": {"PSD_NO_UPPER_ONLY": "1"},
         "chain+upper": {"PSD_CHAIN": "1"}, "chain+full": {"PSD_CHAIN": "1", "PSD_NO_UPPER_ONLY": "1"}}
for rnd in range(3):
    for name, env in modes.items():
        for k in ["PSD_CHAIN", "PSD_NO_UPPER_ONLY"]:
            os.environ.pop(k, None)
        os.environ.update(env)
        f = Filter(filters.remez_half_prefix(6))
        out = torch.empty_like(X)
        for _ in range(5): f.project(X, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(200): f.project(X, out=out)
        b.record(); torch.cuda.synchronize()
        outs[name] = out.clone()
        print(f"round {rnd} {name}: {a.elapsed_time(b) / 200 * 1000:.1f} us/projection", flush=True)
ref = outs["launches+full"]
print({k: bool(torch.equal(v, ref)) for k, v in outs.items()})
