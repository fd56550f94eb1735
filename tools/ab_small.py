"""A/B of an env switch on the batched small-n kernel at c2 (4096 x 64x64), same GPU, alternating
(graphs off so the env var is read per call), outputs compared bitwise:
python tools/ab_small.py ENV_VAR [precisions...]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PSD_NO_GRAPH"] = "1"
import torch
import bench
import synth
from paper_2507_09165_b200 import Filter, filters
var = sys.argv[1]
precs = sys.argv[2:] or ["fp16", "fp16x3"]
cfg = bench.CONFIGS["c2"]
X = bench.make_inputs(cfg, 0, cfg["batch"], synth.SEED_BASE).cuda()
out = torch.empty_like(X)
for prec in precs:
    f = Filter(filters.c2_filter(), precision=prec)
    res = {"off": [], "on": []}
    outs = {}
    for rnd in range(5):
        for mode in ["off", "on"]:
            if mode == "on":
                os.environ[var] = "1"
            else:
                os.environ.pop(var, None)
            for _ in range(3):
                f.project(X, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                f.project(X, out=out)
            e1.record()
            torch.cuda.synchronize()
            res[mode].append(e0.elapsed_time(e1) / 20)
            outs[mode] = out.clone()
    os.environ.pop(var, None)
    same = torch.equal(outs["on"], outs["off"])
    md = (outs["on"] - outs["off"]).abs().max().item()
    print(f"{prec}: {var} off {min(res['off']):.4f} ms (median {sorted(res['off'])[2]:.4f}), "
          f"on {min(res['on']):.4f} ms (median {sorted(res['on'])[2]:.4f}); bitwise equal {same}, max diff {md:.3g}")
