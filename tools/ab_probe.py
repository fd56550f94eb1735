"""A/B of an epilogue switch at c4 on the same GPU, alternating (graphs off so the env var is read
per call): python tools/ab_probe.py ENV_VAR[=VALUE]  -- runs with and without ENV_VAR=1, 3 rounds each."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PSD_NO_GRAPH"] = "1"
import torch
import bench
import synth
from paper_2507_09165_b200 import Filter, filters
var, _, val = sys.argv[1].partition("=")   # VAR or VAR=VALUE
val = val or "1"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp16"
cfg = bench.CONFIGS["c4"]
X = bench.make_inputs(cfg, 0, 32, synth.SEED_BASE).cuda()
out = torch.empty_like(X)
f = Filter(filters.half_filter(), precision=prec)
for _ in range(3):
    f.project(X, out=out)
torch.cuda.synchronize()
ref = out.clone()
res = {"off": [], "on": []}
for rnd in range(3):
    for mode in ["off", "on"]:
        if mode == "on":
            os.environ[var] = val
        else:
            os.environ.pop(var, None)
        f.project(X, out=out)
        torch.cuda.synchronize()
        if rnd == 0:
            print(f"{var}={mode}: output bit-identical to reference: {torch.equal(out, ref)}", flush=True)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        with bench.ClockSampler(0) as clk:
            a.record()
            for _ in range(10 if prec == "fp16" else 3):
                f.project(X, out=out)
            b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / (10 if prec == "fp16" else 3)
        res[mode].append(ms)
        print(f"round {rnd} {var}={mode}: {ms:.2f} ms/step, clocks {clk.summary()['sm_mhz']}", flush=True)
print({k: min(v) for k, v in res.items()})
