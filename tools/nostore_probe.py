"""Power experiment at c4: the same chain with the epilogue's stores skipped (PSD_DEBUG_NOSTORE,
operand buffers keep the realistic values of a previous full run), to see how much of the power
budget (and so of the SM clock) the epilogue's stores cost.  Results are wrong by design."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PSD_NO_GRAPH"] = "1"
import torch
import bench
import synth
from paper_2507_09165_b200 import Filter, filters
cfg = bench.CONFIGS["c4"]
X = bench.make_inputs(cfg, 0, 32, synth.SEED_BASE).cuda()
out = torch.empty_like(X)
f = Filter(filters.half_filter())
for _ in range(3):
    f.project(X, out=out)
torch.cuda.synchronize()
for mode in ["normal", "nostore", "normal"]:
    if mode == "nostore":
        os.environ["PSD_DEBUG_NOSTORE"] = "1"
    else:
        os.environ.pop("PSD_DEBUG_NOSTORE", None)
    f.project(X, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    with bench.ClockSampler(0) as clk:
        a.record()
        for _ in range(20):
            f.project(X, out=out)
        b.record(); torch.cuda.synchronize()
    print(f"{mode}: {a.elapsed_time(b) / 20:.2f} ms/step, clocks {clk.summary()}", flush=True)
