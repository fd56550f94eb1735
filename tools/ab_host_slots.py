"""A/B of the host pipeline's chunk-buffer count (PSD_HOST_SLOTS) and chunk count at c4:
project_host on pinned SDP-shaped inputs, alternating, same GPU."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import synth
from paper_2507_09165_b200 import Filter, filters
cfg = bench.CONFIGS["c4"]
Xh = bench.make_inputs(cfg, 0, 32, synth.SEED_BASE).pin_memory()
Oh = torch.empty_like(Xh).pin_memory()
f = Filter(filters.half_filter())
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
variants = [tuple(map(int, v.split(","))) for v in (sys.argv[1:] or ["3,16", "6,16", "8,16", "6,32", "8,32"])]
res = {v: [] for v in variants}
ref = None
for rnd in range(int(os.environ.get("AB_ROUNDS", "3"))):
    for slots, chunks in variants:
        os.environ["PSD_HOST_SLOTS"] = str(slots)
        res[(slots, chunks)].append(timed(lambda: f.project_host(Xh, out=Oh, chunks=chunks)))
        if ref is None:
            ref = Oh.clone()
        elif not torch.equal(ref, Oh):
            print("MISMATCH", slots, chunks)
for (slots, chunks), ts in res.items():
    print(f"slots {slots} chunks {chunks}: best {min(ts):.2f} ms ({32 / min(ts) * 1e3:.0f}/s), all {[round(t, 2) for t in ts]}", flush=True)
