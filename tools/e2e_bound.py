"""What bounds e2e at c4: pinned H2D and D2H alone and concurrently (two streams), the projection
alone, and the projection with both copy directions running beside it."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_09165_b200 import Filter, filters
n, batch = 4096, 32
Xh = torch.randn(batch, n, n).pin_memory()
Oh = torch.empty_like(Xh).pin_memory()
Xd = torch.randn(batch, n, n, device="cuda"); Xd = (Xd + Xd.transpose(1, 2)) / 2
Od = torch.empty_like(Xd)
Cd = torch.empty(batch // 2, n, n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
f = Filter(filters.half_filter())
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
half = batch // 2
gb = half * n * n * 4 / 1e9
def h2d():
    with torch.cuda.stream(s1): Cd.copy_(Xh[:half], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): Oh[:half].copy_(Cd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    with torch.cuda.stream(s1): Cd.copy_(Xh[:half], non_blocking=True)
    with torch.cuda.stream(s2): Oh[half:].copy_(Od[:half], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
print(f"H2D alone {gb / timed(h2d) * 1e3:.1f} GB/s; D2H alone {gb / timed(d2h) * 1e3:.1f} GB/s; "
      f"concurrent: {gb / timed(both) * 1e3:.1f} GB/s each direction", flush=True)
tp = timed(lambda: f.project(Xd, out=Od))
def proj_and_copies():
    with torch.cuda.stream(s1): Cd.copy_(Xh[:half], non_blocking=True)
    with torch.cuda.stream(s2): Oh[half:].copy_(Od[half:], non_blocking=True)
    f.project(Xd, out=Od)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
tpc = timed(proj_and_copies)
print(f"projection alone {tp:.2f} ms ({batch / tp * 1e3:.0f}/s); with {gb:.1f} GB each way beside it {tpc:.2f} ms", flush=True)
Xs = (Xh + Xh.transpose(1, 2)).mul_(0.5).pin_memory()
th = timed(lambda: f.project_host(Xs, out=Oh, chunks=16))
print(f"project_host (16 chunks) {th:.2f} ms ({batch / th * 1e3:.0f}/s)", flush=True)
