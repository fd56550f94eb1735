"""Cost of the Lanczos bound vs Frobenius at the bench shapes (CUDA events, warm)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_09165_b200 as pkg
import synth

for n, batch in [(4096, 32), (1024, 1), (64, 4096)]:
    X = torch.tensor(synth.batch("goe", n, min(batch, 4), 5), dtype=torch.float32, device="cuda")
    X = X.repeat((batch + X.shape[0] - 1) // X.shape[0], 1, 1)[:batch].contiguous()
    out = torch.empty_like(X)
    res = {}
    for bnd in ("frobenius", "lanczos"):
        f = pkg.Filter(pkg.filters.half_filter(), bound=bnd)
        for _ in range(3):
            f.project(X, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            f.project(X, out=out)
        e1.record()
        torch.cuda.synchronize()
        res[bnd] = e0.elapsed_time(e1) / reps
    print(f"n={n} batch={batch}: frobenius {res['frobenius']:.3f} ms, lanczos {res['lanczos']:.3f} ms, "
          f"overhead {res['lanczos'] / res['frobenius'] - 1:+.1%}", flush=True)
