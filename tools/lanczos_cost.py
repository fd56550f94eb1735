"""Cost of the Lanczos/Theorem-2 bound (default: the c4 shape, n = 4096, batch 32; argv: n batch), CUDA
events, warm.

Times psd_project with the Frobenius and the Lanczos bound for f~*_half (T = 7, 22 products) and
for a product-free filter (one degree-1 stage: the bound + scale + reconstruction only), so the
bound's own cost is the difference of the two product-free runs."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_09165_b200 as pkg
import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 32
uniq = min(4, batch)
X = torch.tensor(synth.batch("goe", n, uniq, 5), dtype=torch.float32, device="cuda")
X = X.repeat(batch // uniq, 1, 1).contiguous()
out = torch.empty_like(X)


def timed(f, reps=5):
    for _ in range(3):
        f.project(X, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f.project(X, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
for name, stages in [("half", pkg.filters.half_filter()), ("none", [[1.0]])]:
    for bnd in ("frobenius", "lanczos"):
        res[(name, bnd)] = timed(pkg.Filter(stages, bound=bnd))
        print(f"{name:5s} {bnd:9s} {res[(name, bnd)]:8.3f} ms", flush=True)
bound = res[("none", "lanczos")] - res[("none", "frobenius")]
chain = res[("half", "frobenius")]
print(f"lanczos bound cost {bound:.3f} ms = {bound / chain:.1%} of the f~*_half projection; "
      f"end to end {res[('half', 'lanczos')] / chain - 1:+.1%}")
