"""One small invocation of every kernel path, for compute-sanitizer (memcheck / racecheck /
synccheck): python tools/sanitize.py [quick]

Covers: the batched small-n kernel (fp16 / fp16x3, ragged n, sign, ADMM), the 1-CTA product
kernel (fp16, fp16x3, bf16, tf32; cluster split-K with the push reduction), the CTA-pair kernel (fp16, fp16x3 with K-chunked accumulation),
the Lanczos bound, the row-panel paths (NCCL-free virtual ranks, peer-memory virtual ranks), the
pipelined host path and psd_sym_product.  Each case is checked against nothing -- the sanitizer's
report is the result; the parity suite covers correctness."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2507_09165_b200 import Filter, filters

dev = "cuda"


def mats(n, batch, seed=1):
    return torch.tensor(synth.batch("goe", n, batch, seed), dtype=torch.float32, device=dev)


def run(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


half, single, c2 = filters.half_filter(), filters.single_filter(), filters.c2_filter()
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
run("small fp16 n=64", lambda: Filter(c2).project(mats(64, 6)))
run("small fp16x3 n=64", lambda: Filter(c2, precision="fp16x3").project(mats(64, 5)))
run("small fp16 n=17 sign", lambda: Filter(half).sign(mats(17, 3)))
run("small fp16 n=33", lambda: Filter(half).project(mats(33, 7)))


def admm_small():
    C, K = mats(48, 3, 2), mats(48, 3, 3)
    y = torch.randn(3, 48, device=dev)
    Filter(half).admm_update(C, K, y, 1.5)


run("small ADMM n=48", admm_small)
for prec in ["fp16", "fp16x3", "bf16", "tf32"]:
    run(f"1-CTA {prec} n=300", lambda: Filter(single if prec.endswith("x3") else half, precision=prec).project(mats(300, 2)))
run("1-CTA fp16 sign n=200", lambda: Filter(half).sign(mats(200, 2)))
# cluster split-K (KS = 2, st.async push reduction) and the single-CTA two-run equivalent, n = 1024
ns1 = [[1.5, -0.5]]          # one Newton-Schulz stage: 2 products + the reconstruction
run("1-CTA cluster split-K fp16 n=1024 b=1", lambda: Filter(ns1).project(mats(1024, 1)))
run("1-CTA cluster split-K fp16x3 n=1024 b=1", lambda: Filter(ns1, precision="fp16x3").project(mats(1024, 1)))
run("1-CTA K halves fp16 n=1024 b=3", lambda: Filter(ns1).project(mats(1024, 3)))
run("Lanczos fp16 n=300", lambda: Filter(half, bound="lanczos").project(mats(300, 2)))
if not quick:
    run("pair fp16 n=1024 b=8", lambda: Filter(half).project(mats(1024, 8)))
    run("pair fp16x3 n=1024 b=8", lambda: Filter(single, precision="fp16x3").project(mats(1024, 8)))
run("rowpanel virtual fp16 n=512 P=2", lambda: Filter(half).project_rowpanel_virtual(mats(512, 1), 2))
run("rowpanel p2p virtual fp16 n=512 P=2", lambda: Filter(half).project_rowpanel_p2p_virtual(mats(512, 1), 2))
run("host pipeline fp16 n=256 b=9 chunks=4", lambda: Filter(half).project_host(mats(256, 9).cpu().pin_memory(), chunks=4))
run("sym_product fp16 n=256", lambda: Filter(half).sym_product(mats(256, 1), mats(256, 1), mats(256, 1), 2.0, 0.5))
print("all cases ran")
