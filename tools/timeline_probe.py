"""Per-CTA phase stamps of the 1-CTA product kernel over one c3 projection (debug build,
PSD_DEBUG_TIMELINE, graphs off; every product synchronised, so the PDL overlap between products is
not in these numbers -- the kernel bodies are).  Usage: PSD_LIB_VARIANT=debug python tools/timeline_probe.py [prec]"""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PSD_NO_GRAPH"] = "1"
import torch
import synth
from paper_2507_09165_b200 import Filter, filters

prec = sys.argv[1] if len(sys.argv) > 1 else "fp16"
X = torch.tensor(synth.batch("goe", 1024, 1, 5), dtype=torch.float32, device="cuda")
f = Filter(filters.remez_half_prefix(6), precision=prec)
out = torch.empty_like(X)
for _ in range(3):
    f.project(X, out=out)
torch.cuda.synchronize()
os.environ["PSD_DEBUG_TIMELINE"] = "1"
f.project(X, out=out)
torch.cuda.synchronize()
