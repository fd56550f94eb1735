"""Summarise an ncu session (tools/gpu_session.sh output dir) into profiles/.

    python tools/summarize_ncu.py gpurun_out/<tag> <round-name> [launches.csv] [prof.ncu-rep] [latest.json]

Writes profiles/<round-name>_summary.md (launch-list shares + the top kernel's full-set
metrics) and profiles/ncu_latest.json ({kernel, dram bytes per launch, ...}) which
bench.py reports as roofline.traffic.
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-9))
    tot = sum(sum(v) for v in agg.values())
    return [(k, len(v), sum(v) / len(v), sum(v) / tot) for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            res[k] = (v[i], u[i])
    return res


def main():
    d, name = sys.argv[1], sys.argv[2]
    lfile = sys.argv[3] if len(sys.argv) > 3 else "launches.csv"
    rfile = sys.argv[4] if len(sys.argv) > 4 else "prof_gemm.ncu-rep"
    latest = sys.argv[5] if len(sys.argv) > 5 else "ncu_latest.json"
    lines = [f"# ncu summary: {name}", "", f"Source: `{d}` (tools/gpu_session.sh), B200, `--clock-control none`.", ""]
    lp = os.path.join(d, lfile)
    if os.path.exists(lp):
        lines += ["## Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)", "",
                  "| kernel | launches | avg time | share of step |", "|---|---|---|---|"]
        for k, cnt, avg, share in launch_shares(lp):
            lines.append(f"| `{k[:90]}` | {cnt} | {avg * 1e6:.1f} us | {share:.3f} |")
        lines.append("")
    rep = os.path.join(d, rfile)
    js = {}
    if os.path.exists(rep):
        m = full_metrics(rep)
        lines += ["## Top kernel, `--set full` (one launch)", "", f"`{m['kernel'][:160]}`", "", "| metric | value | unit |",
                  "|---|---|---|"]
        for k in KEYS:
            if k in m:
                lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        rb = float(m["dram__bytes_read.sum"][0].replace(",", "")) * UNIT[m["dram__bytes_read.sum"][1]]
        wb = float(m["dram__bytes_write.sum"][0].replace(",", "")) * UNIT[m["dram__bytes_write.sum"][1]]
        js = {"kernel": m["kernel"], "dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
              "source": f"profiles/{name}_summary.md", "duration": m["gpu__time_duration.sum"],
              "tensor_active_pct": m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", ["?"])[0]}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{name}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if js:
        with open(os.path.join(ROOT, "profiles", latest), "w") as f:
            json.dump(js, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
