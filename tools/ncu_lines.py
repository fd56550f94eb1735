"""Per-source-line instruction and stall shares of an ncu report (source page, cuda+sass):
python tools/ncu_lines.py REP [N]"""
import collections
import csv
import subprocess
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    f = None
    hdr = None
    agg, st, src, ops = collections.Counter(), collections.Counter(), {}, collections.Counter()
    for r in csv.reader(out.splitlines()):
        if len(r) >= 2 and r[0] == 'File Path':
            f = r[1].split('/')[-1]
            continue
        if len(r) >= 2 and r[0] == 'Line No':
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        agg[(f, ln)] += num(r[7])
        st[(f, ln)] += num(r[4])
        src[(f, ln)] = r[1][:90]
    tot, totw = sum(agg.values()), sum(st.values())
    print('warp instructions', tot, 'stall samples', totw)
    for k, c in agg.most_common(top):
        print(f'{k[0]:16s}{k[1]:5d} {c / tot:6.3f} stall {st[k] / max(totw, 1):6.3f}  {src[k]}')
    print('--- by stall samples')
    for k, c in st.most_common(top // 2):
        print(f'{k[0]:16s}{k[1]:5d} {agg[k] / tot:6.3f} stall {c / max(totw, 1):6.3f}  {src[k]}')


if __name__ == '__main__':
    main()
