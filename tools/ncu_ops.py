"""Executed-instruction mix by SASS opcode of an ncu report: python tools/ncu_ops.py REP [N]"""
import collections
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    i_s, i_e, i_w = hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
    op, st = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= i_e or not r[i_e].isdigit():
            continue
        toks = r[i_s].split()
        m = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
        m = m.split('.')[0]
        op[m] += int(r[i_e])
        st[m] += int(r[i_w] or 0)
    tot, totw = sum(op.values()), max(sum(st.values()), 1)
    print('total warp instructions', tot)
    for m, c in op.most_common(top):
        print(f'{m:10s} {c:12d} {c / tot:6.3f}  stall {st[m] / totw:6.3f}')


if __name__ == '__main__':
    main()
