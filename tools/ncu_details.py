"""Print selected metrics of an ncu report's details page: python tools/ncu_details.py REP [substr ...]"""
import csv
import subprocess
import sys

KEEP = ['Duration', 'Elapsed Cycles', 'SM Frequency', 'Executed Ipc Active', 'Issue Slots Busy',
        'Registers Per Thread', 'Achieved Active Warps Per SM', 'Theoretical Occupancy', 'Block Limit',
        'No Eligible', 'Eligible Warps', 'Warp Cycles Per Issued', 'Executed Instructions', 'DRAM Throughput',
        'L1/TEX Hit', 'L2 Hit', 'Memory Throughput', 'Compute (SM) Throughput']


def main():
    rep = sys.argv[1]
    keep = sys.argv[2:] or KEEP
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ik, im, iu, iv = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Unit'), h.index('Metric Value')
    for r in rows[1:]:
        if len(r) > iv and r[im] and any(k in r[im] for k in keep):
            print(f'{r[ik][:30]:30s} {r[im][:50]:50s} {r[iv]} {r[iu]}')


if __name__ == '__main__':
    main()
