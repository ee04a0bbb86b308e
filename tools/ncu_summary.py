"""Print the headline metrics + top stall reasons of every kernel in an .ncu-rep."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Mem Busy', 'Max Bandwidth',
        'Issue Slots Busy', 'Achieved Occupancy', 'Registers Per Thread',
        'Warp Cycles Per Issued Instruction', 'L1/TEX Cache Throughput', 'L2 Cache Throughput',
        'Theoretical Occupancy', 'Memory Throughput', 'Executed Ipc Active']
for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr = r[0]
    seen = {}
    for row in r[1:]:
        d = dict(zip(hdr, row))
        if d['Metric Name'] in WANT:
            seen.setdefault((d['ID'], d['Kernel Name'][:40]), {})[d['Metric Name']] = d['Metric Value'] + ' ' + d['Metric Unit']
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr = r[0]
    stalls = {}
    for row in r[2:]:
        d = dict(zip(hdr, row))
        st = {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''): float(v)
              for h, v in d.items() if h.startswith('smsp__average_warps_issue_stalled_')
              and h.endswith('_per_issue_active.ratio') and v}
        stalls[d['ID']] = sorted(st.items(), key=lambda x: -x[1])[:6]
    for (i, k), m in seen.items():
        print(f'== {rep} [{i}] {k}')
        for n in WANT:
            if n in m:
                print(f'   {n:38s} {m[n]}')
        print('   stalls', [(a, round(b, 1)) for a, b in stalls.get(i, [])])
