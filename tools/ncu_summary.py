"""Write profiles/r02_ncu_summary.md from a `ncu --set full` report and an ncu launch list.

Usage: python tools/ncu_summary.py <report.ncu-rep> <launches.csv> <out.md>
"""
import collections
import csv
import io
import subprocess
import sys

rep, launches, out_path = sys.argv[1:4]
KEEP = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Registers Per Thread',
        'Theoretical Occupancy', 'Achieved Occupancy', 'Executed Ipc Active', 'Issue Slots Busy', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Warp Cycles Per Issued Instruction', 'Static Shared Memory Per Block', 'Block Limit Registers',
        'Block Limit Shared Mem']


def short(name):
    return name.split('<')[0].replace('void ', '').replace('pmap::', '').split('(')[0]


txt = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
per = collections.OrderedDict()
for r in rows[1:]:
    d = dict(zip(h, r))
    if d['Metric Name'] in KEEP:
        per.setdefault(short(d['Kernel Name']), {})[d['Metric Name']] = d['Metric Value'] + ' ' + d['Metric Unit']
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
H = rr[0]
stalls, dram = {}, {}
for r in rr[2:]:
    k = short(r[H.index('Kernel Name')])
    st = [(H[i], r[i]) for i in range(len(H))
          if H[i].startswith('smsp__pcsamp_warps_issue_stalled') and not H[i].endswith('not_issued')]
    vals = sorted([(float(v.replace(',', '')), n) for n, v in st if v.replace(',', '').replace('.', '').isdigit()],
                  reverse=True)
    tot = sum(v for v, _ in vals)
    stalls[k] = ', '.join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
                          for v, n in vals[:6])
lines = [l for l in open(launches) if l.startswith('"')]
lr = list(csv.reader(io.StringIO(''.join(lines))))
lh = lr[0]
tot, cnt = collections.Counter(), collections.Counter()
for r in lr[1:]:
    if r[lh.index('Metric Name')] != 'gpu__time_duration.sum':
        continue
    k = short(r[lh.index('Kernel Name')])
    tot[k] += float(r[lh.index('Metric Value')].replace(',', ''))
    cnt[k] += 1
out = ['# ncu summary, round 2 (C3: Wiener velocity, T = 1e7, fp64, 1 B200)', '',
       'Command: `python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-seq` (tools/gpu_final.sh), '
       'final round-2 code.',
       'Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` (r02_launches.csv; cold-cache, '
       'serialised).',
       'Full capture: `ncu --set full --clock-control none --import-source on -k regex:k_lb_pass -s 9 -c 3`.', '',
       '## Launch list (solve kernels)', '', '| kernel | launches | mean µs | share of the solve kernels |',
       '|---|---|---|---|']
solve = {k: v for k, v in tot.items() if k.startswith('k_lb_pass')}
S = sum(solve.values())
for k, v in sorted(solve.items(), key=lambda x: -x[1]):
    m = v / cnt[k]
    out.append(f'| {k} | {cnt[k]} | {m / 1000 if m > 1000 else m:.1f} | {100 * v / S:.1f} % |')
out += ['', '## Full capture']
for k, d in per.items():
    out.append(f'### {k}')
    out += [f'- {m}: {d[m]}' for m in KEEP if m in d]
    out.append(f'- top stall reasons (pc sampling): {stalls.get(k, "")}')
    out.append('')
open(out_path, 'w').write('\n'.join(out) + '\n')
print('\n'.join(out))
