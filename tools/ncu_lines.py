"""Per CUDA source line: instructions executed and stall samples of one kernel in an ncu report
(ncu --page source --print-source cuda,sass).  usage: python tools/ncu_lines.py REP [N]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout.splitlines()
agg = collections.defaultdict(lambda: [0, 0, ''])
fname = ''
hdr = None
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == 'File Path':
        fname = row[1].split('/')[-1]
        continue
    if row[0] == 'Line No':
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr) or not row[0].strip().isdigit():
        continue
    try:
        ie = int(row[hdr.index('Instructions Executed')] or 0)
        sp = int(row[hdr.index('Warp Stall Sampling (All Samples)')] or 0)
    except ValueError:
        continue
    k = (fname, int(row[0]))
    agg[k][0] += ie
    agg[k][1] += sp
    agg[k][2] = row[1][:80]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total inst {ti:,} samples {ts:,}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{k[0]:>12}:{k[1]:<5} {v[0]/ti*100:5.1f}% inst {v[1]/ts*100:5.1f}% smp  {v[2].strip()}")
