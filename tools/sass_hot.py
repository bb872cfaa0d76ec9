"""Hot SASS of one kernel from an ncu report: instruction executions and stall samples per
instruction, grouped by opcode, plus the hottest basic-block runs (dev tool)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ai, si, ei, smp = h.index('Address'), h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
recs = []
for r in rows[1:]:
    try:
        recs.append((r[ai], r[si].strip(), int(r[ei] or 0), int(r[smp] or 0)))
    except Exception:
        pass
tot = sum(x[2] for x in recs); ts = sum(x[3] for x in recs)
print(f"total inst {tot:,}  samples {ts:,}")
byop = collections.Counter(); bys = collections.Counter()
for a, s, e, p in recs:
    op = s.split()[0] if s else '?'
    if op.startswith('@'):
        op = s.split()[1]
    op = op.split('.')[0]
    byop[op] += e; bys[op] += p
for op, e in byop.most_common(25):
    print(f"  {op:10s} {e/tot*100:5.1f}% inst  {bys[op]/max(ts,1)*100:5.1f}% samples")
if len(sys.argv) > 2 and sys.argv[2].isdigit():
    n = int(sys.argv[2])
    for i, (a, s, e, p) in enumerate(recs):
        if e >= n:
            print(f"{i:5d} {e:>11,} {p:>7,}  {s[:110]}")
if len(sys.argv) > 2 and sys.argv[2] == 'blocks':
    # contiguous runs with equal execution count ~ basic blocks
    runs = []
    cur = None
    for i, (a, s, e, p) in enumerate(recs):
        if cur and cur[2] == e:
            cur[1] = i; cur[3] += p; cur[4] += 1
        else:
            if cur: runs.append(cur)
            cur = [i, i, e, p, 1]
    runs.append(cur)
    runs.sort(key=lambda r: -r[2] * r[4])
    for r in runs[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
        print(f"  [{r[0]:5d}-{r[1]:5d}] n={r[4]:3d} exec={r[2]:>11,}  inst={r[2]*r[4]/tot*100:5.1f}%  samples={r[3]/max(ts,1)*100:5.1f}%   {recs[r[0]][1][:60]}")
