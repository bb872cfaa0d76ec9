"""Write a markdown summary of one profiling round into profiles/: per-kernel share of the launch
list (ncu gpu__time_duration, cold-cache serialised: compare SHARES) and the key ncu --set full
metrics of each captured kernel.   usage: python tools/profile_report.py TAG [title]"""
import collections
import csv
import glob
import io
import os
import subprocess
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        agg[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean (us) | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    return "\n".join(out)


def main():
    tag = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else tag
    g = os.path.join(ROOT, "gpurun_out")
    lines = [f"# ncu summary {tag}: {title}", ""]
    lc = os.path.join(g, f"{tag}_launches.csv")
    if os.path.exists(lc):
        lines += ["## Launch list (bench.py --views 2 --steps 2 --warmup 3; ncu --metrics gpu__time_duration.sum "
                  "--clock-control none)", "", launch_shares(lc), ""]
    for rep in sorted(glob.glob(os.path.join(g, f"{tag}_*.ncu-rep"))):
        buf = io.StringIO()
        with redirect_stdout(buf):
            ncu_summary.summary(rep)
        lines += ["```", buf.getvalue().rstrip(), "```", ""]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    out = os.path.join(ROOT, "profiles", f"{tag}.md")
    open(out, "w").write("\n".join(lines))
    print(out)


if __name__ == "__main__":
    main()
