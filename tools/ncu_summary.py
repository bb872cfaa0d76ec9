"""Summarise ncu reports: key throughput/occupancy/stall metrics per kernel (reads .ncu-rep via ncu -i)."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'Issue Slots Busy', 'L1/TEX Hit Rate',
        'L2 Hit Rate', 'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp', 'Executed Instructions',
        'Waves Per SM', 'Block Limit Registers', 'Block Limit Shared Mem', 'Grid Size', 'Block Size',
        'Avg. Not Predicated Off Threads Per Warp']


def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if not rows:
        return
    h = rows[0]
    ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    name = rows[1][ki].split('(')[0] if len(rows) > 1 else path
    print(f"== {name}  ({path})")
    for r in rows[1:]:
        if r[mi] in WANT:
            print(f"   {r[mi]:42s} {r[vi]:>14s} {r[ui]}")
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        hh, units, vals = rr[0], rr[1], rr[2]
        keys = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
                'smsp__inst_executed_op_shared_ld.sum', 'smsp__sass_inst_executed_op_shared_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
        for k in keys:
            if k in hh:
                i = hh.index(k)
                print(f"   {k:42s} {vals[i]:>14s} {units[i]}")
        stall = [(hh[i], vals[i]) for i in range(len(hh)) if hh[i].startswith('smsp__average_warp_latency_issue_stalled') or
                 (hh[i].startswith('smsp__pcsamp_warps_issue_stalled_') and not hh[i].endswith('not_issued'))]
        tot = 0.0
        vv = []
        for k, v in stall:
            try:
                f = float(v.replace(',', ''))
            except ValueError:
                continue
            vv.append((f, k))
            tot += f
        vv.sort(reverse=True)
        if tot:
            print("   top stall reasons (pc sampling):", ", ".join(f"{k.split('stalled_')[-1]}={f / tot:.2f}" for f, k in vv[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summary(p)
