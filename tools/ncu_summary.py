"""Summarise an ncu --set full report into a short text block (committed under profiles/).

usage: python tools/ncu_summary.py REPORT.ncu-rep [kernel-regex] > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value", "Metric Unit"))
want = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Size", "Grid Size",
        "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM", "No Eligible",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate"]
seen = {}
kname = None
for r in rows[1:]:
    kname = r[ki]
    if r[mi] in want and r[mi] not in seen:
        seen[r[mi]] = f"{r[vi]} {r[ui]}".strip()
print(f"kernel: {kname}")
for w in want:
    if w in seen:
        print(f"  {w:38s} {seen[w]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hdr, unit, val = rr[0], rr[1], rr[2]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.sum",
                 "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                 "sm__warps_active.avg.pct_of_peak_sustained_active"):
        if name in hdr:
            i = hdr.index(name)
            print(f"  {name:60s} {val[i]} {unit[i]}")
    # stall breakdown
    stalls = [(hdr[i], val[i]) for i in range(len(hdr)) if hdr[i].startswith("smsp__average_warp_latency_issue_stalled_") or
              hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")]
    tot = []
    for n, v in stalls:
        try:
            tot.append((float(v.replace(",", "")), n))
        except ValueError:
            pass
    tot.sort(reverse=True)
    print("  top stall reasons (pc samples):")
    for v, n in tot[:8]:
        print(f"    {n:70s} {v:.0f}")
