"""Top SASS instructions of an ncu report by warp-stall samples, with the per-reason split.

usage: python tools/ncu_sass_top.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
isamp = hdr.index("Warp Stall Sampling (All Samples)")
isrc = hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i != isamp]
data.sort(key=lambda r: -int(r[isamp] or 0))
tot = sum(int(r[isamp] or 0) for r in data)
for r in data[:top]:
    parts = []
    for i in stall_cols:
        try:
            v = float(r[i] or 0)
        except ValueError:
            continue
        if v > 0.05 * int(r[isamp] or 1):
            parts.append(f"{hdr[i]}={v:.0f}")
    print(f"{100 * int(r[isamp]) / tot:5.1f}% {r[0]} {r[isrc].strip()[:60]:60s} {' '.join(parts)[:160]}")
