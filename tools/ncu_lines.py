"""Attribute ncu per-instruction stall samples to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [LIB.so] [top]
Uses `ncu --page source --print-source sass` (samples per SASS address) and
`nvdisasm -g` line tables of the same library's cubin (build container)."""
import csv
import io
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
import os
lib = os.path.abspath(sys.argv[3] if len(sys.argv) > 3 else "paper_2112_10239_b200/libtq_engine.so")
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = rows[0][1]
hdr = rows[1]
ia, isrc, isamp, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [(int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iex] or 0)) for r in rows[2:] if r and r[0].startswith("0x")]
base = min(a for a, *_ in data)
# mangled name from the demangled one: find function in cubin listing
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
import glob
dis = "\n".join(subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
                for cub in sorted(glob.glob(tmp + "/*.cubin")))   # one cubin per translation unit
# split functions
funcs = {}
cur = None
for line in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    if cur:
        funcs[cur].append(line)
demangled = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.split("\n")
want = None


def norm(name):
    return name.replace("(int)", "").replace("(bool)1", "true").replace("(bool)0", "false").replace(" ", "")


for mang, dem in zip(funcs, demangled):
    if re.search(kre, dem) and norm(kname) == norm(dem):
        want = mang
if want is None:
    sys.exit(f"no cubin function matches {kname!r}")
lines = {}
curline = None
for l in funcs[want]:
    m = re.search(r'line (\d+)', l)
    if "## File" in l or "//## File" in l:
        m2 = re.search(r'line (\d+)', l)
        mf = re.search(r'File "([^"]+)"', l)
        if m2:
            curline = (mf.group(1) if mf else "?", int(m2.group(1)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/", l)
    if m:
        lines[int(m.group(1), 16)] = curline
agg = defaultdict(lambda: [0, 0])
tot = 0
for a, src, s, ex in data:
    ln = lines.get(a - base)
    agg[ln][0] += s
    agg[ln][1] += ex
    tot += s
srcs = {}


def source_line(key):
    if not key:
        return None, "?"
    path, ln = key
    if not path.endswith(".cu") or not os.path.exists(path):
        return ln, "?(other file: " + os.path.basename(path) + ")"
    if path not in srcs:
        srcs[path] = open(path).read().split("\n")
    lines_ = srcs[path]
    return ln, (lines_[ln - 1].strip()[:90] if ln <= len(lines_) else "?")


print(f"{kname}: {tot} samples")
for key, (s, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    ln, text = source_line(key)
    print(f"{100*s/tot:5.1f}%  inst={ex:>10d}  L{ln}: {text}")
