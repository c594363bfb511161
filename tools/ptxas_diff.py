"""Per-kernel registers / spills from two ptxas -v logs (old vs new build)."""
import re, sys
def parse(p):
    out, cur = {}, None
    for ln in open(p):
        m = re.search(r"Compiling entry function '(\S+)'", ln)
        if m: cur = m.group(1); continue
        m = re.search(r"(\d+) bytes spill stores", ln)
        if m and cur: out.setdefault(cur, {})["spill"] = int(m.group(1))
        m = re.search(r"Used (\d+) registers", ln)
        if m and cur: out.setdefault(cur, {})["regs"] = int(m.group(1))
    return out
a, b = parse(sys.argv[1]), parse(sys.argv[2])
import subprocess
for k in sorted(set(a) | set(b)):
    if a.get(k) != b.get(k):
        name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        print(a.get(k), "->", b.get(k), name[:110])
