"""Write profiles/ncu_traffic.json (the bench line's roofline.traffic) from ncu summaries.

Usage: python tools/traffic_json.py <round-tag> <summary files ...>
Each summary is a tools/ncu_summary.py output named ncu_<kernel>_<config>.txt; traffic is
dram__bytes_read.sum + dram__bytes_write.sum of the one captured launch."""
import json
import os
import re
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
KERNEL = {"rl": "rl_sweep", "lr": "lr_sweep", "adj": "adj_sweep", "tt": "tt_kernel"}


def dram_bytes(path):
    tot = 0.0
    for line in open(path):
        m = re.match(r"\s*dram__bytes_(read|write)\.sum\s+([\d.]+)\s+(\w+)", line)
        if m:
            tot += float(m.group(2)) * UNITS[m.group(3)]
    return int(round(tot))


def main():
    tag, files = sys.argv[1], sys.argv[2:]
    out = {"_source": f"dram__bytes_read.sum + dram__bytes_write.sum per launch, from the ncu --set full "
                      f"captures summarised in profiles/{tag}_ncu_*.txt (bench.py command, 4th launch of the kernel)"}
    for f in files:
        m = re.match(r".*ncu_(rl|lr|adj|tt)_(\w+)\.txt$", f)
        if m:
            out.setdefault(m.group(2), {})[KERNEL[m.group(1)]] = dram_bytes(f)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
