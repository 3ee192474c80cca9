"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file X.csv) into per-kernel launches / total ns / share.  Usage:
  python scripts/launch_summary.py gpurun_out/launches_k3.csv "<command line>" > profiles/r01/launches_k3_summary.csv"""
import csv
import re
import sys
from collections import defaultdict

SCALE = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9}


def short(name):
    name = re.sub(r"\(.*", "", name)  # drop the argument list
    name = re.sub(r"^void ", "", name)
    return name.replace("drzg::", "")


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    ki, ui, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rd:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        k = short(r[ki])
        tot[k] += v
        cnt[k] += 1
    allns = sum(tot.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none, command: {sys.argv[2] if len(sys.argv) > 2 else '?'}")
    print("# cold-cache serialised launch times: compare shares, not absolutes")
    print("kernel,launches,total_ns,share")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"{k[:140]},{cnt[k]},{int(tot[k])},{tot[k] / allns:.3f}")


if __name__ == "__main__":
    main()
