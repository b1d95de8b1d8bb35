"""Launch-list table from an `ncu --metrics gpu__time_duration.sum --csv --log-file` capture.

    python tools/ncu_launches.py gpurun_out/launches.csv

Prints one markdown row per kernel of ours (namespace blz): launches, mean us, and the share
of our kernel time.  Kernels from torch (synthetic input generation) are left out.
"""
import collections
import csv
import re
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    if "blz::" not in name and not re.match(r"^(void )?k_", name):
        continue
    short = re.sub(r"^void ", "", name)
    short = re.sub(r"blz::(<unnamed>::)?", "", short)
    short = re.sub(r"\(.*$", "", short)
    short = short.replace("(bool)0", "0").replace("(bool)1", "1")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    us = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    rows.append((short, us))

agg = collections.OrderedDict()
for k, us in rows:
    agg.setdefault(k, []).append(us)
total = sum(sum(v) for v in agg.values())
print("| kernel | launches | mean us | share of our kernel time |")
print("|---|---|---|---|")
for k, v in agg.items():
    print(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f}% |")
