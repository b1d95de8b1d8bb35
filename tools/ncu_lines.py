"""Per-source-line instruction and stall-sample totals of one kernel in an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep CUBIN KERNEL_SUBSTR SRC_FILE [--blocks N] [--top 30]

CUBIN is the kernel's object extracted with `cuobjdump -xelf all lib.so`; line info comes
from `nvdisasm -gi` (the library is built with -lineinfo).
"""
import argparse
import collections
import csv
import io
import re
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("cubin")
ap.add_argument("kernel")
ap.add_argument("src")
ap.add_argument("--blocks", type=float, default=4194304)
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--ncu-kernel", help="regex for ncu -k (default: KERNEL_SUBSTR)")
a = ap.parse_args()

dis = subprocess.run(["nvdisasm", "-gi", a.cubin], capture_output=True, text=True).stdout
cur, infn, off2line = None, False, {}
for line in dis.splitlines():
    m = re.match(r"\s*\.section\s+\.text\.(\S+?),", line)
    if m:
        infn = a.kernel in m.group(1)
        continue
    m = re.search(r'"([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/", line)
    if m and infn:
        off2line[int(m.group(1), 16)] = cur

raw = subprocess.run(["ncu", "-i", a.rep, "-k", "regex:" + (a.ncu_kernel or a.kernel), "-c", "1", "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
ia, iex, iss, isrc = (h.index(k) for k in ("Address", "Instructions Executed",
                                           "Warp Stall Sampling (All Samples)", "Source"))
base = int(data[0][ia], 16)
byl, byls, byop = collections.Counter(), collections.Counter(), collections.Counter()
for r in data:
    ln = off2line.get(int(r[ia], 16) - base)
    n = float(r[iex] or 0)
    byl[ln] += n
    byls[ln] += float(r[iss] or 0)
    op = [o for o in r[isrc].split() if not o.startswith("@")]
    byop[op[0].split(".")[0] if op else "?"] += n
nb = a.blocks
print(f"warp-instructions per unit: {sum(byl.values()) / nb:.2f}")
print("by opcode:", {k: round(v / nb, 2) for k, v in byop.most_common(18)})
ts = sum(byls.values()) or 1
src = open(a.src).read().split("\n")
for ln, v in byl.most_common(a.top):
    text = src[ln[1] - 1].strip()[:80] if ln and a.src.endswith(ln[0]) else ""
    print(f"{v / nb:7.2f} {100 * byls[ln] / ts:5.1f}%  {ln[0] if ln else '?'}:{ln[1] if ln else ''}  {text}")
