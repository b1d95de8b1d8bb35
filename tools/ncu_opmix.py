"""Warp instructions and stall samples per SASS opcode of one kernel in an ncu report.

    python tools/ncu_opmix.py REPORT.ncu-rep [--blocks N]

Reads `ncu -i REPORT --page source --csv --print-source sass`; with --blocks, the executed
counts are also printed per block (N = blocks the kernel processed).
"""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--blocks", type=float, default=0)
ap.add_argument("--top", type=int, default=16)
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
j = next((k for k in range(i + 1, len(lines)) if lines[k].startswith('"Kernel Name"')), len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[i:j]))))  # the first kernel of the report
h = rows[0]
ci, cs, cn = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
ex, st = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if len(r) <= max(ci, cs, cn) or not r[cn].strip():
        continue
    toks = r[cn].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    ex[op] += float(r[ci].replace(",", "") or 0)
    st[op] += float(r[cs].replace(",", "") or 0)
tot = sum(ex.values())
print(f"total warp instructions {tot:.0f}" + (f" ({tot / args.blocks:.2f} per block)" if args.blocks else ""))
print("| opcode | warp instr | per block | stall samples |")
print("|---|---|---|---|")
for op, n in ex.most_common(args.top):
    pb = f"{n / args.blocks:.2f}" if args.blocks else "-"
    print(f"| {op} | {n:.0f} | {pb} | {st[op]:.0f} |")
