"""Summarises an ncu --set full report (per kernel: time, DRAM bytes, pipes, stalls).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--md out.md] [--traffic out.json]
"""
import argparse
import collections
import csv
import io
import json
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--md")
ap.add_argument("--traffic")
args = ap.parse_args()
raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]


def val(r, k, default=0.0):
    if k not in h:
        return default
    s = r[h.index(k)].replace(",", "")
    try:
        return float(s)
    except ValueError:
        return default


def to_mb(r, k):
    u = units[h.index(k)] if k in h else "byte"
    return val(r, k) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)


def to_us(r, k):
    u = units[h.index(k)] if k in h else "ns"
    return val(r, k) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)


seen = collections.OrderedDict()
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("blz::", "")
    if name in seen:
        continue
    st = sorted(((k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), val(r, k))
                 for k in h if k.startswith("smsp__average_warps_issue_stalled")), key=lambda x: -x[1])
    seen[name] = {
        "us": to_us(r, "gpu__time_duration.sum"),
        "read_MB": to_mb(r, "dram__bytes_read.sum"),
        "write_MB": to_mb(r, "dram__bytes_write.sum"),
        "dram_pct": val(r, "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed") or val(r, "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        "issue_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fp64_pct": val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "dmma_pct": val(r, "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
        "alu_pct": val(r, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "warps_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "regs": int(val(r, "launch__registers_per_thread")),
        "stalls": ", ".join(f"{k}={v:.2f}" for k, v in st[:4]),
    }
lines = ["| kernel | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | issue % | FP64 % | DMMA % | ALU % | warps % | regs | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for k, v in seen.items():
    lines.append(f"| {k} | {v['us']:.1f} | {v['read_MB']:.1f} | {v['write_MB']:.1f} | {1000.0 * (v['read_MB'] + v['write_MB']) / max(v['us'], 1e-9):.0f} | "
                 f"{v['issue_pct']:.1f} | {v['fp64_pct']:.1f} | {v['dmma_pct']:.1f} | {v['alu_pct']:.1f} | {v['warps_pct']:.1f} | "
                 f"{v['regs']} | {v['stalls']} |")
out = "\n".join(lines)
print(out)
if args.md:
    with open(args.md, "w") as f:
        f.write(out + "\n")
if args.traffic:
    t = {}
    for k, v in seen.items():
        key = ("decompress" if "decompress" in k else "compress" if "compress_pair" in k else
               "add" if "addsub_v2" in k else "scale" if "scale_v2" in k else k)
        t[key] = (v["read_MB"] + v["write_MB"]) * 1e6
    with open(args.traffic, "w") as f:
        json.dump(t, f, indent=1)
