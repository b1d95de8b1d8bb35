#!/usr/bin/env python3
"""Benchmark of the blaz compressed-matrix hot path on B200.

Default workload = BASELINE.json configs[1] ("cfg1"): two 16384x16384 binary64
matrices of seeded per-block quadratic surfaces.  One step = the whole config-1
pipeline on HBM-resident dense inputs:

    compress(A), compress(B) -> A+B, A-B, 3.5*A -> decompress each result

`value` = 8x8 blocks of the input matrix pushed through one step, per second,
summed over ranks (weak scaling: every rank owns its own 16384x16384 pair, the
ops shard by block-rows with no communication).  Per-op blocks/s, GB/s and HBM
fractions are in `ops`; `roofline` is for the dominant kernel (decompress).
`configs` holds BASELINE configs 2-4 block-row sharded over the ranks (strong
scaling, with their collectives) and the fused-GEMM parity statistics.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1|cfg0] [--no-e2e] [--no-cpu-baseline] [--no-extras]

--gpus N without torchrun re-executes itself under torchrun (one rank per GPU).
--impl reference times the reference's own CPU implementation (oracle/_ref) on
the whole config-1 workload on all host cores, without importing our package.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0
BYTES = {  # algorithmic bytes per 8x8 block
    "compress": 512 + 45,
    "decompress": 45 + 512,
    "add": 90 + 45,
    "sub": 90 + 45,
    "scale": 16 + 16,  # metadata-only: f, s read and written; phi / C aliased (32 if aliased)
}
CONFIGS = {
    "cfg0": dict(rows=1024, cols=1024, gen="smooth"),
    "cfg1": dict(rows=16384, cols=16384, gen="quadratic"),
}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", HBM_FALLBACK_GBS)), "measured"
    return HBM_FALLBACK_GBS, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled DURING the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [v for v in sm if smax and v > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# CPU baseline: the reference (oracle/_ref) or the oracle port on host cores
# ---------------------------------------------------------------------------
def load_workloads():
    """paper_2202_13007_b200/workloads.py loaded by path: the generators only need
    torch, and loading them this way keeps the package (and its CUDA library)
    out of the reference arm's process."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_blz_workloads", os.path.join(ROOT, "paper_2202_13007_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def cpu_reference_step_fn(cfg, sample_rows, threads):
    """Returns (kind, threads, fn) where fn() runs one config step on the first
    `sample_rows` rows of the workload and returns seconds."""
    from oracle import oracle as O
    W = load_workloads()
    rows, cols = sample_rows, cfg["cols"]
    a = W.make(cfg["gen"], rows, cols, seed=1).numpy()
    b = W.make(cfg["gen"], rows, cols, seed=2).numpy()
    if O.ref_available():
        r = O.ref()
        ha = r.dense_new(a.ctypes.data, rows, cols)
        hb = r.dense_new(b.ctypes.data, rows, cols)
        del a, b

        def step():
            t0 = time.perf_counter()
            ca = r.h_compress(ha, threads)
            cb = r.h_compress(hb, threads)
            s = r.h_add(ca, cb, threads)
            d = r.h_sub(ca, cb, threads)
            k = r.h_scale(ca, 3.5, threads)
            outs = [r.h_decompress(x, threads) for x in (s, d, k)]
            dt = time.perf_counter() - t0
            for h in (ca, cb, s, d, k):
                r.cm_free(h)
            for h in outs:
                r.dense_free(h)
            return dt
        return "reference", threads, step
    p = O.port()

    def step():
        t0 = time.perf_counter()
        ca = p.compress_matrix(a)
        cb = p.compress_matrix(b)
        outs = [p.mat_add(ca, cb), p.mat_sub(ca, cb), p.mat_scale(ca, 3.5)]
        for o in outs:
            p.decompress_matrix(o, rows, cols)
        return time.perf_counter() - t0
    return "port", 1, step


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_matmul_full(n, gen, seeds, threads):
    """The reference's mat_mul on the whole n^3 problem, once (compressed in and out)."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    W = load_workloads()
    r = O.ref()
    hs = []
    for sd in seeds:
        d = W.make(gen, n, n, seed=sd).numpy()
        hs.append(r.dense_new(d.ctypes.data, n, n))
        del d
    ca, cb = r.h_compress(hs[0], threads), r.h_compress(hs[1], threads)
    for h in hs:
        r.dense_free(h)
    t0 = time.perf_counter()
    cc = r.h_mul(ca, cb, threads)
    dt = time.perf_counter() - t0
    for h in (ca, cb, cc):
        r.cm_free(h)
    return {"workload": f"{n}^3 compressed matmul, {gen} data (reference mat_mul, whole problem, once)",
            "ms": round(dt * 1e3, 1), "tflops": 2.0 * n ** 3 / dt / 1e12, "cores": threads, "kind": "reference"}


def run_reference_arm(args, cfg, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref, the
    reference headers compiled unmodified) on all host cores, over the SAME
    config-1 workload as our arm (both 16384^2 matrices, every block).  Only
    rank 0 works under torchrun; this process never imports the package."""
    if rank != 0:
        return None
    threads = host_threads()
    rows = cfg["rows"] if args.ref_sample_rows <= 0 else min(cfg["rows"], args.ref_sample_rows)
    kind, used_threads, step = cpu_reference_step_fn(cfg, rows, threads)
    blocks = ((rows + 7) // 8) * ((cfg["cols"] + 7) // 8)
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = blocks * args.steps / total
    whole = rows == cfg["rows"]
    sample = (f"{'the whole' if whole else 'a block-row slice of the'} {rows}x{cfg['cols']} {args.config} "
              f"workload ({blocks} blocks/step), reference threads={used_threads}")
    line = {
        "metric": "cfg1 pipeline 8x8 blocks/s (compress 2, add, sub, scale, decompress 3)",
        "value": value, "unit": "blocks/s", "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded per-block quadratics, BASELINE cfg1 distribution; CPU generator)",
        "config": {"workload": args.config, "rows": cfg["rows"], "cols": cfg["cols"],
                   "blocks_per_matrix": blocks, "timed_rows": rows, "same_config": whole},
        "cpu_baseline": {"value": value, "unit": "blocks/s", "cores": used_threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_extras and args.cfg3_size > 0:
        mm = reference_matmul_full(args.cfg3_size, "smooth", (21, 22), threads)
        if mm is not None:
            line["configs"] = {"cfg3": mm}
    # the reference arm runs the reference alone: our package (and its CUDA library) stays unloaded
    assert not any(m.startswith("paper_2202_13007_b200") for m in sys.modules), "reference arm imported the package"
    return line


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfg, rank, world, local):
    import torch

    import paper_2202_13007_b200 as blz
    from paper_2202_13007_b200 import device as dev
    from paper_2202_13007_b200 import workloads as W

    torch.cuda.set_device(local)
    rows, cols = cfg["rows"], cfg["cols"]
    nb = ((rows + 7) // 8) * ((cols + 7) // 8)
    # weak scaling: rank r owns block-rows [r*BR, (r+1)*BR) of an (N*rows) x cols problem
    A = W.make(cfg["gen"], rows, cols, seed=1 + 1000 * rank, device="cuda")
    B = W.make(cfg["gen"], rows, cols, seed=2 + 1000 * rank, device="cuda")
    ctx = dev.context(local)
    cA, cB = dev.DeviceCMat(rows, cols), dev.DeviceCMat(rows, cols)
    cS, cD = (dev.DeviceCMat(rows, cols) for _ in range(2))
    cK = dev.ScaledCMat(cA)  # 3.5*A: own f / s, phi / C shared with A (metadata-only scale)
    oS, oD, oK = (torch.empty((rows, cols), dtype=torch.float64, device="cuda") for _ in range(3))
    stream = torch.cuda.current_stream()
    ops = ["compress", "compress", "add", "sub", "scale", "decompress", "decompress", "decompress"]

    def step(ev=None):
        calls = [lambda: dev.compress(A, cA), lambda: dev.compress(B, cB), lambda: dev.add(cA, cB, cS),
                 lambda: dev.sub(cA, cB, cD), lambda: dev.scale_meta(cA, 3.5, cK), lambda: dev.decompress(cS, oS),
                 lambda: dev.decompress(cD, oD), lambda: dev.decompress(cK, oK)]
        for n, c in enumerate(calls):
            c()
            if ev is not None:
                ev[n + 1].record(stream)

    # The timed step runs the op graph on three streams: scale -> decompress(3.5 A) starts
    # as soon as A is compressed (overlapping compress(B)); add -> decompress and
    # sub -> decompress run side by side.  Each stream has its own device context
    # (scratch / worklists).  Outputs are bitwise those of the sequential order.
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def step_dag():
        stream = torch.cuda.current_stream()  # the capture stream while a CUDA graph records
        dev.compress(A, cA)
        ea = torch.cuda.Event()
        ea.record(stream)
        with torch.cuda.stream(s3):
            s3.wait_event(ea)
            dev.scale_meta(cA, 3.5, cK)
            dev.decompress(cK, oK)
        dev.compress(B, cB)
        eb = torch.cuda.Event()
        eb.record(stream)
        for s_, fn, out_c, out_d in ((s1, dev.add, cS, oS), (s2, dev.sub, cD, oD)):
            with torch.cuda.stream(s_):
                s_.wait_event(eb)
                fn(cA, cB, out_c)
                dev.decompress(out_c, out_d)
        for s_ in (s1, s2, s3):
            e = torch.cuda.Event()
            e.record(s_)
            stream.wait_event(e)

    timed_step = step if args.sequential else step_dag
    for _ in range(args.warmup):
        step()
        step_dag()
    ctx.sync()
    torch.cuda.synchronize()

    def all_launches():
        return sum(c.launches() for c in dev.contexts(local))

    # The op graph captured once as a CUDA graph and replayed: one launch per step
    # from the host, the kernels' dependencies resolved on the device.
    graph_launches = None
    if args.graph and not args.sequential:
        cap = torch.cuda.Stream()
        with torch.cuda.stream(cap):  # warm the capture stream's context (scratch, worklists) outside capture
            step_dag()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        l_cap = all_launches()
        with torch.cuda.graph(g, stream=cap):
            step_dag()
        graph_launches = all_launches() - l_cap
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        timed_step = g.replay

    # timed region: K steps on the launching stream (the DAG joins back into it)
    l0 = all_launches()
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for k in range(args.steps):
            timed_step()
        end.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = all_launches() - l0
    if graph_launches is not None:  # replays do not pass through the host launch counter
        launches = graph_launches * args.steps
    ctx.sync()
    ms_local = start.elapsed_time(end) / args.steps
    ms = max_over_ranks(ms_local, world)
    # per-op breakdown: a separate sequential pass with events between the ops
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(ops) + 1)] for _ in range(args.steps)]
    torch.cuda.synchronize()
    for k in range(args.steps):
        evs[k][0].record(stream)
        step(evs[k])
    torch.cuda.synchronize()
    per_op = {}
    for n, op in enumerate(ops):
        t = [evs[k][n].elapsed_time(evs[k][n + 1]) for k in range(args.steps)]
        per_op.setdefault(op, []).append(sum(t) / len(t))
    hbm, hbm_kind = measured_peaks()
    op_report = {}
    for op, ts in per_op.items():
        t_ms = sum(ts) / len(ts)
        gbs = BYTES[op] * nb / (t_ms * 1e-3) / 1e9
        op_report[op] = {"ms": round(t_ms, 4), "blocks_per_s": nb / (t_ms * 1e-3), "gbs": round(gbs, 1),
                         "hbm_frac": round(gbs / hbm, 4)}

    # parity spot check of this run's outputs (sampled block-rows vs the oracle)
    parity = None
    if rank == 0 and not args.no_parity:
        parity = spot_parity(A, B, cA, cS, oS, cK, oK, rows, cols)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, A, B, rows, cols, nb, world)

    line = None
    if rank == 0:
        dec = op_report["decompress"]
        traffic = load_traffic("decompress")
        line = {
            "metric": "cfg1 pipeline 8x8 blocks/s (compress 2, add, sub, scale, decompress 3)",
            "value": nb * world / (ms * 1e-3), "unit": "blocks/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded per-block quadratics, BASELINE cfg1 distribution), generated on device",
            "config": {"workload": args.config, "rows": rows, "cols": cols, "blocks_per_matrix": nb,
                       "parallelism": f"block-row shards x{world} (no collective)",
                       "l2": "inputs larger than L2 (2 GiB dense operands, 189 MB compressed)",
                       "mode": "bit-exact: verified fast compress + reference-order kernels (-fmad=false)",
                       "schedule": ("one stream, op order" if args.sequential else
                                    "op graph on 3 streams (scale+decompress overlaps compress(B); "
                                    "add+decompress || sub+decompress)"
                                    + (", captured once as a CUDA graph and replayed" if args.graph else "")),
                       "ops_timing": "per-op ms from a separate sequential pass (CUDA events between ops)"},
            "ops": op_report,
            "roofline": {"bound": "hbm", "kernel": "k_decompress_ub", "achieved": dec["gbs"], "peak": hbm,
                         "peak_kind": hbm_kind, "unit": "GB/s", "frac": dec["hbm_frac"],
                         "bytes_per_block": BYTES["decompress"], "traffic": traffic},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "parity": parity,
            "compress_exact_path_blocks": ctx.stats()["compress_exact_blocks"],
        }
        if e2e is not None:
            line["e2e"] = e2e
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args, cfg)
    del A, B, cA, cB, cS, cD, cK, oS, oD, oK
    torch.cuda.empty_cache()
    if not args.no_extras:
        extras = run_extras(args, rank, world)
        if line is not None:
            line["configs"] = extras
    return line


def _time_dist(fn, reps, world, warm=1):
    """Device ms per call of fn(), after `warm` calls: CUDA events on the launching
    stream between barriers, max over ranks."""
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(e0.elapsed_time(e1) / reps, world)


def _shard_compress(gen, r0, nrows, cols, seed, chunk_rows=8192):
    """Compresses rows [r0, r0 + nrows) of the seeded `gen` field (chunk by chunk,
    bounded memory).  Returns the DeviceCMat and the first 64 dense rows."""
    import torch

    from paper_2202_13007_b200 import device as dev
    from paper_2202_13007_b200 import workloads as W
    out = dev.DeviceCMat(nrows, cols)
    bc = (cols + 7) // 8
    head = None
    for c0 in range(0, nrows, chunk_rows):
        nr = min(chunk_rows, nrows - c0)
        if gen == "smooth":
            d = W.smooth_field(nr, cols, seed, device="cuda", row0=r0 + c0)
        else:
            d = W.make(gen, nr, cols, seed + r0 + c0, device="cuda")
        part = dev.compress(d)
        b0 = (c0 // 8) * bc
        b1 = b0 + part.nblocks
        out.first[b0:b1].copy_(part.first)
        out.slope[b0:b1].copy_(part.slope)
        out.coeffs[b0:b1].copy_(part.coeffs)
        out.scale[b0:b1].copy_(part.scale)
        if c0 == 0:
            head = d[:64].cpu().numpy()
        del d, part
    torch.cuda.synchronize()
    return out, head


def _block_rows(cm, br0, nbr):
    """Host AoS blocks of block-rows [br0, br0 + nbr) of a DeviceCMat (packed on the device)."""
    from paper_2202_13007_b200 import device as dev
    bc = cm.block_cols
    rows = min(8 * nbr, cm.rows - 8 * br0)
    sub = dev.DeviceCMat(rows, cm.cols)
    lo, hi = br0 * bc, (br0 + nbr) * bc
    sub.first.copy_(cm.first[lo:hi])
    sub.slope.copy_(cm.slope[lo:hi])
    sub.coeffs.copy_(cm.coeffs[lo:hi])
    sub.scale.copy_(cm.scale[lo:hi])
    return sub.to_host().blocks


def _same_blocks(x, y):
    return all(np.array_equal(np.ascontiguousarray(x[f]).view(np.uint8), np.ascontiguousarray(y[f]).view(np.uint8))
               for f in ("first", "slope", "scale_factor", "coeffs"))


def fp64_peaks():
    """FP64 roofline denominators measured live on this GPU by
    tools/microbench/fp64_peaks (DFMA / DMMA chains on every SM); falls back to
    the committed measurement (profiles/r01_fp64_peaks.txt) if the binary is absent."""
    exe = os.path.join(ROOT, "tools", "microbench", "fp64_peaks")
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
            for ln in out.splitlines():
                if ln.startswith("{"):
                    d = json.loads(ln)
                    if d.get("ok"):
                        d["kind"] = "measured live (tools/microbench/fp64_peaks)"
                        return d
        except (OSError, subprocess.TimeoutExpired, ValueError):
            pass
    return {"dfma_tops": 18.29, "dfma_tflops": 36.58, "dmma_tflops": 36.6,
            "kind": "committed measurement (profiles/r01_fp64_peaks.txt)"}


# FP64 operations of the reference's own sequence, the algorithmic
# count behind the FP64 rooflines: decompress_block = 28 divisions (dequantize) +
# 2 x 512 mul + 2 x 512 add (idct2, H/dct.hpp:53-70) + 224 (integrate_rows,
# H/codec.hpp:164-174); a row-dot block pair = two decompressions + 64 mul + 64 add.
FP64_OPS_DECOMPRESS = 28 + 2048 + 224
FP64_OPS_ROWDOT_PAIR = 2 * FP64_OPS_DECOMPRESS + 128
# FP64 operations the row-dot kernel executes per block pair (DADD + DMUL + DFMA thread
# instructions / pairs, ncu capture r2_rowdot65k, profiles/r02_ncu_summary.md): the zero
# structure of the 28 kept coefficients and the shared products of the repeated basis entries
# remove a third of the reference sequence's operations, so the pipe fraction uses this count.
FP64_OPS_ROWDOT_PAIR_EXECUTED = 3129


def run_extras(args, rank, world):
    """BASELINE configs 2, 3 and 4, block-row sharded over the ranks (strong scaling:
    the problem is fixed, world=1 is one GPU doing all of it).

    cfg2: local row dots, then an all-gather of the r_i and one ascending total
          (bit-exact for every world size), and the allreduce-of-partials variant.
    cfg3/cfg4: A row-sharded; compressed B all-gathered (45 B/block over NVLink)
          in every step, then the local decompress + GEMM + compress; both GEMM
          modes, with the fused mode's flip counts / tolerances against exact mode."""
    import torch

    from paper_2202_13007_b200 import compare as CMP
    from paper_2202_13007_b200 import device as dev
    from paper_2202_13007_b200 import shard as S
    out = {}
    peaks = fp64_peaks()
    out["fp64_peaks"] = peaks
    fp64_tflops = float(peaks["dfma_tflops"])
    fp64_tops = float(peaks["dfma_tops"])
    # ---- config 2: row dots + Frobenius of two 65536^2 smooth fields -------------------
    n2 = args.cfg2_size
    if n2 > 0:
        r0, nr = S.local_rows(n2, rank, world)
        A, a_head = _shard_compress("smooth", r0, nr, n2, 11)
        B, b_head = _shard_compress("smooth", r0, nr, n2, 12)
        res = {}

        def gather_variant():
            res["r"], res["t"] = S.rowdot_frobenius(A, B)

        def allreduce_variant():
            res["t2"] = S.frobenius_allreduce(A, B)
        # ~15 ms per call: more repetitions than the GEMM configs at negligible cost
        ms = _time_dist(gather_variant, max(10, args.extra_reps), world, warm=3)
        ms_ar = _time_dist(allreduce_variant, max(10, args.extra_reps), world, warm=3)
        pairs = ((n2 + 7) // 8) ** 2
        ach = pairs * FP64_OPS_ROWDOT_PAIR_EXECUTED / (ms * 1e-3) / 1e12
        ach_ref = pairs * FP64_OPS_ROWDOT_PAIR / (ms * 1e-3) / 1e12
        rec = {"workload": f"cfg2 rowdot+frobenius {n2}x{n2} (smooth fields), block-row shards x{world}",
               "ms": round(ms, 3), "value": pairs / (ms * 1e-3), "unit": "block pairs/s",
               "collective": "all-gather of the r_i (8 B/row) + ascending total: bit-exact for every world size",
               "bytes_gathered_per_rank": 8 * n2,
               "allreduce_variant": {"ms": round(ms_ar, 3), "value": pairs / (ms_ar * 1e-3),
                                     "bytes_reduced": 8, "parity": "tolerance (per-rank partials summed by NCCL)"},
               "roofline": {"bound": "fp64", "achieved": round(ach, 3), "peak": round(fp64_tops, 3),
                            "unit": "T FP64 ops/s", "frac": round(ach / fp64_tops, 4),
                            "ops_per_pair": FP64_OPS_ROWDOT_PAIR_EXECUTED,
                            "ops_basis": "FP64 instructions the kernel executes per pair (ncu, profiles/r02_ncu_summary.md)",
                            "reference_sequence_ops_per_pair": FP64_OPS_ROWDOT_PAIR,
                            "reference_sequence_rate": round(ach_ref, 3),
                            "peak_kind": peaks["kind"]}}
        if not args.no_parity:
            tot_g, tot_a = float(res["t"].item()), float(res["t2"].item())
            rec["parity"] = {"allreduce_vs_gather_rel": abs(tot_a - tot_g) / max(abs(tot_g), 1e-300)}
            if rank == 0:
                from oracle import oracle as O
                port = O.port()
                want = port.rowdot(_block_rows(A, 0, 8), _block_rows(B, 0, 8), min(64, nr), n2)
                got = res["r"][: min(64, nr)].cpu().numpy()
                rec["parity"].update({"sampled_rows": int(min(64, nr)),
                                      "bit_exact": bool(np.array_equal(got.view(np.uint64), want.view(np.uint64)))})
        if rank == 0 and not args.no_cpu_baseline and world == 1:
            rec["cpu_baseline"] = cpu_baseline_rowdot(a_head, b_head, n2)
        out["cfg2"] = rec
        del A, B, res
        torch.cuda.empty_cache()
    # ---- configs 3 and 4: compressed matmul -------------------------------------------------
    for name, gen, n, seeds, reps in (("cfg3", "smooth", args.cfg3_size, (21, 22), args.extra_reps),
                                      ("cfg4", "rough", args.cfg4_size, (41, 42), 1)):
        if n <= 0:
            continue
        r0, nr = S.local_rows(n, rank, world)
        A, a_head = _shard_compress(gen, r0, nr, n, seeds[0])
        Bl, _ = _shard_compress(gen, r0, nr, n, seeds[1])
        Bf = S.allgather_cmat(Bl, n, n)
        C = dev.DeviceCMat(nr, n)
        scratch = dev.matmul_scratch(A, Bf)
        flops = 2.0 * n ** 3
        rec = {"workload": (f"{name} compressed matmul {n}^3, {gen} data, A row-sharded x{world}, "
                            f"compressed B all-gathered every step (compressed in and out)"),
               "bytes_gathered_per_rank": int(Bf.nblocks * 45 - Bl.nblocks * 45)}
        for mode, mname in ((1, "fused"), (0, "exact")):
            ms = _time_dist(lambda: S.matmul(A, Bl, n, n, mode=mode, b_full=Bf, out=C, scratch=scratch),
                            reps, world)
            tf = flops / (ms * 1e-3) / 1e12
            rec[mname] = {"ms": round(ms, 3), "tflops": round(tf, 2), "frac_fp64_peak": round(tf / fp64_tflops, 3)}
        rec["exact"]["note"] = "DMUL+DADD in the reference's order: at most 50% of the FP64 FMA peak"
        rec["fused"]["note"] = "FP64 FMA chains (tolerance mode, BLZ_GEMM_FUSED)"
        if world > 1:
            # the same product with the all-gather fused into B's decompression: every
            # rank's shard opened as peer memory (CUDA IPC), read by the kernel itself
            try:
                views = S.peer_shards(Bl, n, n)
                C2 = dev.DeviceCMat(nr, n)
                ms = _time_dist(lambda: S.matmul_peer(A, views, mode=1, out=C2, scratch=scratch), reps, world)
                tf = flops / (ms * 1e-3) / 1e12
                S.matmul(A, Bl, n, n, mode=1, b_full=Bf, out=C, scratch=scratch)
                dev.sync()
                same = torch.tensor([0.0 if all(torch.equal(getattr(C, f), getattr(C2, f))
                                                for f in ("first", "slope", "scale", "coeffs")) else 1.0])
                import torch.distributed as dist
                same = same.cuda() if dist.get_backend() == "nccl" else same
                dist.all_reduce(same)
                rec["fused_peer_gather"] = {"ms": round(ms, 3), "tflops": round(tf, 2),
                                            "equals_nccl_path": bool(same.item() == 0),
                                            "note": "B decompressed straight from the ranks' shards over peer "
                                                    "memory (blz_matmul_gather_dev): no separate all-gather"}
                dist.barrier()
                del views, C2
            except Exception as e:  # peer access unavailable: the NCCL path above stands
                rec["fused_peer_gather"] = {"unavailable": repr(e)[:200]}
        rec["peak"] = {"tflops": round(fp64_tflops, 2), "kind": peaks["kind"]}
        if not args.no_parity:
            # C holds the exact-mode result of the last timed call
            par = {}
            dctx = dev.context()
            dense_x = dev.matmul_dense(A, Bf, mode=0, scratch=scratch)
            cx = dev.compress(dense_x)
            dctx.set_mode(1)  # BLZ_MODE_EXACT: the reference-order compress of the same dense C
            try:
                cx_exact = dev.compress(dense_x)
                dev.sync()
            finally:
                dctx.set_mode(0)
            eq = lambda x, y: all(torch.equal(getattr(x, f), getattr(y, f))  # noqa: E731
                                  for f in ("first", "slope", "scale", "coeffs"))
            bad = torch.tensor([0 if eq(cx, C) else 1, 0 if eq(cx, cx_exact) else 1], dtype=torch.float64,
                               device="cuda")
            if world > 1:
                import torch.distributed as dist
                if dist.get_backend() == "nccl":
                    dist.all_reduce(bad)
                else:
                    h = bad.cpu()
                    dist.all_reduce(h)
                    bad = h
            par["epilogue_equals_compress_of_dense"] = bool(bad[0].item() == 0)
            par["epilogue_fast_equals_exact_compress_every_block"] = bool(bad[1].item() == 0)
            del cx_exact
            dense_f = dev.matmul_dense(A, Bf, mode=1, scratch=scratch)
            cf = dev.compress(dense_f)
            st = CMP.cmat_stats(cf, C)
            st.update(CMP.dense_stats(dense_f, dense_x))
            par["fused"] = CMP.summarize(CMP.allreduce(st))
            del dense_f, cf, dense_x, cx
            if rank == 0:
                # block-rows 0 and the last local one of exact C against the reference itself
                from oracle import oracle as O
                nbr = A.block_rows
                rows_chk = sorted({0, nbr - 1})
                ha = np.concatenate([_block_rows(A, b, 1) for b in rows_chk], axis=0)
                hb = Bf.to_host().blocks
                hc = np.concatenate([_block_rows(C, b, 1) for b in rows_chk], axis=0)
                if O.ref_available():
                    want = O.ref().mat_mul(ha, 8 * len(rows_chk), n, hb, n, n, host_threads())
                    against = "the reference (oracle/_ref) mat_mul"
                else:
                    want = O.port().mat_mul(ha, 8 * len(rows_chk), n, hb, n, n)
                    against = "the C restatement (oracle/blaz_oracle.c)"
                par["oracle"] = {"block_rows": [r0 // 8 + b for b in rows_chk],
                                 "exact_mode_bit_exact": _same_blocks(hc, want), "against": against}
                del hb
            rec["parity"] = par
        if rank == 0 and not args.no_cpu_baseline and world == 1:
            rec["cpu_baseline"] = cpu_baseline_matmul(a_head, n, gen=gen, seed_b=seeds[1])
        out[name] = rec
        del A, Bl, Bf, C, scratch
        torch.cuda.empty_cache()
    return out


def cpu_baseline_rowdot(a_rows, b_rows, n):
    """Reference decompress_matrix (all host threads) + ascending row sums on a 64-row slice."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    r = O.ref()
    threads = host_threads()
    ca = r.compress_matrix(a_rows, threads)
    cb = r.compress_matrix(b_rows, threads)
    t0 = time.perf_counter()
    da = r.decompress_matrix(ca, 64, n, threads)
    db = r.decompress_matrix(cb, 64, n, threads)
    _ = np.einsum("ij,ij->i", da, db)
    dt = time.perf_counter() - t0
    pairs = 8 * ((n + 7) // 8)
    return {"value": pairs / dt, "unit": "block pairs/s", "cores": threads, "kind": "reference",
            "sample": f"64 x {n} slice: reference decompress_matrix of A and B + row sums"}


def cpu_baseline_matmul(a_rows, n, gen="smooth", seed_b=22):
    """Reference mat_mul of an 8-row slice of A by the full B (all host threads)."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    W = load_workloads()
    r = O.ref()
    threads = host_threads()
    b = W.make(gen, n, n, seed_b).numpy()
    ca = r.compress_matrix(a_rows[:8], threads)
    cb = r.compress_matrix(b, threads)
    del b
    t0 = time.perf_counter()
    r.mat_mul(ca, 8, n, cb, n, n, threads)
    dt = time.perf_counter() - t0
    flops = 2.0 * 8 * n * n
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "reference",
            "sample": f"8 x {n} by {n} x {n}: reference mat_mul (includes decompressing all of B)"}


def load_traffic(kernel):
    """dram bytes per launch from the committed ncu summary, if any (profiles/*.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(kernel)
    return None


def spot_parity(A, B, cA, cS, oS, cK, oK, rows, cols):
    """Bitwise check of 2 sampled block-rows of compress / add / scale / decompress against the oracle."""
    import torch

    from oracle import oracle as O
    port = O.port()
    res = {}
    mism = 0
    for br in (0, (rows // 8) // 2):
        r0 = 8 * br
        a = A[r0:r0 + 8].cpu().numpy()
        b = B[r0:r0 + 8].cpu().numpy()
        oa, ob = port.compress_matrix(a), port.compress_matrix(b)
        osum = port.mat_add(oa, ob)
        bc = (cols + 7) // 8
        t0, t1 = br * bc, (br + 1) * bc
        u64 = np.uint64
        mism += int((cA.first[t0:t1].cpu().numpy().view(u64) != oa["first"].reshape(-1).view(u64)).sum())
        mism += int((cA.slope[t0:t1].cpu().numpy().view(u64) != oa["slope"].reshape(-1).view(u64)).sum())
        mism += int((cA.scale[t0:t1].cpu().numpy() != oa["scale_factor"].reshape(-1)).sum())
        mism += int((cA.coeffs[t0:t1].cpu().numpy() != oa["coeffs"].reshape(-1, 28)).sum())
        mism += int((cS.coeffs[t0:t1].cpu().numpy() != osum["coeffs"].reshape(-1, 28)).sum())
        mism += int((cS.slope[t0:t1].cpu().numpy().view(u64) != osum["slope"].reshape(-1).view(u64)).sum())
        dec = port.decompress_matrix(osum, 8, cols)
        mism += int((oS[r0:r0 + 8].cpu().numpy().view(u64) != dec.view(u64)).sum())
        oscl = port.mat_scale(oa, 3.5)
        mism += int((cK.first[t0:t1].cpu().numpy().view(u64) != oscl["first"].reshape(-1).view(u64)).sum())
        mism += int((cK.slope[t0:t1].cpu().numpy().view(u64) != oscl["slope"].reshape(-1).view(u64)).sum())
        mism += int((cK.coeffs[t0:t1].cpu().numpy() != oscl["coeffs"].reshape(-1, 28)).sum())
        deck = port.decompress_matrix(oscl, 8, cols)
        mism += int((oK[r0:r0 + 8].cpu().numpy().view(u64) != deck.view(u64)).sum())
    res["sampled_block_rows"] = 2
    res["mismatches"] = mism
    res["bit_exact"] = mism == 0
    return res


def run_e2e(args, A, B, rows, cols, nb, world):
    """The same pipeline through the reference-facing host C ABI (blz_* host calls),
    from pinned host buffers: H2D and D2H inside the timed region."""
    import torch

    import paper_2202_13007_b200 as blz
    ctx = blz.Context(torch.cuda.current_device())
    hA = torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)
    hB = torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)
    hA.copy_(A)
    hB.copy_(B)
    nbr, nbc = (rows + 7) // 8, (cols + 7) // 8

    def pinned_blocks():
        t = torch.empty(nb * 48, dtype=torch.uint8, pin_memory=True)
        return t.numpy().view(blz.BLOCK_DTYPE).reshape(nbr, nbc)

    def pinned_dense():
        return torch.empty((rows, cols), dtype=torch.float64, pin_memory=True).numpy()

    cA, cB, cS, cD, cK = (pinned_blocks() for _ in range(5))
    recs2 = [pinned_blocks() for _ in range(5)]  # the other parity's records (pipelined steps)
    # the three decompressed results land in one pinned buffer in turn (same bytes
    # over PCIe; keeps the pinned footprint at ~7 GB per rank for 8-rank runs)
    dS = pinned_dense()
    dD = dK = dS
    npA, npB = hA.numpy(), hB.numpy()
    lib, h = ctx.lib, ctx.handle
    P = lambda a: a.ctypes.data  # noqa: E731

    def step(xA, xB, bA, bB, bS, bD, bK, dS, dD, dK):
        ctx.check(lib.blz_compress_matrix(h, P(xA), rows, cols, P(bA), 0))
        ctx.check(lib.blz_compress_matrix(h, P(xB), rows, cols, P(bB), 0))
        ctx.check(lib.blz_mat_add(h, P(bA), rows, cols, P(bB), rows, cols, P(bS), 0))
        ctx.check(lib.blz_mat_sub(h, P(bA), rows, cols, P(bB), rows, cols, P(bD), 0))
        ctx.check(lib.blz_mat_scale(h, P(bA), rows, cols, 3.5, P(bK), 0))
        for c, d in ((bS, dS), (bD, dD), (bK, dK)):
            ctx.check(lib.blz_decompress_matrix(h, P(c), rows, cols, P(d), 0))

    pinned = (npA, npB, cA, cB, cS, cD, cK, dS, dD, dK)
    # The same calls issued as the op graph from two host threads, each with its own
    # context (the drop-in's per-thread contexts): compress(B)'s upload overlaps
    # decompress(3.5 A)'s download, add -> decompress and sub -> decompress run side by
    # side.  Results are those of the sequential order (the calls are independent).
    import threading
    ctx2 = blz.Context(torch.cuda.current_device())
    dS2 = pinned_dense()  # the second thread's decompressed results

    def step_dag(xA, xB, bA, bB, bS, bD, bK, d1, d2):
        h1, h2 = h, ctx2.handle
        ready = threading.Event()
        err = []

        def t2():
            try:
                ready.wait()
                ctx2.check(lib.blz_compress_matrix(h2, P(xB), rows, cols, P(bB), 0))
            except Exception as e:  # re-raised by the caller
                err.append(e)
        th = threading.Thread(target=t2)
        th.start()
        ctx.check(lib.blz_compress_matrix(h1, P(xA), rows, cols, P(bA), 0))
        ready.set()
        ctx.check(lib.blz_mat_scale(h1, P(bA), rows, cols, 3.5, P(bK), 0))
        ctx.check(lib.blz_decompress_matrix(h1, P(bK), rows, cols, P(d1), 0))
        th.join()
        if err:
            raise err[0]

        def t3():
            try:
                ctx2.check(lib.blz_mat_sub(h2, P(bA), rows, cols, P(bB), rows, cols, P(bD), 0))
                ctx2.check(lib.blz_decompress_matrix(h2, P(bD), rows, cols, P(d2), 0))
            except Exception as e:
                err.append(e)
        th = threading.Thread(target=t3)
        th.start()
        ctx.check(lib.blz_mat_add(h1, P(bA), rows, cols, P(bB), rows, cols, P(bS), 0))
        ctx.check(lib.blz_decompress_matrix(h1, P(bS), rows, cols, P(d1), 0))
        th.join()
        if err:
            raise err[0]

    dag = (npA, npB, cA, cB, cS, cD, cK, dS, dS2)

    # A stream of independent steps, pipelined: one host thread issues the
    # upload-side calls of step k+1 (compress A, scale, compress B, add, sub) while a
    # second one issues step k's three decompressions (the downloads); the records
    # are double-buffered by step parity.  Every step's uploads and downloads stay
    # inside the timed region; consecutive steps overlap on PCIe (full duplex).
    recs = [(cA, cB, cS, cD, cK), tuple(recs2)]

    def run_pipe(n_steps):
        ev = {(k, t): threading.Event() for k in range(n_steps) for t in ("k", "s", "d", "done")}
        err = []

        def producer():
            try:
                for k in range(n_steps):
                    if k >= 2:
                        ev[(k - 2, "done")].wait()  # parity k % 2 records are free again
                    bA, bB, bS, bD, bK = recs[k % 2]
                    ctx.check(lib.blz_compress_matrix(h, P(npA), rows, cols, P(bA), 0))
                    ctx.check(lib.blz_mat_scale(h, P(bA), rows, cols, 3.5, P(bK), 0))
                    ev[(k, "k")].set()
                    ctx.check(lib.blz_compress_matrix(h, P(npB), rows, cols, P(bB), 0))
                    ctx.check(lib.blz_mat_add(h, P(bA), rows, cols, P(bB), rows, cols, P(bS), 0))
                    ev[(k, "s")].set()
                    ctx.check(lib.blz_mat_sub(h, P(bA), rows, cols, P(bB), rows, cols, P(bD), 0))
                    ev[(k, "d")].set()
            except Exception as e:  # re-raised by the caller
                err.append(e)
                for x in ev.values():
                    x.set()
        th = threading.Thread(target=producer)
        th.start()
        try:
            for k in range(n_steps):
                bA, bB, bS, bD, bK = recs[k % 2]
                for tag, c in (("k", bK), ("s", bS), ("d", bD)):
                    ev[(k, tag)].wait()
                    if err:
                        break
                    ctx2.check(lib.blz_decompress_matrix(ctx2.handle, P(c), rows, cols, P(dS), 0))
                ev[(k, "done")].set()
        finally:
            for x in ev.values():
                x.set()
            th.join()
        if err:
            raise err[0]

    step(*pinned)  # warm-up (scratch allocation)
    step_dag(*dag)
    run_pipe(2)
    torch.cuda.synchronize()
    n = max(1, min(args.steps, args.e2e_steps))
    dense, blk = rows * cols * 8, nb * 48
    h2d = 2 * dense + 2 * (2 * blk) + blk + 3 * blk
    d2h = 2 * blk + 3 * blk + 3 * dense

    def timed(fn, bufs, reps):
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(reps):
            fn(*bufs)
        torch.cuda.synchronize()
        return max_over_ranks((time.perf_counter() - t0) / reps, world)
    dt_seq = timed(step, pinned, n)
    dt_dag = timed(step_dag, dag, n)
    barrier(world)
    t0 = time.perf_counter()
    run_pipe(n)
    torch.cuda.synchronize()
    dt = max_over_ranks((time.perf_counter() - t0) / n, world)
    res = {"value": nb * world / dt, "unit": "blocks/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": dt * 1e3, "steps": n,
           "api": "C ABI host entry points blz_compress_matrix / blz_mat_add / blz_mat_sub / "
                  "blz_mat_scale / blz_decompress_matrix (pinned host buffers); a stream of independent "
                  "steps, one host thread (context) issuing step k+1's compressions / add / sub / scale "
                  "while a second issues step k's decompressions; every step's H2D and D2H inside the "
                  "timed region (total time / steps)",
           "single_step_dag": {"value": nb * world / dt_dag, "ms_per_step": dt_dag * 1e3,
                               "note": "one step at a time, issued as the op graph from two host threads"},
           "sequential": {"value": nb * world / dt_seq, "ms_per_step": dt_seq * 1e3,
                          "note": "the same calls one after another from one thread"}}
    del dS2
    # the drop-in's usual case: pageable std::vector-like buffers (plain numpy arrays)
    del hA, hB, cA, cB, cS, cD, cK, dS, pinned, dag, recs, recs2
    pA, pB = np.array(npA), np.array(npB)
    del npA, npB
    pbl = [np.zeros((nbr, nbc), blz.BLOCK_DTYPE) for _ in range(5)]
    pd = np.empty((rows, cols), np.float64)
    pageable = (pA, pB, *pbl, pd, pd, pd)
    step(*pageable)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    step(*pageable)
    torch.cuda.synchronize()
    dtp = max_over_ranks(time.perf_counter() - t0, world)
    # the same pipelined stream of steps as the headline, from pageable buffers
    npA, npB, dS = pA, pB, pd
    recs = [tuple(pbl), tuple(np.zeros((nbr, nbc), blz.BLOCK_DTYPE) for _ in range(5))]
    n_pg = max(2, min(4, n))
    run_pipe(2)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    run_pipe(n_pg)
    torch.cuda.synchronize()
    dtpp = max_over_ranks((time.perf_counter() - t0) / n_pg, world)
    res["pageable"] = {"value": nb * world / dtpp, "unit": "blocks/s", "ms_per_step": dtpp * 1e3, "steps": n_pg,
                       "note": "the pipelined stream of steps from pageable host memory (the C++ drop-in's "
                               "std::vector case)",
                       "one_step_sequential": {"value": nb * world / dtp, "ms_per_step": dtp * 1e3}}
    ctx2.close()
    ctx.close()
    return res


def cpu_baseline(args, cfg):
    threads = host_threads()
    kind, used, step = cpu_reference_step_fn(cfg, args.cpu_sample_rows, threads)
    blocks = (args.cpu_sample_rows // 8) * ((cfg["cols"] + 7) // 8)
    step()
    times = [step() for _ in range(args.cpu_repeats)]
    med = statistics.median(times)
    return {"value": blocks / med, "unit": "blocks/s", "cores": used, "kind": kind,
            "sample": f"{args.cpu_sample_rows}x{cfg['cols']} block-row slice of {args.config} "
                      f"({blocks} blocks), median of {args.cpu_repeats} after 1 warm-up"}


def reexec_under_torchrun(n):
    """`bench.py --gpus N` without a launcher: re-run this command under torchrun
    with one rank per GPU (the driver's own launch form)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg1", choices=sorted(CONFIGS))
    ap.add_argument("--sequential", action="store_true", help="time the one-stream op order instead of the DAG")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="issue the op graph from the host each step instead of replaying a captured CUDA graph")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--ref-sample-rows", type=int, default=0,
                    help="reference arm: rows of the workload timed (0 = all of it, the default)")
    ap.add_argument("--cpu-sample-rows", type=int, default=2048, help="our arm's bounded cpu_baseline sample")
    ap.add_argument("--cpu-repeats", type=int, default=5)
    ap.add_argument("--no-extras", action="store_true", help="skip the config-2/3/4 measurements")
    ap.add_argument("--cfg2-size", type=int, default=65536)
    ap.add_argument("--cfg3-size", type=int, default=8192)
    ap.add_argument("--extra-reps", type=int, default=3)
    ap.add_argument("--cfg4-size", type=int, default=32768, help="0 skips config 4")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps
    cfg = CONFIGS.get(args.config)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        reexec_under_torchrun(args.gpus)
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU", file=sys.stderr)
        sys.exit(2)

    if args.impl == "reference":
        line = run_reference_arm(args, cfg, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        # one rank per GPU over NCCL (NCCL_DEBUG=INFO shows the ranks and transports);
        # BENCH_DIST_BACKEND=gloo only exercises the N > 1 plumbing with several ranks
        # on one GPU (no timing meaning)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    line = run_ours(args, cfg, rank, world, local)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
