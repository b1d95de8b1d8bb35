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

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1|cfg0|cfg3] [--no-e2e] [--no-cpu-baseline]
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
    "scale": 45 + 45,
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
def cpu_reference_step_fn(cfg, sample_rows, threads):
    """Returns (kind, fn) where fn() runs one config step on a block-row sample and returns seconds."""
    import torch

    from oracle import oracle as O
    from paper_2202_13007_b200 import workloads as W
    rows, cols = sample_rows, cfg["cols"]
    a = W.make(cfg["gen"], rows, cols, seed=1).numpy()
    b = W.make(cfg["gen"], rows, cols, seed=2).numpy()
    del torch
    if O.ref_available():
        r = O.ref()
        ha = r.dense_new(a.ctypes.data, rows, cols)
        hb = r.dense_new(b.ctypes.data, rows, cols)

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


def run_reference_arm(args, cfg, rank, world):
    """--impl reference: the reference's own CPU implementation on host cores."""
    if rank != 0:
        return None
    threads = host_threads()
    sample_rows = args.ref_sample_rows
    kind, used_threads, step = cpu_reference_step_fn(cfg, sample_rows, threads)
    blocks = (sample_rows // 8) * ((cfg["cols"] + 7) // 8)
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    value = blocks * args.steps / total
    sample = (f"{sample_rows}x{cfg['cols']} block-row slice of {args.config} "
              f"({blocks} blocks/step), reference threads={used_threads}")
    line = {
        "metric": "cfg1 pipeline 8x8 blocks/s (compress 2, add, sub, scale, decompress 3)",
        "value": value, "unit": "blocks/s", "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded per-block quadratics, BASELINE cfg1 distribution)",
        "config": {"workload": args.config, "rows": cfg["rows"], "cols": cfg["cols"], "sample_rows": sample_rows},
        "cpu_baseline": {"value": value, "unit": "blocks/s", "cores": used_threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "blocks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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
    cS, cD, cK = (dev.DeviceCMat(rows, cols) for _ in range(3))
    oS, oD, oK = (torch.empty((rows, cols), dtype=torch.float64, device="cuda") for _ in range(3))
    stream = torch.cuda.current_stream()
    ops = ["compress", "compress", "add", "sub", "scale", "decompress", "decompress", "decompress"]

    def step(ev=None):
        calls = [lambda: dev.compress(A, cA), lambda: dev.compress(B, cB), lambda: dev.add(cA, cB, cS),
                 lambda: dev.sub(cA, cB, cD), lambda: dev.scale(cA, 3.5, cK), lambda: dev.decompress(cS, oS),
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
        dev.compress(A, cA)
        ea = torch.cuda.Event()
        ea.record(stream)
        with torch.cuda.stream(s3):
            s3.wait_event(ea)
            dev.scale(cA, 3.5, cK)
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
        parity = spot_parity(A, B, cA, cS, oS, rows, cols)

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
                                    "add+decompress || sub+decompress)"),
                       "ops_timing": "per-op ms from a separate sequential pass (CUDA events between ops)"},
            "ops": op_report,
            "roofline": {"bound": "hbm", "kernel": "k_decompress", "achieved": dec["gbs"], "peak": hbm,
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
    if not args.no_extras and world == 1:
        extras = run_extras(args)
        if line is not None:
            line["configs"] = extras
    return line


def _chunked_compress(gen, rows, cols, seed, chunk_rows=8192):
    """Compresses a rows x cols matrix generated chunk by chunk (bounded memory);
    returns the DeviceCMat and the dense rows of chunk 0 (for parity sampling)."""
    import torch

    from paper_2202_13007_b200 import device as dev
    from paper_2202_13007_b200 import workloads as W
    full = dev.DeviceCMat(rows, cols)
    bc = (cols + 7) // 8
    first_rows = None
    for r0 in range(0, rows, chunk_rows):
        nr = min(chunk_rows, rows - r0)
        if gen == "smooth":
            d = W.smooth_field(nr, cols, seed, device="cuda", row0=r0)
        else:
            d = W.make(gen, nr, cols, seed + r0, device="cuda")
        part = dev.compress(d)
        b0, b1 = (r0 // 8) * bc, (r0 // 8) * bc + part.nblocks
        full.first[b0:b1].copy_(part.first)
        full.slope[b0:b1].copy_(part.slope)
        full.coeffs[b0:b1].copy_(part.coeffs)
        full.scale[b0:b1].copy_(part.scale)
        if r0 == 0:
            first_rows = d[:64].cpu().numpy()
        del d, part
    torch.cuda.synchronize()
    return full, first_rows


def _time(fn, reps, warm=1):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_extras(args):
    """Configs 2, 3 and (one GPU of) 4 of BASELINE.json (reported beside the cfg1 headline)."""
    import numpy as np
    import torch

    from paper_2202_13007_b200 import device as dev
    out = {}
    fp64_peak = 36.6  # TFLOP/s, DMMA/DFMA measured (profiles/r01_fp64_peaks.txt)
    # ---- config 2: row dots + Frobenius of two 65536^2 smooth fields -------------------
    n2 = args.cfg2_size
    A, a_rows = _chunked_compress("smooth", n2, n2, 11)
    B, b_rows = _chunked_compress("smooth", n2, n2, 12)
    r_holder = {}

    def frob():
        r_holder["r"], r_holder["t"] = dev.frobenius(A, B)
    ms = _time(frob, reps=args.extra_reps)
    nb2 = A.nblocks
    rec = {"workload": f"cfg2 rowdot+frobenius {n2}x{n2} (smooth fields)", "ms": round(ms, 3),
           "value": nb2 / (ms * 1e-3), "unit": "block pairs/s",
           "fp64_note": "exact: two reference-order decompressions per block pair (~3.4k FP64 ops) + serial row chains"}
    if not args.no_parity:
        from oracle import oracle as O
        port = O.port()
        bc = (n2 + 7) // 8
        ha, hb = A.to_host(), B.to_host()
        want = port.rowdot(ha.blocks[:8], hb.blocks[:8], 64, n2)
        got = r_holder["r"][:64].cpu().numpy()
        rec["parity"] = {"sampled_rows": 64, "bit_exact": bool(np.array_equal(got.view(np.uint64), want.view(np.uint64)))}
        del ha, hb
    if not args.no_cpu_baseline:
        rec["cpu_baseline"] = cpu_baseline_rowdot(a_rows, b_rows, n2)
    out["cfg2"] = rec
    del A, B, r_holder
    torch.cuda.empty_cache()
    # ---- config 3: compressed matmul 8192^3 ------------------------------------------------
    n3 = args.cfg3_size
    A, a_rows = _chunked_compress("smooth", n3, n3, 21)
    B, _ = _chunked_compress("smooth", n3, n3, 22)
    C = dev.DeviceCMat(n3, n3)
    scratch = dev.matmul_scratch(A, B)
    flops = 2.0 * n3 ** 3
    rec = {"workload": f"cfg3 compressed matmul {n3}^3 (compressed in, compressed out)"}
    for mode, name in ((0, "exact"), (1, "fused_dmma")):
        ms = _time(lambda: dev.matmul(A, B, mode=mode, out=C, scratch=scratch), reps=args.extra_reps)
        tf = flops / (ms * 1e-3) / 1e12
        rec[name] = {"ms": round(ms, 3), "tflops": round(tf, 2), "frac_fp64_peak": round(tf / fp64_peak, 3)}
    rec["exact"]["note"] = "DMUL+DADD in the reference's order: capped at 50% of the FP64 FMA peak"
    rec["fused_dmma"]["note"] = "FP64 tensor cores; = ascending-k FMA chain; tolerance parity"
    if not args.no_parity:
        from oracle import oracle as O
        port = O.port()
        dev.matmul(A, B, mode=0, out=C, scratch=scratch)
        # row block 0 of C vs the oracle (A's first block-row against all of B)
        ha, hb = A.to_host(), B.to_host()
        want = port.mat_mul(ha.blocks[:1], 8, n3, hb.blocks, n3, n3)
        hc = C.to_host().blocks[:1]
        same = all(np.array_equal(np.ascontiguousarray(hc[f]).view(np.uint8), np.ascontiguousarray(want[f]).view(np.uint8))
                   for f in ("first", "slope", "scale_factor", "coeffs"))
        rec["parity"] = {"sampled_block_rows": 1, "exact_mode_bit_exact": bool(same)}
        del ha, hb
    if not args.no_cpu_baseline:
        rec["cpu_baseline"] = cpu_baseline_matmul(a_rows, n3)
    out["cfg3"] = rec
    del A, B, C, scratch
    torch.cuda.empty_cache()
    # ---- config 4 (one GPU of the sharded case): rough-data matmul 32768^3 --------------
    n4 = args.cfg4_size
    if n4 > 0:
        A, a_rows = _chunked_compress("rough", n4, n4, 41)
        B, _ = _chunked_compress("rough", n4, n4, 42)
        C = dev.DeviceCMat(n4, n4)
        scratch = dev.matmul_scratch(A, B)
        flops = 2.0 * n4 ** 3
        rec = {"workload": f"cfg4 compressed matmul {n4}^3, rough U[-1,1] data, one GPU (compressed in and out)"}
        for mode, name in ((1, "fused_dmma"), (0, "exact")):
            ms = _time(lambda: dev.matmul(A, B, mode=mode, out=C, scratch=scratch), reps=1)
            tf = flops / (ms * 1e-3) / 1e12
            rec[name] = {"ms": round(ms, 1), "tflops": round(tf, 2), "frac_fp64_peak": round(tf / fp64_peak, 3)}
        if not args.no_parity:  # C is the exact-mode result (last run)
            from oracle import oracle as O
            if O.ref_available():
                r = O.ref()
                ha, hb = A.to_host(), B.to_host()
                want = r.mat_mul(ha.blocks[:1], 8, n4, hb.blocks, n4, n4, host_threads())
                hc = C.to_host().blocks[:1]
                same = all(np.array_equal(np.ascontiguousarray(hc[f]).view(np.uint8),
                                          np.ascontiguousarray(want[f]).view(np.uint8))
                           for f in ("first", "slope", "scale_factor", "coeffs"))
                rec["parity"] = {"sampled_block_rows": 1, "exact_mode_bit_exact": bool(same),
                                 "against": "the reference (oracle/_ref) mat_mul"}
                del ha, hb
        if not args.no_cpu_baseline:
            rec["cpu_baseline"] = cpu_baseline_matmul(a_rows, n4, gen="rough")
        out["cfg4_1gpu"] = rec
        del A, B, C, scratch
        torch.cuda.empty_cache()
    return out


def _shard_compress(gen, r0, nrows, cols, seed, chunk_rows=8192):
    """Compresses rows [r0, r0 + nrows) of the seeded `gen` field (chunk by chunk)."""
    import torch

    from paper_2202_13007_b200 import device as dev
    from paper_2202_13007_b200 import workloads as W
    out = dev.DeviceCMat(nrows, cols)
    bc = (cols + 7) // 8
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
        del d, part
    torch.cuda.synchronize()
    return out


def run_sharded(args, rank, world, local):
    """--config cfg2 / cfg4: BASELINE configs 2 and 4 block-row sharded over the ranks
    (strong scaling: the total problem is fixed).  cfg2: local row dots, an all-gather of
    the r_i and the ascending total (bit-exact for every world size).  cfg4: A row-sharded,
    compressed B all-gathered every step (45 B/block over NVLink), local matmul."""
    import torch

    from paper_2202_13007_b200 import device as dev
    from paper_2202_13007_b200 import shard as S
    torch.cuda.set_device(local)
    if args.config == "cfg2":
        n = args.cfg2_size
        r0, nr = S.local_rows(n, rank, world)
        A = _shard_compress("smooth", r0, nr, n, 11)
        B = _shard_compress("smooth", r0, nr, n, 12)
        step = lambda: S.rowdot_frobenius(A, B)  # noqa: E731
        units, unit, metric = (n // 8) * ((n + 7) // 8), "block pairs/s", \
            "cfg2 row dots + Frobenius inner product, 8x8 block pairs/s"
        workload = f"cfg2 {n}x{n} smooth fields, block-row shards x{world}, all-gather of r_i + ascending total"
    else:
        n = args.cfg4_size
        r0, nr = S.local_rows(n, rank, world)
        A = _shard_compress("rough", r0, nr, n, 41)
        Bl = _shard_compress("rough", r0, nr, n, 42)
        mode = 1 if args.gemm == "fused" else 0
        step = lambda: S.matmul(A, Bl, n, n, mode=mode)  # noqa: E731
        units, unit, metric = 2.0 * n ** 3, "TFLOP/s", "cfg4 compressed matmul FP64 TFLOP/s"
        workload = (f"cfg4 {n}^3 rough U[-1,1], A row-sharded x{world}, compressed B all-gathered per step, "
                    f"{args.gemm} GEMM")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(world)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    value = units / (ms * 1e-3)
    if unit == "TFLOP/s":
        value /= 1e12
    if rank != 0:
        return None
    return {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded per shard, BASELINE distribution)",
            "config": {"workload": workload, "n": n, "parallelism": f"block-row shards x{world}"},
            "clocks": clk.summary(),
            "e2e": None, "note": "secondary config mode: inputs generated on device; e2e is measured by the cfg1 mode"}


def cpu_baseline_rowdot(a_rows, b_rows, n):
    """Reference decompress_matrix (all host threads) + ascending row sums on a 64-row slice."""
    import numpy as np

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


def cpu_baseline_matmul(a_rows, n, gen="smooth"):
    """Reference mat_mul of an 8-row slice of A by the full B (all host threads)."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    import paper_2202_13007_b200.workloads as W
    r = O.ref()
    threads = host_threads()
    b = W.smooth_field(n, n, 22).numpy() if gen == "smooth" else W.rough_uniform(n, n, 42).numpy()
    ca = r.compress_matrix(a_rows[:8], threads)
    cb = r.compress_matrix(b, threads)
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


def spot_parity(A, B, cA, cS, oS, rows, cols):
    """Bitwise check of 2 sampled block-rows of compress / add / decompress against the oracle."""
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
    # the three decompressed results land in one pinned buffer in turn (same bytes
    # over PCIe; keeps the pinned footprint at ~7 GB per rank for 8-rank runs)
    dS = pinned_dense()
    dD = dK = dS
    npA, npB = hA.numpy(), hB.numpy()
    lib, h = ctx.lib, ctx.handle
    P = lambda a: a.ctypes.data  # noqa: E731

    def step():
        ctx.check(lib.blz_compress_matrix(h, P(npA), rows, cols, P(cA), 0))
        ctx.check(lib.blz_compress_matrix(h, P(npB), rows, cols, P(cB), 0))
        ctx.check(lib.blz_mat_add(h, P(cA), rows, cols, P(cB), rows, cols, P(cS), 0))
        ctx.check(lib.blz_mat_sub(h, P(cA), rows, cols, P(cB), rows, cols, P(cD), 0))
        ctx.check(lib.blz_mat_scale(h, P(cA), rows, cols, 3.5, P(cK), 0))
        for c, d in ((cS, dS), (cD, dD), (cK, dK)):
            ctx.check(lib.blz_decompress_matrix(h, P(c), rows, cols, P(d), 0))

    step()  # warm-up (scratch allocation)
    torch.cuda.synchronize()
    n = max(1, min(args.steps, args.e2e_steps))
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    dt = max_over_ranks(dt, world)
    dense, blk = rows * cols * 8, nb * 48
    h2d = 2 * dense + 2 * (2 * blk) + blk + 3 * blk
    d2h = 2 * blk + 3 * blk + 3 * dense
    ctx.close()
    return {"value": nb * world / dt, "unit": "blocks/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt * 1e3, "steps": n,
            "api": "C ABI host entry points blz_compress_matrix / blz_mat_add / blz_mat_sub / "
                   "blz_mat_scale / blz_decompress_matrix (pinned host buffers)"}


def cpu_baseline(args, cfg):
    threads = host_threads()
    kind, used, step = cpu_reference_step_fn(cfg, args.ref_sample_rows, threads)
    blocks = (args.ref_sample_rows // 8) * ((cfg["cols"] + 7) // 8)
    step()
    times = [step() for _ in range(args.cpu_repeats)]
    med = statistics.median(times)
    return {"value": blocks / med, "unit": "blocks/s", "cores": used, "kind": kind,
            "sample": f"{args.ref_sample_rows}x{cfg['cols']} block-row slice of {args.config} "
                      f"({blocks} blocks), median of {args.cpu_repeats} after 1 warm-up"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg1", choices=sorted(CONFIGS) + ["cfg2", "cfg4"])
    ap.add_argument("--gemm", default="fused", choices=["fused", "exact"], help="cfg4 GEMM mode")
    ap.add_argument("--sequential", action="store_true", help="time the one-stream op order instead of the DAG")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--ref-sample-rows", type=int, default=512)
    ap.add_argument("--cpu-repeats", type=int, default=3)
    ap.add_argument("--no-extras", action="store_true", help="skip the config-2/3 measurements")
    ap.add_argument("--cfg2-size", type=int, default=65536)
    ap.add_argument("--cfg3-size", type=int, default=8192)
    ap.add_argument("--extra-reps", type=int, default=3)
    ap.add_argument("--cfg4-size", type=int, default=32768, help="0 skips the config-4 one-GPU matmul")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps
    cfg = CONFIGS.get(args.config)
    rank, world, local = dist_env()

    if args.config in ("cfg2", "cfg4"):
        if args.impl == "reference":
            if rank == 0:
                print(json.dumps({"impl": "reference", "unavailable": "the reference arm is measured on the cfg1 "
                                  "workload; cfg2/cfg4 report their CPU baselines in the default run's configs"}))
            return
        if world > 1:
            import torch
            import torch.distributed as dist
            backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
        line = run_sharded(args, rank, world, local)
        if line is not None:
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    if args.impl == "reference":
        line = run_reference_arm(args, cfg, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        # one rank per GPU over NCCL; BENCH_DIST_BACKEND=gloo only for exercising the
        # N > 1 plumbing with several ranks on one GPU (no timing meaning)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if backend == "nccl":
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
