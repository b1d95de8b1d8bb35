"""Parity statistics between two compressed results of the same operation.

Used for the tolerance-mode GEMM (``GEMM_FUSED``: FP64 tensor cores / FMA
chains instead of the reference's separately rounded products and sums,
H/matrix.hpp:188-202) against the bit-exact mode, as ``north_star`` asks: phi
and C[28] flips are counted and reported, f and s are compared against a
stated relative tolerance, and the dense results by a normwise error
||x - x_ref||_inf / max(1, ||x_ref||_inf).

Everything is computed on the device with torch reductions; `merge` combines
per-rank statistics (sums of counts, maxima of errors) for sharded runs.
"""
from __future__ import annotations

import torch

# Tolerances stated for the fused GEMM mode (tests/test_fullsize_parity.py asserts them).
FUSED_TOL = {
    "f_normwise": 1e-12,      # max|f - f_ref| / max|f_ref| over the output blocks
    "s_normwise": 1e-12,      # max|s - s_ref| / max|s_ref|
    "dense_normwise": 1e-12,  # ||C - C_ref||_inf / max(1, ||C_ref||_inf)
    "coeff_delta_same_phi": 1,  # where phi agrees, a coefficient may move by at most 1 LSB
    "flip_block_frac": 1e-3,  # at most 0.1 % of the output blocks may differ in phi or C at all
}

_SUMS = ("blocks", "blocks_differing", "blocks_flipped", "phi_flips", "coeff_flips", "coeff_flips_same_phi_gt1")
_MAXS = ("max_coeff_delta", "f_max_abs_diff", "f_max_abs_ref", "s_max_abs_diff", "s_max_abs_ref",
         "dense_max_abs_diff", "dense_max_abs_ref", "f_max_rel", "s_max_rel")


def cmat_stats(got, ref) -> dict:
    """Raw statistics of `got` against `ref` (two DeviceCMat of the same shape)."""
    phi_diff = got.scale != ref.scale
    cd = (got.coeffs.to(torch.int16) - ref.coeffs.to(torch.int16)).abs()
    cflip = cd != 0
    blk_c = cflip.any(dim=1)
    df = (got.first - ref.first).abs()
    ds = (got.slope - ref.slope).abs()
    af, as_ = ref.first.abs(), ref.slope.abs()
    tiny = torch.finfo(torch.float64).tiny
    same_phi = ~phi_diff

    def mx(t):
        return float(t.max()) if t.numel() else 0.0

    return {
        "blocks": int(ref.scale.numel()),
        "blocks_differing": int((phi_diff | blk_c | (df != 0) | (ds != 0)).sum()),
        "blocks_flipped": int((phi_diff | blk_c).sum()),
        "phi_flips": int(phi_diff.sum()),
        "coeff_flips": int(cflip.sum()),
        "coeff_flips_same_phi_gt1": int(((cd > 1) & same_phi.view(-1, 1)).sum()),
        "max_coeff_delta": int(cd.max()) if cd.numel() else 0,
        "f_max_abs_diff": mx(df), "f_max_abs_ref": mx(af),
        "s_max_abs_diff": mx(ds), "s_max_abs_ref": mx(as_),
        "f_max_rel": mx(df / af.clamp_min(tiny)), "s_max_rel": mx(ds / as_.clamp_min(tiny)),
    }


def dense_stats(got: torch.Tensor, ref: torch.Tensor) -> dict:
    return {"dense_max_abs_diff": float((got - ref).abs().max()), "dense_max_abs_ref": float(ref.abs().max())}


def merge(parts: list[dict]) -> dict:
    out = {}
    for k in _SUMS:
        out[k] = sum(p.get(k, 0) for p in parts)
    for k in _MAXS:
        vals = [p[k] for p in parts if k in p]
        if vals:
            out[k] = max(vals)
    return out


def allreduce(stats: dict) -> dict:
    """Combines per-rank statistics over the default process group (no-op without one)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return stats
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    s = torch.tensor([float(stats.get(k, 0)) for k in _SUMS], dtype=torch.float64, device=dev)
    m = torch.tensor([float(stats.get(k, 0.0)) for k in _MAXS], dtype=torch.float64, device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    out = {k: int(v) for k, v in zip(_SUMS, s.tolist())}
    out.update({k: (int(v) if k == "max_coeff_delta" else v) for k, v in zip(_MAXS, m.tolist())})
    return out


def summarize(stats: dict, tol: dict = FUSED_TOL) -> dict:
    """Normwise errors and the verdict against `tol`."""
    s = dict(stats)
    s["f_normwise"] = s["f_max_abs_diff"] / max(s["f_max_abs_ref"], 1e-300)
    s["s_normwise"] = s["s_max_abs_diff"] / max(s["s_max_abs_ref"], 1e-300)
    if "dense_max_abs_diff" in s:
        s["dense_normwise"] = s["dense_max_abs_diff"] / max(1.0, s["dense_max_abs_ref"])
    s["flip_block_frac"] = s["blocks_flipped"] / max(1, s["blocks"])
    checks = {
        "f_normwise": s["f_normwise"] <= tol["f_normwise"],
        "s_normwise": s["s_normwise"] <= tol["s_normwise"],
        "coeff_delta_same_phi": s["coeff_flips_same_phi_gt1"] == 0,
        "flip_block_frac": s["flip_block_frac"] <= tol["flip_block_frac"],
    }
    if "dense_normwise" in s:
        checks["dense_normwise"] = s["dense_normwise"] <= tol["dense_normwise"]
    s["tolerance"] = dict(tol)
    s["within_tolerance"] = all(checks.values())
    s["checks"] = checks
    return s
