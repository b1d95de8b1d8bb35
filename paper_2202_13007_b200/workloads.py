"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset exists for this path; BASELINE.json defines the input
distributions and these generators follow them (choices BASELINE leaves open
are documented in DESIGN.md):

* cfg0/cfg2/cfg3 ``smooth_field``: sum of 4 sinusoids, frequencies U[0,0.05]
  cycles/element (x and y), amplitudes U[0.5,2], phases U[0,2pi), plus
  N(0, 1e-3) noise.
* cfg1 ``quadratic_blocks``: per 8x8 block a+bx+cy+dxy+ex^2+fy^2 with
  coefficients N(0,1) and block-local x = 0.1*j, y = 0.1*i.
* cfg4 ``rough_uniform``: i.i.d. U[-1,1].

Torch does the generation (CPU for small parity cases, CUDA for full sizes);
the same seed on the same device type gives the same bits.
"""
from __future__ import annotations

import math

import torch


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def smooth_field(rows: int, cols: int, seed: int, device="cpu", row0: int = 0) -> torch.Tensor:
    """Rows row0..row0+rows-1 of the seeded smooth field (so shards agree with the whole)."""
    gp = _gen(seed, "cpu")  # sinusoid parameters always from the CPU generator
    p = torch.rand((4, 4), generator=gp, dtype=torch.float64)
    fx, fy = 0.05 * p[:, 0], 0.05 * p[:, 1]
    amp, ph = 0.5 + 1.5 * p[:, 2], 2 * math.pi * p[:, 3]
    i = torch.arange(row0, row0 + rows, dtype=torch.float64, device=device).view(-1, 1)
    j = torch.arange(cols, dtype=torch.float64, device=device).view(1, -1)
    out = torch.zeros((rows, cols), dtype=torch.float64, device=device)
    for k in range(4):
        out += float(amp[k]) * torch.sin(2 * math.pi * (float(fx[k]) * j + float(fy[k]) * i) + float(ph[k]))
    g = _gen(seed * 1000003 + row0, device)
    out += 1e-3 * torch.randn((rows, cols), generator=g, dtype=torch.float64, device=device)
    return out


def quadratic_blocks(rows: int, cols: int, seed: int, device="cpu") -> torch.Tensor:
    br, bc = (rows + 7) // 8, (cols + 7) // 8
    g = _gen(seed, device)
    c = torch.randn((6, br, 1, bc, 1), generator=g, dtype=torch.float64, device=device)
    y = 0.1 * torch.arange(8, dtype=torch.float64, device=device).view(1, 8, 1, 1)
    x = 0.1 * torch.arange(8, dtype=torch.float64, device=device).view(1, 1, 1, 8)
    v = c[0] + c[1] * x + c[2] * y + c[3] * x * y + c[4] * x * x + c[5] * y * y  # (br, 8, bc, 8)
    return v.reshape(br * 8, bc * 8)[:rows, :cols].contiguous()


def rough_uniform(rows: int, cols: int, seed: int, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    return torch.rand((rows, cols), generator=g, dtype=torch.float64, device=device) * 2.0 - 1.0


def make(config: str, rows: int, cols: int, seed: int, device="cpu") -> torch.Tensor:
    if config in ("cfg0", "cfg2", "cfg3", "smooth"):
        return smooth_field(rows, cols, seed, device)
    if config in ("cfg1", "quadratic"):
        return quadratic_blocks(rows, cols, seed, device)
    if config in ("cfg4", "rough"):
        return rough_uniform(rows, cols, seed, device)
    raise ValueError(config)
