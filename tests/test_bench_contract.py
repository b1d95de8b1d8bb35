"""bench.py's JSON-line contract on small sizes (needs a B200).

Runs both arms the way the driver does (one process, N = 1) on config 0 with
small config-2/3/4 sizes and checks every key the contract asks for: metric,
value, steps / warmup, timing fields, roofline, cpu_baseline, e2e with the
copied bytes, gpu_launches, clocks, the per-config records with their parity
verdicts, and the reference arm's line.
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SMALL = ["--config", "cfg0", "--steps", "3", "--warmup", "3", "--cfg2-size", "2048", "--cfg3-size", "512",
         "--cfg4-size", "1024", "--e2e-steps", "2", "--cpu-sample-rows", "64", "--extra-reps", "2"]


def _run(extra, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + SMALL + extra, capture_output=True,
                       text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run([])
    for k in ("metric", "unit", "dtype", "data", "scaling"):
        assert isinstance(d[k], str) and d[k]
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["vs_baseline"] is None
    assert d["config"]["workload"] == "cfg0"
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert 0 < rf["frac"] <= 1.2 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("reference", "port") and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    ck = d["clocks"]
    assert ck["sm_max_mhz"] > 0 and isinstance(ck["reasons"], list)
    assert d["parity"]["bit_exact"] is True
    c = d["configs"]
    assert c["cfg2"]["parity"]["bit_exact"] is True and c["cfg2"]["roofline"]["frac"] > 0
    for name in ("cfg3", "cfg4"):
        rec = c[name]
        assert rec["exact"]["tflops"] > 0 and rec["fused"]["tflops"] > 0
        assert rec["parity"]["oracle"]["exact_mode_bit_exact"] is True
        assert rec["parity"]["fused"]["within_tolerance"] is True


def test_bench_reference_arm_line():
    d = _run(["--impl", "reference"])
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "blocks/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_bench_two_ranks_relaunch():
    """--gpus 2 without a launcher re-executes under torchrun; gloo lets both ranks
    share the one GPU for the plumbing (not for timing): the line says n_gpus 2 and
    the sharded configs carry their bitwise cross-checks."""
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    d = _run(["--gpus", "2"], env=env)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["parity"]["bit_exact"] is True
    assert d["configs"]["cfg2"]["parity"]["bit_exact"] is True
    for name in ("cfg3", "cfg4"):
        assert d["configs"][name]["fused_peer_gather"]["equals_nccl_path"] is True
