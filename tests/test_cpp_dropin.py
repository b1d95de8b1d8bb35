"""C++ drop-in (include/blaz/blaz.hpp over libblaz_cuda.so) on the GPU.

* tests/cpp/dropin_test: our C++ suite, drop-in vs the C oracle port, bitwise.
* oracle/_ref/ref_{matrix,block_ops,codec,dct,io,bench}_test_on_dropin: the
  REFERENCE's own proj/tests/*_test.cpp (all six files), compiled from
  /root/reference against the drop-in header instead of the reference headers
  (oracle/Makefile target dropin-ref-tests; built where /root/reference
  exists, shipped to the GPU box as binaries).
"""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BINARIES = [
    os.path.join(ROOT, "tests", "cpp", "dropin_test"),
    os.path.join(ROOT, "oracle", "_ref", "ref_matrix_test_on_dropin"),
    os.path.join(ROOT, "oracle", "_ref", "ref_block_ops_test_on_dropin"),
    os.path.join(ROOT, "oracle", "_ref", "ref_io_test_on_dropin"),
    os.path.join(ROOT, "oracle", "_ref", "ref_bench_test_on_dropin"),
    os.path.join(ROOT, "oracle", "_ref", "ref_codec_test_on_dropin"),
    os.path.join(ROOT, "oracle", "_ref", "ref_dct_test_on_dropin"),
]


@pytest.mark.parametrize("binary", BINARIES, ids=os.path.basename)
def test_cpp_suite(binary):
    if not os.path.exists(binary):
        if "_ref" in binary:
            pytest.skip("reference test binaries are built only where /root/reference exists")
        pytest.fail(f"{binary} not built (run __graft_entry__.build())")
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "0 failed" in r.stdout
