"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""
import ctypes
import os
import re

from conftest import ROOT


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for name in os.listdir(inc):
        if not name.endswith(".h"):
            continue
        text = open(os.path.join(inc, name)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(blz_[a-z0-9_]+)\s*\(", text):
            syms.add(m.group(1))
    return syms


def test_library_exports_header_symbols():
    from paper_2202_13007_b200 import _native as N
    lib = ctypes.CDLL(N.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 35, syms
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding covers the whole declared surface
    assert syms == set(N.SIGNATURES), syms ^ set(N.SIGNATURES)


def test_abi_version_and_layout():
    from paper_2202_13007_b200 import _native as N
    lib = N.load()
    assert lib.blz_abi_version() == 1
    assert N.BLOCK_DTYPE.itemsize == 48
    assert N.BLOCK_DTYPE.fields["coeffs"][1] == 17
    # SoA sizing: 45 payload bytes per block plus 256-byte alignment slack per array
    nb = 2048 * 2048
    assert lib.blz_cmat_bytes(16384, 16384) >= 45 * nb
    assert lib.blz_cmat_bytes(16384, 16384) <= 45 * nb + 4 * 256
