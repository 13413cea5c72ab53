"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads, and exports every symbol
include/megascan/scan.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "megascan", "scan.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(scan_[a-z_]+)\s*\(", src)))


def test_header_declares_boundary_calls():
    names = _declared()
    for n in ("scan_create", "scan_load_events", "scan_match_collectives", "scan_detect", "scan_localize", "scan_export"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2507_19845_b200 as ms
    so = ms._build.build()
    lib = ctypes.CDLL(so)
    for n in _declared():
        assert hasattr(lib, n), n
    assert set(_declared()) == set(ms.EXPORTED_SYMBOLS)


def test_library_is_sm100a():
    import paper_2507_19845_b200 as ms
    so = ms._build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product path fails loudly instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2507_19845_b200 as ms
    with pytest.raises(ms.ScanError):
        ms.Scan(0)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2507_19845_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.cpp" not in txt, f
