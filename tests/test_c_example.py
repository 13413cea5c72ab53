"""The C ABI used from plain C (examples/c_api_demo.c): it compiles and links against the in-tree
libmegascan.so with gcc on CPU; on a B200 (-m gpu) it runs and checks its own results."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2507_19845_b200")


def _build(tmp_path):
    from paper_2507_19845_b200 import _build as b
    b.build()
    exe = str(tmp_path / "c_api_demo")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", LIBDIR, "-lmegascan",
                           f"-Wl,-rpath,{LIBDIR}", "-o", exe])
    return exe


def test_c_example_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    p = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "instances 12" in p.stdout and "verdict 0 1 label" in p.stdout  # rank 1 ComputeSlow; its own checks pass
