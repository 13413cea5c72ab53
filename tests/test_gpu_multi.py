"""Multi-GPU parity (-m gpu, row A9): tests/multigpu_parity.py under torchrun on 2 GPUs (4 when
available): per-shard analyses reassembled == the oracle on the whole trace. Skipped on a box
with fewer than 2 GPUs (the single-GPU parity suite covers the shard's local pass)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("nproc", [2, 4])
def test_multigpu_parity(nproc):
    import torch
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(HERE, "multigpu_parity.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    sys.stdout.write(p.stdout[-6000:])
    sys.stderr.write(p.stderr[-6000:])
    assert p.returncode == 0, f"multi-GPU parity failed (rc={p.returncode})"
