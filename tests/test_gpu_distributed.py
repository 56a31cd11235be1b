"""The multi-GPU path on real GPUs with NCCL (one process per GPU,
torch.distributed): the config-3 search sharded over the ranks and combined
with one all-reduce equals one GPU searching the whole space; a sharded trace
batch equals the same traces on one GPU.  Runs whenever >= 2 GPUs are
visible (gpurun --gpus 2); the gloo world-2 test covers the host logic."""

import os
import pathlib
import socket
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _gpus() -> int:
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2, 4])
def test_nccl_search_and_sharded_replay(world):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tests" / "nccl_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ))
    assert r.returncode == 0 and "NCCL_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
