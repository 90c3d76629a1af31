"""The NCCL strip partition with one PROCESS per GPU (the production multi-GPU path): real halo
send/recv between ranks, all-reduces, per-iteration CUDA graphs with NCCL nodes.  Needs at least
two GPUs on the box and is skipped otherwise (the pool of these rounds had one per box; the
partitioned arithmetic itself is proven on one GPU by tests/test_gpu_strips.py through the
in-process group transport)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nproc", [2, 4])
def test_nccl_strips_one_process_per_gpu(nproc):
    if not torch.cuda.is_available() or torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "scripts", "nccl_strip_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("nccl strips ok") == 2
