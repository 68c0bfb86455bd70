"""The library's NCCL transport with more than one rank (the ncclSend/Recv halos,
the coarse AllGather and the NCCL calls inside the captured solve graph had only run on a
communicator of size 1).  Needs two GPUs; skipped on a one-GPU box, where the same exchange
pattern is covered by the loopback ranks (tests/test_gpu_multirank.py) and the gloo replay
(tests/test_slab_decomposition.py)."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("nr", [2, 3])
def test_nccl_slab_solve_matches_one_gpu(nr):
    if torch.cuda.device_count() < nr:
        pytest.skip("needs %d GPUs (the box has %d)" % (nr, torch.cuda.device_count()))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nr),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(HERE, "nccl_slab_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    for r in range(nr):
        assert "NCCL_SLAB_OK rank %d" % r in out.stdout
