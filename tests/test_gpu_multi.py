"""Multi-GPU engines on real GPUs (one process per GPU, torchrun + NCCL).

Spawns ``tests/dist_check_worker.py`` under ``torch.distributed.run`` on 2
GPUs (and 4 when visible), which checks the peer engine (one persistent
kernel across GPUs over CUDA-IPC peer memory) and the NCCL host level loop,
both executor policies, ``bfs_batch`` (full and per-rank outputs) and a DPG1
round trip against the oracle (the reference's multi-worker run_bfs,
engine.py:98-330 with comm.py:75-197).  Skips on a one-GPU box; the
host-side logic of the multi-process path is covered on CPU by
tests/test_dist_gloo.py.
"""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "dist_check_worker.py")


def _gpus():
    from paper_1803_03922_b200 import _lib
    return _lib.device_count()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(n, *args, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), WORKER, *map(str, args)]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("n,scale,graph", [(2, 17, "rmat"), (2, 16, "er"), (4, 18, "rmat")])
def test_distributed_engines_match_oracle(n, scale, graph):
    have = _gpus()
    if have < n:
        pytest.skip(f"needs {n} GPUs, {have} visible")
    rc, out = _torchrun(n, scale, "-", *(["er"] if graph == "er" else []))
    assert rc == 0 and "DIST CHECK PASS" in out, out[-4000:]
