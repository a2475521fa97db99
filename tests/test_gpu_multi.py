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


def test_single_process_device_group_matches_golden():
    """partition_graph(g, theta, ClusterShape) in ONE process puts worker w on
    GPU w when p GPUs are visible (reference partition.py:47-76 simulates the
    p workers in one process): every golden run with p <= visible GPUs --
    levels, iterations, per-iteration directions / FV / BV / inspections and
    comm accounting incl. local_all2all / uniquify -- equals the reference's;
    benchmark(), bfs() and the certificate work on the group."""
    have = _gpus()
    if have < 2:
        pytest.skip(f"needs >= 2 GPUs, {have} visible")
    import numpy as np

    import paper_1803_03922_b200 as api
    from golden_utils import iter_partitions, load
    from paper_1803_03922_b200.group import GroupPartitionedGraph
    gold = load()
    checked = 0
    for g, p in iter_partitions(gold, max_scale=14):
        P = p["p_rank"] * p["p_gpu"]
        if P < 2 or P > have:
            continue
        a, b, c, dq = g["quads"]
        params = api.RmatParams(scale=g["scale"], seed=g["seed"], edge_factor=g["edge_factor"], a=a, b=b, c=c,
                                d_quad=dq)
        pg = api.partition_graph(api.build_rmat_graph(params), p["theta"], api.ClusterShape(p["p_rank"], p["p_gpu"]),
                                 devices=list(range(P)))  # "auto" would keep graphs this small on one GPU
        assert isinstance(pg, GroupPartitionedGraph) and pg.group.size == P
        assert pg.classification.d == p["d"] and pg.kind_totals == p["kind_totals"]
        assert api.memory_footprint(pg).to_dict() == p["memory"]
        for r in p["runs"]:
            got = api.run_bfs(pg, api.BfsOptions(mode=r["mode"], source=r["source"], local_all2all=r["local_all2all"],
                                                 uniquify=r["uniquify"])).to_dict()
            want = r["report"]
            for key in ("levels_digest", "iterations", "inspections", "b_measured", "per_iteration", "comm"):
                assert got[key] == want[key], (g["scale"], p["theta"], P, r["source"], r["mode"], key)
            checked += 1
        rep = api.benchmark(pg, [r["source"] for r in p["runs"] if not r["local_all2all"] and r["mode"] == "dobfs"],
                            api.BfsOptions())
        for run in rep["runs"]:
            ref = next(x["report"] for x in p["runs"] if x["source"] == run["source"] and x["mode"] == "dobfs"
                       and not x["local_all2all"])
            assert run["levels_digest"] == ref["levels_digest"]
            assert run["total_inspections"] == ref["total_inspections"]
            assert run["mask_bytes"] == ref["comm"]["total_mask_bytes"]
        root = p["runs"][0]["source"]
        lv, pa = api.bfs(pg, root)
        assert api.validate_bfs_tree(pg, root, lv, pa) == 0
        assert np.array_equal(api.bfs(pg, root, parents="min")[0], lv)
        pg.close()
    assert checked > 0


def test_device_group_auto_placement_at_scale():
    """The drop-in call itself: partition_graph(build_rmat_graph(scale 20),
    theta, ClusterShape(1, 2)) spreads the two workers over two GPUs and the
    run equals the oracle's two-worker run_bfs; the group survives a failing
    call (source out of range) and keeps working."""
    have = _gpus()
    if have < 2:
        pytest.skip(f"needs >= 2 GPUs, {have} visible")
    import oracle as O
    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200.group import GroupPartitionedGraph
    scale, theta = 20, 16
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, seed=4)), theta, api.ClusterShape(1, 2))
    assert isinstance(pg, GroupPartitionedGraph)
    og = O.partition_rmat(scale, theta, 1, 2, seed=4)
    for root in (3, 12345):
        for mode in ("dobfs", "bfs"):
            got = api.run_bfs(pg, api.BfsOptions(mode=mode, source=root)).to_dict()
            ref = O.run_bfs(og, root, mode=mode)
            for key in ("levels_digest", "iterations", "inspections", "per_iteration", "comm", "b_measured"):
                assert got[key] == ref[key], (root, mode, key)
    with pytest.raises(ValueError):
        api.run_bfs(pg, api.BfsOptions(source=1 << scale))
    assert api.run_bfs(pg, api.BfsOptions(source=3)).levels_digest == O.run_bfs(og, 3)["levels_digest"]
    pg.close()


def test_nvls_multicast_delegate_masks(monkeypatch):
    """DBFS_NVLS=1: the delegate masks of a device group live in NVSwitch
    multicast memory and F ORs them with one multimem.ld_reduce per word
    (comm.py:75-98); every report equals the oracle's (the peer reads are the
    default path checked above)."""
    have = _gpus()
    if have < 2:
        pytest.skip(f"needs >= 2 GPUs, {have} visible")
    import oracle as O
    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200 import _lib
    monkeypatch.setenv("DBFS_NVLS", "1")
    P = min(have, 4)
    scale, theta = 18, 16
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, seed=2)), theta,
                             api.ClusterShape(1, P), devices=list(range(P)))
    og = O.partition_rmat(scale, theta, 1, P, seed=2)
    for root in (5, 777):
        for mode in ("dobfs", "bfs"):
            got = api.run_bfs(pg, api.BfsOptions(mode=mode, source=root)).to_dict()
            ref = O.run_bfs(og, root, mode=mode)
            for key in ("levels_digest", "iterations", "inspections", "per_iteration", "comm"):
                assert got[key] == ref[key], (root, mode, key)
    active = [_lib.load().dbfs_graph_nvls_active(pt.handle) for pt in pg.parts]
    pg.close()
    if not all(active):
        pytest.skip("NVSwitch multicast unavailable on this box (peer reads were used)")
