"""CPU: host-side logic of the reference-facing API (no device work)."""

import math

import numpy as np
import pytest

import oracle as O
from paper_1803_03922_b200 import traversal
from paper_1803_03922_b200.engine import BfsOptions, compute_teps, levels_digest
from paper_1803_03922_b200.partition import ClusterShape
from paper_1803_03922_b200.rmat import RmatParams, ResourceError
from paper_1803_03922_b200.storage import CsrSubgraph


def test_cluster_shape_parse_and_mapping():
    s = ClusterShape.parse("2x2x2")
    assert (s.p_rank, s.p_gpu, s.p) == (4, 2, 8)
    assert ClusterShape.parse("4x2").p == 8
    with pytest.raises(ValueError):
        ClusterShape.parse("4")
    with pytest.raises(ValueError):
        ClusterShape(0, 1)
    sh = ClusterShape(3, 2)
    for w in range(sh.p):
        r, g = sh.rank_gpu(w)
        assert r + sh.p_rank * g == w


def test_rmat_params_validation():
    with pytest.raises(ValueError, match="sum"):
        RmatParams(scale=4, a=0.5, b=0.3, c=0.1, d_quad=0.3)
    with pytest.raises(ResourceError):
        RmatParams(scale=30)
    assert RmatParams(scale=26, scale_cap=26).n == 1 << 26
    assert RmatParams(scale=20).num_edges == 16_777_216


def test_bfs_options_validation():
    with pytest.raises(ValueError, match="mode"):
        BfsOptions(mode="dfs")
    o = BfsOptions(mode="bfs", source=5).to_c()
    assert o.mode == 0 and o.source == 5 and o.factor0[3] == 0.5 and o.factor0[1] == 1e-7


def test_teps_and_digest():
    assert compute_teps((1 << 20) * 32, 1.0) == (1 << 20) * 16
    with pytest.raises(ValueError):
        compute_teps(10, 0.0)
    assert levels_digest(np.array([0, 1, -1], dtype=np.int32)) == levels_digest([0, 1, -1])


def test_direction_rule_matches_oracle_and_reference_kats():
    # traversal tests: BV(100, 10, 30) = 400, BV(100, 10, 0) = 100, q=0 -> inf
    assert traversal.estimate_backward_workload(100, 10, 30) == 400
    assert traversal.estimate_backward_workload(100, 10, 0) == 100
    assert math.isinf(traversal.estimate_backward_workload(5, 0, 3))
    ds = traversal.DirectionState("dd", factor0=0.5, factor1=0.0)
    assert traversal.decide_direction(traversal.WorkloadEstimate(fv=1000, u_size=100, q=100, s=0), ds) == "backward"
    rng = np.random.default_rng(1)
    for _ in range(500):
        u, q, s = (int(x) for x in rng.integers(0, 2**30, size=3))
        fv = int(rng.integers(0, 2**33))
        bv = traversal.estimate_backward_workload(u, q, s)
        assert O.bv(u, q, s) == bv
        for d0 in (0, 1):
            ds = traversal.DirectionState("dn", factor0=0.05, factor1=0.3,
                                          direction=("forward", "backward")[d0])
            want = traversal.decide_direction(traversal.WorkloadEstimate(fv=fv, u_size=u, q=q, s=s), ds)
            got = O.decide(d0, fv, O.bv(u, q, s), 0.05, 0.3)
            assert ("forward", "backward")[got] == want


def test_csr_container_invariants():
    with pytest.raises(ValueError, match="close"):
        CsrSubgraph("nn", np.array([0, 1]), np.array([5, 6]))
    with pytest.raises(ValueError, match="non-decreasing"):
        CsrSubgraph("nn", np.array([0, 2, 1]), np.array([5]))
    c = CsrSubgraph("dn", np.array([0, 2, 2, 3]), np.array([4, 5, 6]))
    assert c.degrees().tolist() == [2, 0, 1] and c.neighbors(0).tolist() == [4, 5]


def test_traversal_helpers_equal_reference(reference):
    from delegate_bfs import traversal as rt
    for args in ((100, 10, 30), (7, 3, 2), (0, 1, 0)):
        assert traversal.estimate_backward_workload(*args) == rt.estimate_backward_workload(*args)
    assert traversal.DEFAULT_FACTOR0 == rt.DEFAULT_FACTOR0


def test_device_group_placement_rule(monkeypatch):
    """group_for: ClusterShape(.., P) in one process goes on P GPUs only when P
    are visible, n >= 2^20 and DBFS_DEVICE_GROUP is not 0 (CPU-only check of
    the decision; the groups themselves are tested on GPUs)."""
    from paper_1803_03922_b200 import _lib, group
    made = []
    monkeypatch.setattr(group, "DeviceGroup", lambda devs: made.append(devs) or ("group", tuple(devs)))
    monkeypatch.setattr(group, "_groups", {})
    monkeypatch.setattr(_lib, "device_count", lambda: 4)
    assert group.group_for(1, "auto", 1 << 24) is None
    assert group.group_for(2, None, 1 << 24) is None
    assert group.group_for(8, "auto", 1 << 24) is None          # more workers than GPUs: simulated
    assert group.group_for(4, "auto", 1 << 16) is None          # small graph: one device
    assert group.group_for(4, "auto", 1 << 24) == ("group", (0, 1, 2, 3))
    assert group.group_for(2, [2, 3], 1 << 10) == ("group", (2, 3))  # explicit devices: any size
    with pytest.raises(ValueError):
        group.group_for(2, [0, 1, 2], 1 << 24)
    monkeypatch.setenv("DBFS_DEVICE_GROUP", "0")
    assert group.group_for(4, "auto", 1 << 24) is None
    assert made == [[0, 1, 2, 3], [2, 3]]


def test_digest_sharing_roundtrip(monkeypatch):
    """benchmark() across ranks: rank 0's hex digests survive the int64 round
    trip used to share them over NCCL (sum with zeros)."""
    import numpy as np
    from paper_1803_03922_b200 import engine
    digests = ["ffffffffffffffff", "0000000000000001", "8000000000000000", "03be53e75d9c90ed"]
    vals = np.array([int(d, 16) for d in digests], dtype=np.uint64).view(np.int64)
    back = [f"{int(v):016x}" for v in vals.view(np.uint64)]
    assert back == digests
