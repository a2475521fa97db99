"""Scrambled RMAT labeling (this build's option, rmat.RmatParams.scramble):
a Feistel relabeling applied after the reference hash.  The graph is an
isomorphic relabeling of the reference graph; worker loads balance."""

import numpy as np
import pytest

import oracle as O

KINDS = ("nn", "nd", "dn", "dd")


def _loads(og):
    return np.array([sum(len(getattr(w, k).col_indices) for k in KINDS) for w in og.workers], dtype=np.float64)


def test_scramble_is_a_relabeling():
    s0, d0 = O.rmat_edges(14)
    s1, d1 = O.rmat_edges(14, scramble=True)
    n = 1 << 14
    # same degree multiset and the same number of non-isolated vertices
    assert np.array_equal(np.sort(np.bincount(s0, minlength=n)), np.sort(np.bincount(s1, minlength=n)))
    # the relabeling is a function: build the map from edge order and check it is a bijection
    m = np.full(n, -1, dtype=np.int64)
    m[s0] = s1
    m[d0] = d1
    used = m[m >= 0]
    assert len(np.unique(used)) == len(used)
    assert np.array_equal(m[s0], s1) and np.array_equal(m[d0], d1)


def test_scramble_balances_workers():
    ref = _loads(O.partition_rmat(16, 16, 1, 4))
    scr = _loads(O.partition_rmat(16, 16, 1, 4, scramble=True))
    assert ref.max() / ref.mean() > 1.5       # the reference hash: skewed owners
    assert scr.max() / scr.mean() < 1.1


def test_scramble_bfs_is_isomorphic():
    s0, d0 = O.rmat_edges(13)
    s1, d1 = O.rmat_edges(13, scramble=True)
    n = 1 << 13
    m = np.full(n, -1, dtype=np.int64)
    m[s0] = s1
    m[d0] = d1
    root = int(s0[5])
    l0 = O.bfs_levels(s0, d0, n, root)
    l1 = O.bfs_levels(s1, d1, n, int(m[root]))
    mapped = np.flatnonzero(m >= 0)
    assert np.array_equal(l0[mapped], l1[m[mapped]])


@pytest.mark.gpu
def test_gpu_scrambled_graph_matches_oracle():
    import paper_1803_03922_b200 as api
    from golden_utils import digest
    prm = api.RmatParams(scale=15, seed=3, scramble=True)
    el = api.build_rmat_graph(prm)
    src, dst = O.rmat_edges(15, seed=3, scramble=True)
    assert digest(np.concatenate([el.src, el.dst]).astype("<i8")) == digest(np.concatenate([src, dst]).astype("<i8"))
    pg = api.partition_graph(api.build_rmat_graph(prm), 16, api.ClusterShape(1, 4))
    og = O.partition_rmat(15, 16, 1, 4, seed=3, scramble=True)
    for root in (1, 999, 20000):
        for mode in ("dobfs", "bfs"):
            got = api.run_bfs(pg, api.BfsOptions(mode=mode, source=root)).to_dict()
            ref = O.run_bfs(og, root, mode=mode)
            for key in ("levels_digest", "iterations", "inspections", "per_iteration", "comm"):
                assert got[key] == ref[key], (mode, root, key)
