"""CPU: live cross-check of the C oracle against the reference package.

Skipped where /root/reference is absent (the GPU box); there the golden
fixtures in tests/golden/ stand in for it.
"""

import numpy as np
import pytest

import oracle as O


@pytest.mark.parametrize("shape", [(1, 1), (2, 2), (4, 2), (1, 4)])
def test_oracle_equals_reference_grid(reference, shape):
    from delegate_bfs import engine, partition, rmat
    from delegate_bfs.engine import BfsOptions
    from delegate_bfs.partition import ClusterShape

    g = rmat.build_rmat_graph(rmat.RmatParams(scale=11, seed=4))
    src, dst = O.rmat_edges(11, seed=4)
    assert np.array_equal(src, g.src) and np.array_equal(dst, g.dst)
    for theta in (3, 16, 64):
        pg = partition.partition_graph(g, theta, ClusterShape(*shape))
        og = O.partition(src, dst, g.n, theta, *shape)
        for w in range(og.p):
            for k in O.KINDS:
                a, b = getattr(pg.workers[w], k), getattr(og.workers[w], k)
                assert np.array_equal(a.row_offsets, b.row_offsets)
                assert np.array_equal(a.col_indices, b.col_indices)
        for mode in ("bfs", "dobfs"):
            for la, uq in ((False, False), (True, False), (False, True), (True, True)):
                for s in (0, 5, 333, 2047):
                    r = engine.run_bfs(pg, BfsOptions(mode=mode, source=s, local_all2all=la,
                                                      uniquify=uq)).to_dict()
                    o = O.run_bfs(og, s, mode=mode, local_all2all=la, uniquify=uq)
                    for key in ("iterations", "per_iteration", "inspections", "comm",
                                "b_measured", "levels_digest"):
                        assert r[key] == o[key], (theta, mode, la, uq, s, key)


def test_oracle_levels_equal_reference_oracle(reference):
    from delegate_bfs import oracle as ref_oracle, rmat

    g = rmat.build_rmat_graph(rmat.RmatParams(scale=12, seed=8))
    for s in (0, 99, 4000):
        assert np.array_equal(O.bfs_levels(g.src, g.dst, g.n, s), ref_oracle.bfs_levels(g, s))


def test_uniform_quadrants_equal_reference(reference):
    from delegate_bfs import rmat

    p = rmat.RmatParams(scale=10, seed=2, a=0.25, b=0.25, c=0.25, d_quad=0.25, edge_factor=4)
    g = rmat.build_rmat_graph(p)
    src, dst = O.rmat_edges(10, 4, 0.25, 0.25, 0.25, 2)
    assert np.array_equal(src, g.src) and np.array_equal(dst, g.dst)
