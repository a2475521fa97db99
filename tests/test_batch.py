"""bfs_batch (dbfs_bfs_batch): the multi-root loop with overlapped result copies
returns, for every root, exactly what one bfs() call returns (depths equal the
oracle's; the parent tree passes the Graph500 certificate)."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200 import _lib
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible for a -m gpu test")
    return api


@pytest.mark.parametrize("compact", [True, False])
@pytest.mark.parametrize("shape", [(1, 1), (2, 2)])
def test_batch_matches_single_calls_and_oracle(api, shape, compact):
    from paper_1803_03922_b200 import _lib
    scale, seed, theta = 12, 3, 16
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, seed=seed)), theta,
                             api.ClusterShape(*shape))
    src, dst = O.rmat_edges(scale, seed=seed)
    og = O.partition(src, dst, 1 << scale, theta, *shape)
    roots = [7, 100, 7, 4000, 17, 2]
    outs, st = api.bfs_batch(pg, roots, stats=True, compact=compact)
    assert len(outs) == len(roots) and len(st) == len(roots)
    for r, (lv, pa), s in zip(roots, outs, st):
        ref = O.run_bfs(og, r, mode="dobfs")
        assert api.levels_digest(lv) == ref["levels_digest"]
        assert s.iterations == ref["iterations"]
        assert api.validate_bfs_tree(pg, r, lv, pa) == 0
        lv1, _ = api.bfs(pg, r)
        assert np.array_equal(lv, lv1)
    # two pinned pairs used alternately: the last two roots' results survive
    pairs = [(_lib.pinned_empty(pg.n, np.int32), _lib.pinned_empty(pg.n, np.int64)) for _ in range(2)]
    outs = [(pairs[i % 2][0].array, pairs[i % 2][1].array) for i in range(len(roots))]
    api.bfs_batch(pg, roots, outs=outs, mode="bfs", compact=compact)
    for i in (len(roots) - 2, len(roots) - 1):
        lv, pa = outs[i]
        assert api.levels_digest(lv) == O.run_bfs(og, roots[i], mode="bfs")["levels_digest"]
        assert api.validate_bfs_tree(pg, roots[i], lv, pa) == 0


def test_batch_errors(api):
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=8, seed=1)), 16, api.ClusterShape(1, 1))
    with pytest.raises(ValueError):
        api.bfs_batch(pg, [0, 1 << 8])
    with pytest.raises(ValueError):
        api.bfs_batch(pg, [0], outs=[(np.empty(3, np.int32), None)])
    assert api.bfs_batch(pg, []) == []
    lv = api.bfs_batch(pg, [5], parents=None)[0][0]
    assert lv[5] == 0


def test_compact_batch_escapes_deep_levels(api):
    """Depths >= 127 do not fit the int8 wire form: such roots are re-run with
    full arrays, results identical to single calls (a 400-vertex path)."""
    n = 400
    src = np.arange(n - 1, dtype=np.int64)
    g = api.EdgeList(np.concatenate([src, src + 1]), np.concatenate([src + 1, src]), n=n, symmetric=True)
    pg = api.partition_graph(g, 1, api.ClusterShape(1, 1))
    roots = [0, 200, 5, 399]
    outs = api.bfs_batch(pg, roots, compact=True)
    for r, (lv, pa) in zip(roots, outs):
        assert lv.tolist() == [abs(v - r) for v in range(n)]
        assert api.validate_bfs_tree(pg, r, lv, pa) == 0
        ref_lv, _ = api.bfs(pg, r)
        assert np.array_equal(lv, ref_lv)


def test_compact_rerun_leaves_device_state_consistent(api):
    """An early root escapes (depth >= 127) and is re-run after the batch while
    the last root does not: the device result, last source and iteration count
    must then describe the re-run root (validate / min_parents without arrays
    use them)."""
    n = 400
    src = np.arange(n - 1, dtype=np.int64)
    # path of 400 plus a shallow last root: centre of a short component glued on
    n2 = n + 5
    s2 = np.concatenate([src, np.array([n, n, n, n])])
    d2 = np.concatenate([src + 1, np.array([n + 1, n + 2, n + 3, n + 4])])
    g2 = api.EdgeList(np.concatenate([s2, d2]), np.concatenate([d2, s2]), n=n2, symmetric=True)
    pg2 = api.partition_graph(g2, 2, api.ClusterShape(1, 1))
    outs = api.bfs_batch(pg2, [0, n], compact=True, parents="any")
    assert outs[0][0][n - 1] == n - 1 and outs[1][0][n] == 0
    # the device now holds root 0's result (re-run last): certificate on device arrays
    assert api.validate_bfs_tree(pg2, 0) == 0
    par = api.min_parents(pg2)
    assert par[0] == 0 and par[1] == 0 and par[n - 1] == n - 2
    # min-ID parents requested in a batch are computed on device per root
    outs = api.bfs_batch(pg2, [n, 2], parents="min", compact=False)
    lv, pa = outs[1]
    assert pa[2] == 2 and pa[1] == 2 and pa[3] == 2 and pa[0] == 1 and pa[n] == -1


@pytest.mark.parametrize("split", ["0", "0.4", "1"])
def test_compact_split_into_pinned_outputs(api, split, monkeypatch):
    """The compact transfer into page-locked caller arrays: the first
    DBFS_COMPACT_SPLIT of the depths travel as int32 straight into the caller's
    array, the rest as int8 widened on the host (AVX2 streaming stores into an
    arbitrarily aligned destination) -- every split gives the oracle's depths."""
    from paper_1803_03922_b200 import _lib
    monkeypatch.setenv("DBFS_COMPACT_SPLIT", split)
    scale, seed, theta = 13, 5, 16
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, seed=seed)), theta,
                             api.ClusterShape(1, 1))
    src, dst = O.rmat_edges(scale, seed=seed)
    og = O.partition(src, dst, 1 << scale, theta, 1, 1)
    roots = [3, 4000, 77, 1234, 9]
    n = pg.n
    # one page-locked block, views at 4-byte offsets: destinations not 32-byte aligned
    held = _lib.pinned_empty(len(roots) * (n + 3) + 8, np.int32)
    outs = [(held.array[1 + i * (n + 3): 1 + i * (n + 3) + n], None) for i in range(len(roots))]
    api.bfs_batch(pg, roots, outs=outs, parents=None, compact=True)
    for r, (lv, _) in zip(roots, outs):
        assert api.levels_digest(lv) == O.run_bfs(og, r, mode="dobfs")["levels_digest"], (split, r)
    # benchmark() (its own pinned level arrays) reports the same digests
    rep = api.benchmark(pg, roots, api.BfsOptions(mode="dobfs"))
    for run in rep["runs"]:
        assert run["levels_digest"] == O.run_bfs(og, run["source"], mode="dobfs")["levels_digest"]
