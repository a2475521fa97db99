"""GPU parity: libdbfs (via the reference-facing API / C-ABI) against the
golden fixtures made from the reference and against the C oracle.

Bar: bit-exact for every integer output -- edge lists, CSR arrays, levels,
iteration counts, per-iteration directions / inspections / FV / BV, comm
accounting.  Parents (no reference) must pass the Graph500 certificate and,
in min-ID mode, equal the oracle's min-ID rule exactly.
"""

import numpy as np
import pytest

import oracle as O
from golden_utils import KINDS, digest, graph_id, iter_partitions, iter_runs, load

pytestmark = pytest.mark.gpu

GOLD = load()


@pytest.fixture(scope="module")
def api():
    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200 import _lib
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible for a -m gpu test")
    return api


def _params(api, g):
    a, b, c, dq = g["quads"]
    return api.RmatParams(scale=g["scale"], seed=g["seed"], edge_factor=g["edge_factor"], a=a, b=b, c=c, d_quad=dq)


_pg_cache = {}


def _pg(api, g, p):
    key = (g["scale"], g["seed"], g["edge_factor"], p["theta"], p["p_rank"], p["p_gpu"])
    if key not in _pg_cache:
        _pg_cache.clear()
        _pg_cache[key] = api.partition_graph(api.build_rmat_graph(_params(api, g)), p["theta"],
                                             api.ClusterShape(p["p_rank"], p["p_gpu"]))
    return _pg_cache[key]


@pytest.mark.parametrize("g", GOLD["graphs"], ids=lambda g: graph_id(g))
def test_gpu_edges_match_golden(api, g):
    el = api.build_rmat_graph(_params(api, g))
    assert el.m == g["m"]
    assert digest(np.concatenate([el.src, el.dst]).astype("<i8")) == g["edge_digest"]


def test_gpu_generate_and_hash_kats(api):
    k = GOLD["kats"]
    gr = api.generate_rmat(api.RmatParams(scale=16))
    assert [[int(gr.src[i]), int(gr.dst[i])] for i in range(3)] == k["s16_generate_first_pairs"]
    from paper_1803_03922_b200.rmat import hash_randomize_vertices, EdgeList
    ids = np.arange(8)
    assert hash_randomize_vertices(EdgeList(ids, ids, n=1 << 16), 0).src.tolist() == k["s16_hash_0_7"]


@pytest.mark.parametrize("gp", list(iter_partitions(GOLD)), ids=lambda gp: graph_id(*gp))
def test_gpu_partition_matches_golden(api, gp):
    g, p = gp
    pg = _pg(api, g, p)
    assert pg.classification.d == p["d"]
    assert pg.kind_totals == p["kind_totals"]
    assert digest(pg.classification.delegate_global_ids.astype("<i8")) == p["delegates_digest"]
    assert api.memory_footprint(pg).to_dict() == p["memory"]
    for w, gw in zip(pg.workers, p["workers"]):
        assert w.n_local == gw["n_local"]
        for k in KINDS:
            csr = w.subgraph(k)
            assert [digest(csr.row_offsets.astype("<i8")), digest(csr.col_indices)] == gw["csr"][k], k
        assert digest(w.nd_source_list.astype("<i8")) == gw["nd_source_list"]
        assert digest(w.dn_source_mask.astype(np.uint8)) == gw["dn_source_mask"]
        assert digest(w.dd_source_mask.astype(np.uint8)) == gw["dd_source_mask"]


_RUNS = list(iter_runs(GOLD))


@pytest.mark.parametrize("policy", ["cost", "push", "reported"])
@pytest.mark.parametrize("gpr", _RUNS, ids=lambda x: graph_id(*x))
def test_gpu_run_bfs_matches_golden(api, gpr, policy):
    """Every reported output equals the reference's, whatever the executor runs:
    'cost' (the default), 'push' (every BACKWARD-reported kind as a counting
    push, counters recovered from twin positions), 'reported' (pulls exactly
    where the reference pulls)."""
    g, p, r = gpr
    pg = _pg(api, g, p)
    run = api.run_bfs(pg, api.BfsOptions(mode=r["mode"], source=r["source"], local_all2all=r["local_all2all"],
                                         uniquify=r["uniquify"], exec_policy=policy))
    want = r["report"]
    got = run.to_dict()
    assert got["levels_digest"] == want["levels_digest"]
    assert got["iterations"] == want["iterations"]
    assert got["inspections"] == want["inspections"]
    assert got["b_measured"] == want["b_measured"]
    assert got["per_iteration"] == want["per_iteration"]
    assert got["comm"] == want["comm"]
    assert api.validate_bfs_tree(pg, r["source"]) == 0


@pytest.mark.parametrize("engine", ["host", "persistent"])
@pytest.mark.parametrize("shape", [(1, 1), (2, 2)])
def test_engines_agree_with_oracle(api, engine, shape):
    scale, seed, theta = 14, 5, 16
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, seed=seed)), theta,
                             api.ClusterShape(*shape))
    src, dst = O.rmat_edges(scale, seed=seed)
    og = O.partition(src, dst, 1 << scale, theta, *shape)
    for root in (1, 4242, 9000):
        for mode in ("bfs", "dobfs"):
            run = api.run_bfs(pg, api.BfsOptions(mode=mode, source=root, engine=engine))
            ref = O.run_bfs(og, root, mode=mode)
            got = run.to_dict()
            for key in ("iterations", "per_iteration", "inspections", "comm", "b_measured", "levels_digest"):
                assert got[key] == ref[key], (engine, shape, mode, root, key)


def test_min_parents_equal_oracle(api):
    scale, seed = 13, 2
    el = api.build_rmat_graph(api.RmatParams(scale=scale, seed=seed))
    src, dst = O.rmat_edges(scale, seed=seed)
    for shape in ((1, 1), (2, 1)):
        pg = api.partition_graph(el, 16, api.ClusterShape(*shape))
        for root in (3, 777):
            lv, par = api.bfs(pg, root, parents="min")
            ref_lv = O.bfs_levels(src, dst, 1 << scale, root)
            assert np.array_equal(lv, ref_lv)
            assert np.array_equal(par, O.min_parents(src, dst, 1 << scale, root, lv))
            lv2, par_any = api.bfs(pg, root, parents="any")
            assert O.validate(src, dst, 1 << scale, root, lv2, par_any) == 0
            assert api.validate_bfs_tree(pg, root, lv2, par_any) == 0
            bad = par_any.copy()
            reached = np.flatnonzero((lv2 > 1))
            bad[reached[0]] = root  # root sits >= 2 levels above
            assert api.validate_bfs_tree(pg, root, lv2, bad) != 0


def test_scale18_dobfs_matches_oracle(api):
    scale, theta = 18, 16
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, scale_cap=30)), theta,
                             api.ClusterShape(1, 1))
    og = O.partition_rmat(scale, theta)
    rng = np.random.default_rng(0)
    for root in rng.integers(0, 1 << scale, size=4):
        for mode in ("dobfs", "bfs"):
            run = api.run_bfs(pg, api.BfsOptions(mode=mode, source=int(root)))
            ref = O.run_bfs(og, int(root), mode=mode)
            assert run.levels_digest == ref["levels_digest"]
            assert run.inspections == ref["inspections"]
            assert run.per_iteration == ref["per_iteration"]


def test_edge_cases(api):
    E = api.EdgeList
    # isolated source (engine.py tests): one iteration, only the source reached
    g = E(np.array([0, 1]), np.array([1, 0]), n=4)
    pg = api.partition_graph(g, 1, api.ClusterShape(2, 1))
    run = api.run_bfs(pg, api.BfsOptions(source=3))
    assert run.levels.tolist() == [-1, -1, -1, 0] and run.iterations == 1
    # out of range source
    with pytest.raises(ValueError, match="out of range"):
        api.run_bfs(pg, api.BfsOptions(source=10 ** 9))
    # empty graph
    pg0 = api.partition_graph(E(np.array([], dtype=np.int64), np.array([], dtype=np.int64), n=8), 4,
                              api.ClusterShape(2, 1))
    r0 = api.run_bfs(pg0, api.BfsOptions(source=5))
    assert r0.levels.tolist() == [-1] * 5 + [0] + [-1] * 2
    for w in pg0.workers:
        for k in KINDS:
            assert w.subgraph(k).num_edges == 0
    # star: centre is the only delegate (partition tests)
    pairs = [(0, i) for i in range(1, 11)]
    s = np.array([u for u, v in pairs] + [v for u, v in pairs])
    d = np.array([v for u, v in pairs] + [u for u, v in pairs])
    pgs = api.partition_graph(E(s, d, n=11), 5, api.ClusterShape(1, 1))
    assert pgs.classification.delegate_global_ids.tolist() == [0]
    assert pgs.kind_totals["nd"] == 10 and pgs.kind_totals["dn"] == 10
    for root in (0, 3):
        for mode in ("bfs", "dobfs"):
            og = O.partition(s, d, 11, 5)
            assert api.run_bfs(pgs, api.BfsOptions(mode=mode, source=root)).to_dict()["per_iteration"] == \
                O.run_bfs(og, root, mode=mode)["per_iteration"]
    # path graph + disconnected vertex, all shapes
    s = np.array([0, 1, 1, 2]); d = np.array([1, 0, 2, 1])
    for shape in ((1, 1), (2, 1), (1, 3)):
        pgp = api.partition_graph(E(s, d, n=4), 1, api.ClusterShape(*shape))
        assert api.run_bfs(pgp, api.BfsOptions(source=0)).levels.tolist() == [0, 1, 2, -1]


def test_errors_map_to_reference_types(api):
    from paper_1803_03922_b200.rmat import ResourceError
    with pytest.raises(ResourceError):
        api.RmatParams(scale=30)
    with pytest.raises(ValueError):
        api.partition_graph(api.EdgeList(np.array([0]), np.array([1]), n=2), -1, api.ClusterShape(1, 1))
    with pytest.raises(ValueError):
        api.BfsOptions(mode="dfs")


def test_benchmark_api(api):
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=10, seed=7)), 16, api.ClusterShape(2, 2))
    rep = api.benchmark(pg, [3, 9], api.BfsOptions())
    assert rep["num_runs"] == 2 and rep["geomean_teps"] > 0 and rep["harmonic_teps"] > 0
    g = api.EdgeList(np.array([0, 1]), np.array([1, 0]), n=8)
    pg2 = api.partition_graph(g, 1, api.ClusterShape(2, 1))
    with pytest.raises(api.EmptyReportError):
        api.benchmark(pg2, [4, 5, 6], api.BfsOptions())


@pytest.mark.parametrize("scale,theta", [(14, 16), (16, 16), (15, 64)])
def test_exec_policy_does_not_change_results(api, scale, theta):
    """Pulling a FORWARD-reported kind (symmetric graphs) must leave every
    reported output identical to executing the reported directions."""
    pg = api.partition_graph(api.build_rmat_graph(api.RmatParams(scale=scale, seed=1)), theta, api.ClusterShape(1, 1))
    rng = np.random.default_rng(scale)
    for root in rng.integers(0, 1 << scale, size=6):
        b = api.run_bfs(pg, api.BfsOptions(source=int(root), exec_policy="reported"))
        db = b.to_dict()
        for policy in ("cost", "push"):
            a = api.run_bfs(pg, api.BfsOptions(source=int(root), exec_policy=policy))
            da = a.to_dict()
            for key in ("iterations", "per_iteration", "inspections", "comm", "levels_digest"):
                assert da[key] == db[key], (policy, key)
            assert api.validate_bfs_tree(pg, int(root), a.levels, a.parents) == 0
