"""Edge-list and DPG1 files next to the path.

CPU (no GPU needed): the text parser / writer in libdbfs's host code and the
numpy binary format against the reference's behaviour recorded in
tests/golden/io_golden.json (tests/golden/make_io_golden.py), plus the
reference's own TestIo cases (tests/test_rmat.py:127-179 in the reference).
GPU: DPG1 files written from the device partition are byte-identical to the
reference's; reference-written files load into a device partition whose
arrays and BFS results equal the oracle's.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_1803_03922_b200.rmat import EdgeList, FormatError, load_edge_list, save_edge_list

HERE = os.path.dirname(os.path.abspath(__file__))
IO = json.load(open(os.path.join(HERE, "golden", "io_golden.json")))


def fdigest(path) -> str:
    with open(path, "rb") as f:
        return hashlib.blake2b(f.read(), digest_size=8).hexdigest()


@pytest.mark.parametrize("i", range(len(IO["text"])))
def test_text_parse_matches_reference(tmp_path, i):
    rec = IO["text"][i]
    path = tmp_path / "g.txt"
    with open(path, "w", newline="") as f:
        f.write(rec["text"])
    if "error" in rec:
        with pytest.raises(FormatError) as ei:
            load_edge_list(path, fmt="text")
        assert rec["error"]["type"] == "FormatError"
        assert str(ei.value).replace(str(path), "<path>") == rec["error"]["message"]
    else:
        g = load_edge_list(path, fmt="text")
        assert g.src.tolist() == rec["result"]["src"]
        assert g.dst.tolist() == rec["result"]["dst"]
        assert g.n == rec["result"]["n"]


@pytest.mark.parametrize("entry", IO["edges"], ids=lambda e: f"s{e['scale']}-seed{e['seed']}")
@pytest.mark.parametrize("fmt", ["binary", "text"])
def test_saved_files_byte_identical(tmp_path, entry, fmt):
    src, dst = O.rmat_edges(entry["scale"], seed=entry["seed"])
    g = EdgeList(src, dst, n=1 << entry["scale"], symmetric=True)
    path = tmp_path / f"g.{fmt}"
    save_edge_list(g, path, fmt=fmt)
    assert fdigest(path) == entry[fmt]
    back = load_edge_list(path)
    assert back.n == g.n and np.array_equal(back.src, src) and np.array_equal(back.dst, dst)


def test_auto_detect_truncation_and_headerless(tmp_path):
    path = tmp_path / "g.bin"
    save_edge_list(EdgeList([0], [1], n=2), path, fmt="binary")
    g = load_edge_list(path, fmt="auto")
    assert g.m == 1 and g.n == 2
    data = path.read_bytes()
    path.write_bytes(data[:-3])
    with pytest.raises(FormatError, match="truncated"):
        load_edge_list(path)
    # headerless packed pairs are read as binary when asked; n = 1 + max id
    raw = np.array([[3, 4], [5, 0]], dtype="<u8").tobytes()
    path.write_bytes(raw)
    g = load_edge_list(path, fmt="binary")
    assert g.src.tolist() == [3, 5] and g.dst.tolist() == [4, 0] and g.n == 6
    path.write_bytes(np.array([[1 << 62, 0]], dtype="<u8").tobytes())
    with pytest.raises(FormatError, match="overflow"):
        load_edge_list(path, fmt="binary")


def test_unknown_format_and_missing_file(tmp_path):
    with pytest.raises(ValueError):
        save_edge_list(EdgeList([0], [1], n=2), tmp_path / "x", fmt="csv")
    (tmp_path / "x").write_text("0 1\n")
    with pytest.raises(ValueError):
        load_edge_list(tmp_path / "x", fmt="csv")
    with pytest.raises(OSError):
        load_edge_list(tmp_path / "missing.txt")
    with pytest.raises(OSError):
        save_edge_list(EdgeList([0], [1], n=2), tmp_path / "no" / "dir.txt", fmt="text")


def test_text_writer_negative_and_large_ids(tmp_path):
    g = EdgeList(np.array([0, 5, 2]), np.array([1, 3, 1 << 40]), n=1 << 41)
    path = tmp_path / "g.txt"
    save_edge_list(g, path, fmt="text")
    assert path.read_text() == f"# n {1 << 41}\n0 1\n5 3\n2 {1 << 40}\n"
    back = load_edge_list(path)
    assert back == g


# ---------------------------------------------------------------------------
# DPG1 (GPU: the partition lives on the device)
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def api():
    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200 import _lib
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible for a -m gpu test")
    return api


def _params(api, e):
    a, b, c, dq = e["quads"]
    return api.RmatParams(scale=e["scale"], seed=e["seed"], edge_factor=e["edge_factor"], a=a, b=b, c=c, d_quad=dq)


@pytest.mark.gpu
@pytest.mark.parametrize("entry", IO["dpg"], ids=lambda e: f"s{e['scale']}-t{e['theta']}-{e['p_rank']}x{e['p_gpu']}")
def test_dpg_save_byte_identical_and_round_trip(tmp_path, api, entry):
    from paper_1803_03922_b200.partition import load_partitioned_graph, save_partitioned_graph
    pg = api.partition_graph(api.build_rmat_graph(_params(api, entry)), entry["theta"],
                             api.ClusterShape(entry["p_rank"], entry["p_gpu"]))
    save_partitioned_graph(pg, tmp_path / "pg")
    files = sorted(os.listdir(tmp_path / "pg"))
    assert files == sorted(entry["files"])
    for f in files:
        assert fdigest(tmp_path / "pg" / f) == entry["files"][f], f
    back = load_partitioned_graph(tmp_path / "pg", verify=True)
    assert back.n == pg.n and back.m == pg.m and back.kind_totals == pg.kind_totals
    assert back.classification.d == pg.classification.d
    root = int(np.flatnonzero(pg.classification.out_degree)[0])
    for mode in ("dobfs", "bfs"):
        a = api.run_bfs(pg, api.BfsOptions(mode=mode, source=root))
        b = api.run_bfs(back, api.BfsOptions(mode=mode, source=root))
        assert a.levels_digest == b.levels_digest and a.inspections == b.inspections
        assert a.per_iteration == b.per_iteration


@pytest.mark.gpu
def test_dpg_load_reference_files_matches_oracle(api):
    from paper_1803_03922_b200.partition import load_partitioned_graph
    fx = IO["dpg_fixture"]
    pg = load_partitioned_graph(os.path.join(HERE, "golden", fx["dir"]), verify=True)
    assert pg.shape.p_rank == fx["p_rank"] and pg.shape.p_gpu == fx["p_gpu"]
    assert pg.classification.d == fx["d"] and pg.m == fx["m"]
    src, dst = O.rmat_edges(fx["scale"], seed=fx["seed"])
    og = O.partition(src, dst, 1 << fx["scale"], fx["theta"], fx["p_rank"], fx["p_gpu"])
    for root in (0, 17, 200):
        for mode in ("dobfs", "bfs"):
            run = api.run_bfs(pg, api.BfsOptions(mode=mode, source=root))
            ref = O.run_bfs(og, root, mode=mode)
            assert run.levels_digest == ref["levels_digest"]
            assert run.inspections == ref["inspections"]
        assert api.validate_bfs_tree(pg, root) == 0


@pytest.mark.gpu
def test_dpg_errors(tmp_path, api):
    from paper_1803_03922_b200.partition import load_partitioned_graph
    with pytest.raises(FileNotFoundError):
        load_partitioned_graph(tmp_path)
    (tmp_path / "worker_00000.dpg").write_bytes(b"XXXX" + bytes(64))
    with pytest.raises(ValueError, match="bad magic"):
        load_partitioned_graph(tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1, 1), (2, 1), (2, 2), (4, 2)])
def test_upload_reference_shaped_partition(shape):
    """dbfs_graph_upload_partitioned: a partition built elsewhere (here the
    oracle's restatement of the reference's partition_graph, in the reference's
    PartitionedGraph shape) goes to the device as is; BFS reports equal the
    oracle's, the exported arrays equal the uploaded ones, with and without
    out_degree (DPG1 files carry none)."""
    from types import SimpleNamespace

    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200 import _lib
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible for a -m gpu test")
    scale, seed, theta = 12, 3, 16
    src, dst = O.rmat_edges(scale, seed=seed)
    og = O.partition(src, dst, 1 << scale, theta, *shape)
    for with_degree in (True, False):
        ref = SimpleNamespace(
            shape=api.ClusterShape(*shape), n=og.n, m=og.m,
            classification=SimpleNamespace(theta=theta, out_degree=og.degrees if with_degree else None,
                                           delegate_global_ids=og.delegate_global_ids),
            workers=[SimpleNamespace(index=w.index, subgraph=(lambda k, w=w: getattr(w, k))) for w in og.workers])
        pg = api.upload_partitioned_graph(ref, symmetric=True)
        assert pg.classification.d == og.d and pg.kind_totals == og.kind_totals
        assert np.array_equal(pg.classification.out_degree, og.degrees)
        for w, ow in zip(pg.workers, og.workers):
            for k in ("nn", "nd", "dn", "dd"):
                assert np.array_equal(w.subgraph(k).row_offsets, getattr(ow, k).row_offsets)
                assert np.array_equal(w.subgraph(k).col_indices, getattr(ow, k).col_indices)
            assert np.array_equal(w.nd_source_list, ow.nd_source_list)
        for root in (7, 100, 4000):
            for mode in ("dobfs", "bfs"):
                got = api.run_bfs(pg, api.BfsOptions(mode=mode, source=root)).to_dict()
                want = O.run_bfs(og, root, mode=mode)
                for key in ("levels_digest", "iterations", "per_iteration", "inspections", "comm"):
                    assert got[key] == want[key], (shape, root, mode, key)
        pg.close()
