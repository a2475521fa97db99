"""delegate-bfs command line, after the reference's
tests/test_cli.py: threshold curve, config handling and argument errors on
the CPU; every subcommand end to end on the GPU."""

import csv
import json

import numpy as np
import pytest

import oracle as O
from paper_1803_03922_b200 import rmat
from paper_1803_03922_b200.cli import main, resolve_theta, suggested_theta


def test_theta_curve():
    assert suggested_theta(30) == 64 and suggested_theta(32) == 128 and suggested_theta(40) == 512
    assert all(suggested_theta(s) == 16 for s in range(10, 17))
    assert resolve_theta(64, n=1 << 12) == 64 and resolve_theta("auto", n=1 << 12) == 16


def test_theta_curve_matches_reference(reference):
    from delegate_bfs import cli as R
    for s in range(0, 48):
        assert suggested_theta(s) == R.suggested_theta(s), s
    for n in (1, 2, 3, 1000, 1 << 20, (1 << 27) + 1):
        assert resolve_theta("auto", n) == R.resolve_theta("auto", n)


def test_cost_csv(tmp_path):
    out = tmp_path / "cost.csv"
    assert main(["cost", "--n", str(1 << 20), "--m", str((1 << 20) * 32), "--p", "16", "--d", "4096",
                 "--p-sweep", "16,64,256", "--out", str(out)]) == 0
    rows = list(csv.DictReader(open(out)))
    assert [int(r["p"]) for r in rows] == [16, 64, 256]
    assert all(float(r["time_delegate"]) > 0 for r in rows)


def test_cost_csv_matches_reference(tmp_path, reference):
    from delegate_bfs import cli as R
    argv = ["cost", "--n", "262144", "--m", "8388608", "--p", "4", "--p-gpu", "2", "--d", "777", "--e-nn", "99",
            "--p-sweep", "4,16,64", "--strong-scaling"]
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    assert main(argv + ["--out", str(a)]) == 0
    assert R.main(argv + ["--out", str(b)]) == 0
    assert a.read_text() == b.read_text()


def test_config_and_argument_errors(tmp_path, monkeypatch, capsys):
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"scale": 10, "bogus": 1}))
    assert main(["run", "--config", str(cfg)]) == 1
    with pytest.raises(SystemExit):
        main(["run", "--source", "0"])
    assert main(["generate", "--scale", "31", "--out", str(tmp_path / "x.bin")]) == 1
    assert "error" in capsys.readouterr().err
    monkeypatch.setenv("DELEGATE_BFS_THREADS", "zero")
    assert main(["verify", "--scale", "8", "--sources", "1"]) == 2
    assert "DELEGATE_BFS_THREADS" in capsys.readouterr().err


@pytest.fixture(scope="module")
def gpu():
    from paper_1803_03922_b200 import _lib
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible for a -m gpu test")


@pytest.mark.gpu
def test_generate_partition_memory(tmp_path, gpu, capsys):
    out = tmp_path / "g.bin"
    assert main(["generate", "--scale", "8", "--seed", "4", "--out", str(out)]) == 0
    g = rmat.load_edge_list(out)
    src, dst = O.rmat_edges(8, seed=4)
    assert g.m == 2 * 256 * 16 and np.array_equal(g.src, src) and np.array_equal(g.dst, dst)
    assert "wrote" in capsys.readouterr().out
    txt = tmp_path / "g.txt"
    assert main(["generate", "--scale", "8", "--seed", "4", "--format", "text", "--out", str(txt)]) == 0
    assert rmat.load_edge_list(txt) == g
    capsys.readouterr()
    assert main(["partition", "--scale", "10", "--shape", "1x2x2", "--theta", "auto"]) == 0
    summary = json.loads(capsys.readouterr().out)
    assert summary["theta"] == 16 and summary["n"] == 1024 and sum(summary["kind_totals"].values()) == summary["m"]
    assert main(["partition", "--scale", "8", "--shape", "2x1x1", "--out", str(tmp_path / "pg")]) == 0
    assert len(list((tmp_path / "pg").glob("*.dpg"))) == 2
    mem = tmp_path / "mem.json"
    assert main(["memory", "--scale", "10", "--shape", "1x2x2", "--out", str(mem)]) == 0
    rep = json.loads(mem.read_text())
    assert rep["total_bytes"] == sum(rep["offsets_bytes"].values()) + sum(rep["indices_bytes"].values())


@pytest.mark.gpu
def test_run_reports_match_oracle(tmp_path, gpu):
    out = tmp_path / "run.json"
    assert main(["run", "--scale", "10", "--shape", "2x2x2", "--mode", "dobfs", "--source", "3",
                 "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    src, dst = O.rmat_edges(10)
    ref = O.run_bfs(O.partition(src, dst, 1 << 10, 16, 4, 2), 3, mode="dobfs")
    assert rep["levels_digest"] == ref["levels_digest"] and rep["inspections"] == ref["inspections"]
    assert rep["params"]["mode"] == "dobfs"
    bench = tmp_path / "bench.json"
    assert main(["run", "--scale", "10", "--sources", "5", "--out", str(bench)]) == 0
    rep = json.loads(bench.read_text())
    assert rep["num_runs"] >= 1 and rep["geomean_teps"] > 0
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"scale": 10, "shape": "1x2x2", "source": 3, "mode": "bfs",
                               "out": str(tmp_path / "r.json")}))
    assert main(["run", "--scale", "12", "--config", str(cfg)]) == 0
    rep = json.loads((tmp_path / "r.json").read_text())
    assert rep["params"]["scale"] == 10 and rep["params"]["mode"] == "bfs"


@pytest.mark.gpu
def test_run_from_edge_file(tmp_path, gpu):
    """--graph: a text edge list (not symmetric) is loaded, symmetrized and run."""
    path = tmp_path / "g.txt"
    path.write_text("# n 6\n0 1\n1 2\n2 3\n0 4\n")
    out = tmp_path / "r.json"
    assert main(["run", "--graph", str(path), "--theta", "1", "--source", "0", "--mode", "bfs",
                 "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["iterations"] == 4


@pytest.mark.gpu
def test_verify_and_sweep(tmp_path, gpu, capsys):
    assert main(["verify", "--scale", "10", "--shape", "1x2x2", "--sources", "5"]) == 0
    assert "0 mismatches" in capsys.readouterr().out
    out = tmp_path / "sweep.csv"
    assert main(["sweep-theta", "--scale", "10", "--seed", "7", "--thetas", "16,32,64", "--sources", "2",
                 "--out", str(out)]) == 0
    rows = {int(r["theta"]): r for r in csv.DictReader(open(out))}
    src, dst = O.rmat_edges(10, seed=7)
    deg = np.bincount(src, minlength=1 << 10)
    for theta in (16, 32, 64):
        assert int(rows[theta]["d"]) == int((deg > theta).sum())
        normal = deg <= theta
        assert int(rows[theta]["e_nn"]) == int((normal[src] & normal[dst]).sum())
