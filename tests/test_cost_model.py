"""Cost model: the reference's formulas (cost_model.py:1-118,
tests/test_cost_model.py in the reference) and the delegate model's volume
bound against the reference's own byte accounting of every golden run."""

import itertools
import math
from types import SimpleNamespace

import pytest

from golden_utils import iter_partitions, load
from paper_1803_03922_b200 import cost_model as C


def params(**kw):
    base = dict(n=1 << 20, m=(1 << 20) * 32, p=16, p_rank=16, p_gpu=1, g=1e-9, S=6, S_b=3, d=0, E_nn=0)
    base.update(kw)
    return C.CostModelParams(**base)


def test_validation():
    with pytest.raises(ValueError, match="p_rank"):
        params(p=16, p_rank=4, p_gpu=2)
    with pytest.raises(ValueError):
        params(S_b=-1)
    assert params().n_t == 1 << 20


def test_known_values():
    vol, t = C.cost_1d(params(m=1 << 25, p=4, p_rank=4))
    assert vol == float(1 << 28) and t == pytest.approx((1 << 26) * 1e-9)
    assert C.cost_2d(params(p=1, p_rank=1)) == (0.0, 0.0, 0.0)
    with pytest.raises(ValueError, match="square"):
        C.cost_2d(params(p=8, p_rank=8))
    fwd, bwd, t = C.cost_2d(params())
    assert fwd == pytest.approx(8 * (1 << 20) * 4 * 2)
    assert bwd == pytest.approx(2 * (1 << 20) * 3 * 4 * 2 / 8)
    assert t == pytest.approx((4 * (1 << 20) + (1 << 20) * 3 / 8) * (2 / 4) * 1e-9)
    _, t = C.cost_delegate(params(p=4, p_rank=1, p_gpu=4, d=100, E_nn=1 << 16))
    assert t == pytest.approx(4 * (1 << 16) / 4 * 1e-9)
    vol, _ = C.cost_delegate(params(d=4096, E_nn=10))
    assert vol == 4096 * 16 / 4 * 6 + 40
    assert C.cost_delegate_weak_scaling(params(p=16, p_rank=16)) == pytest.approx((1 << 20) * 4 / 16 * 6 * 1e-9)


def test_sweep_rows():
    rows = C.sweep_p(params(d=4096), [16, 32, 64], p_gpu=1)
    assert [r["p"] for r in rows] == [16, 32, 64]
    assert "time_2d" in rows[0] and "time_2d" not in rows[1]
    with pytest.raises(ValueError):
        C.sweep_p(params(), [6], p_gpu=4)


def test_matches_reference_module(reference):
    from delegate_bfs import cost_model as R
    grid = itertools.product([1, 4, 16, 64], [1, 2, 4], [0, 4096], [0, 1 << 16], [True, False])
    for p, p_gpu, d, e_nn, weak in grid:
        if p % p_gpu:
            continue
        kw = dict(n=1 << 18, m=1 << 23, p=p, p_rank=p // p_gpu, p_gpu=p_gpu, g=2e-9, S=7, S_b=2, d=d, E_nn=e_nn)
        a, b = C.CostModelParams(**kw), R.CostModelParams(**kw)
        assert C.cost_1d(a) == R.cost_1d(b)
        assert C.cost_delegate(a) == pytest.approx(R.cost_delegate(b), rel=1e-15)
        assert C.cost_delegate_weak_scaling(a) == pytest.approx(R.cost_delegate_weak_scaling(b), rel=1e-15)
        if math.isqrt(p) ** 2 == p:
            assert C.cost_2d(a) == pytest.approx(R.cost_2d(b), rel=1e-15)
        ra = C.sweep_p(a, [p, 4 * p], p_gpu=p_gpu, weak_scaling=weak)
        rb = R.sweep_p(b, [p, 4 * p], p_gpu=p_gpu, weak_scaling=weak)
        assert [list(x) for x in ra] == [list(x) for x in rb]
        for x, y in zip(ra, rb):
            for k in x:
                assert x[k] == pytest.approx(y[k], rel=1e-15)


def test_delegate_bound_holds_for_every_golden_run():
    """The reference's accounting of each golden run (mask bytes d*p_rank/4 per
    dirty iteration + 4 B per normal record) never exceeds the model's bound."""
    checked = 0
    for g, p in iter_partitions(load()):
        shape = SimpleNamespace(p=p["p_rank"] * p["p_gpu"], p_rank=p["p_rank"], p_gpu=p["p_gpu"])
        pg = SimpleNamespace(n=g["n"], m=g["m"], shape=shape, classification=SimpleNamespace(d=p["d"]),
                             kind_totals=p["kind_totals"])
        for r in p["runs"]:
            c = r["report"]["comm"]
            comm = SimpleNamespace(total_mask_bytes=c["total_mask_bytes"], total_normal_bytes=c["total_normal_bytes"],
                                   s_prime=c["s_prime"], wire_bytes=0)
            run = SimpleNamespace(iterations=r["report"]["iterations"], comm_stats=comm)
            out = C.delegate_comm_check(pg, run)
            assert out["within_bound"], (g["scale"], p["theta"], r["source"], out)
            assert out["accounted_mask"] == c["s_prime"] * p["d"] * p["p_rank"] / 4
            checked += 1
    assert checked > 300
