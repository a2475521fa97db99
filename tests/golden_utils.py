"""Helpers to iterate the golden fixtures made by tests/golden/make_golden.py."""

import hashlib
import json
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")
KINDS = ("nn", "nd", "dn", "dd")


def load():
    with open(PATH) as f:
        return json.load(f)


def digest(arr) -> str:
    a = np.ascontiguousarray(arr)
    return hashlib.blake2b(a.tobytes(), digest_size=8).hexdigest()


def iter_partitions(golden, max_scale=99):
    for g in golden["graphs"]:
        if g["scale"] > max_scale:
            continue
        for p in g["partitions"]:
            yield g, p


def iter_runs(golden, max_scale=99):
    for g, p in iter_partitions(golden, max_scale):
        for r in p["runs"]:
            yield g, p, r


def graph_id(g, p=None, r=None):
    s = f"s{g['scale']}-seed{g['seed']}-ef{g['edge_factor']}"
    if p is not None:
        s += f"-t{p['theta']}-{p['p_rank']}x{p['p_gpu']}"
    if r is not None:
        s += f"-src{r['source']}-{r['mode']}" + ("-LU" if r["local_all2all"] else "")
    return s


def run_matches(report: dict, got: dict, keys=("iterations", "per_iteration", "inspections",
                                               "total_inspections", "comm", "b_measured",
                                               "levels_digest")):
    """Return the list of keys where ``got`` differs from the golden ``report``."""
    bad = []
    for k in keys:
        if report[k] != got[k]:
            bad.append(k)
    return bad
