"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``delegate_bfs`` from
/root/reference/pkg/src and records, for a grid of small configurations,
digests of its outputs: RMAT edge lists (rmat.py:125-208), partitioned CSRs
(partition.py:343-351), memory footprints (storage.py:89-117) and full
``run_bfs`` reports (engine.py:98-330, ``BfsRun.to_dict`` minus timing).
The resulting ``golden.json`` travels with the repo (the reference does not),
so the GPU box can check both the oracle and the CUDA path against it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def digest(arr) -> str:
    a = np.ascontiguousarray(arr)
    return hashlib.blake2b(a.tobytes(), digest_size=8).hexdigest()


def run_record(run) -> dict:
    d = run.to_dict()
    d.pop("elapsed")
    d.pop("teps")
    d.pop("m_prime")
    return d


def c1_roots(g) -> list:
    """BASELINE configs[0] roots on the scale-16 graph: the 64 Graph500 roots
    (first 64 distinct vertices with out-degree > 0 drawn from
    default_rng(0).integers(0, n); the same rule as bench.py's
    graph500_roots) followed by the reference CLI's own 64 draws
    (cli.py:151-152, with replacement, degree 0 allowed) not already listed."""
    deg = np.bincount(g.src, minlength=g.n)
    rng = np.random.default_rng(0)
    roots, seen = [], set()
    while len(roots) < 64:
        for v in rng.integers(0, g.n, size=4096).tolist():
            if v not in seen and deg[v] > 0:
                seen.add(v)
                roots.append(v)
                if len(roots) == 64:
                    break
    for v in np.random.default_rng(0).integers(0, g.n, size=64).tolist():
        if v not in seen:
            seen.add(v)
            roots.append(v)
    return [int(v) for v in roots]


def main():
    sys.path.insert(0, REF)
    from delegate_bfs import rmat, storage
    from delegate_bfs.cli import resolve_theta
    from delegate_bfs.engine import BfsOptions, run_bfs
    from delegate_bfs.partition import ClusterShape, partition_graph

    out = {"source": "reference delegate_bfs @ /root/reference/pkg/src", "graphs": [], "kats": {}}

    # --- known-answer values
    g16 = rmat.generate_rmat(rmat.RmatParams(scale=16, seed=0))
    out["kats"]["s16_generate_first_pairs"] = [[int(g16.src[i]), int(g16.dst[i])] for i in range(3)]
    ids = np.arange(8, dtype=np.int64)
    h = rmat.hash_randomize_vertices(rmat.EdgeList(ids, ids, n=1 << 16), seed=0)
    out["kats"]["s16_hash_0_7"] = h.src.tolist()
    for k, seed in ((1, 5), (4, 123456789), (10, 11), (20, 2**63 - 1)):
        n = 1 << k
        ids = np.arange(min(n, 64), dtype=np.int64)
        hh = rmat.hash_randomize_vertices(rmat.EdgeList(ids, ids, n=n), seed=seed)
        out["kats"][f"hash_k{k}_seed{seed}"] = hh.src.tolist()

    configs = [
        # (scale, seed, edge_factor, quads, thetas, shapes, sources)
        (8, 5, 16, None, [3, 16], ["1x1", "2x1", "1x4"], [0, 1, 77]),
        (10, 7, 16, None, [16, 64], ["1x1", "2x2", "4x2"], [0, 3, 9, 512]),
        (12, 3, 16, None, [16, "auto", 256], ["1x1", "2x2", "1x4"], [7, 11, 17, 100]),
        (12, 21, 16, None, ["auto"], ["4x2"], [17]),
        (12, 0, 16, None, [16], ["2x2"], [3, 100, 999]),
        (11, 9, 8, (0.25, 0.25, 0.25, 0.25), [64, 16], ["1x1", "1x2"], [5, 1000]),
        (16, 0, 16, None, [16], ["1x1"], "C1"),
        (14, 0, 16, None, ["auto"], ["2x2"], [5, 77]),
    ]
    for scale, seed, ef, quads, thetas, shapes, sources in configs:
        kw = {}
        if quads:
            kw = dict(a=quads[0], b=quads[1], c=quads[2], d_quad=quads[3])
        params = rmat.RmatParams(scale=scale, seed=seed, edge_factor=ef, **kw)
        g = rmat.build_rmat_graph(params)
        if sources == "C1":
            sources = c1_roots(g)
            out["kats"]["c1_roots"] = sources
        gentry = {
            "scale": scale, "seed": seed, "edge_factor": ef,
            "quads": list(quads) if quads else [0.57, 0.19, 0.19, 0.05],
            "n": g.n, "m": g.m,
            "edge_digest": digest(np.concatenate([g.src, g.dst]).astype("<i8")),
            "first_pairs": [[int(g.src[i]), int(g.dst[i])] for i in range(2)],
            "partitions": [],
        }
        for theta_spec in thetas:
            theta = resolve_theta(theta_spec, g.n)
            for shape_s in shapes:
                pr, pgpu = (int(x) for x in shape_s.split("x"))
                pg = partition_graph(g, theta, ClusterShape(pr, pgpu))
                rep = storage.memory_footprint(pg)
                pentry = {
                    "theta": theta, "p_rank": pr, "p_gpu": pgpu,
                    "d": pg.classification.d,
                    "delegates_digest": digest(pg.classification.delegate_global_ids.astype("<i8")),
                    "kind_totals": pg.kind_totals,
                    "memory": rep.to_dict(),
                    "workers": [],
                    "runs": [],
                }
                for w in pg.workers:
                    pentry["workers"].append({
                        "n_local": w.n_local,
                        "csr": {k: [digest(w.subgraph(k).row_offsets.astype("<i8")),
                                    digest(w.subgraph(k).col_indices)]
                                for k in ("nn", "nd", "dn", "dd")},
                        "nd_source_list": digest(w.nd_source_list.astype("<i8")),
                        "dn_source_mask": digest(w.dn_source_mask.astype(np.uint8)),
                        "dd_source_mask": digest(w.dd_source_mask.astype(np.uint8)),
                    })
                for src in sources:
                    if src >= g.n:
                        continue
                    for mode in ("bfs", "dobfs"):
                        opts_list = [(False, False)]
                        if pr * pgpu > 1:
                            opts_list.append((True, True))
                        for la, uq in opts_list:
                            run = run_bfs(pg, BfsOptions(mode=mode, source=int(src),
                                                         local_all2all=la, uniquify=uq))
                            pentry["runs"].append({
                                "source": int(src), "mode": mode,
                                "local_all2all": la, "uniquify": uq,
                                "report": run_record(run),
                            })
                gentry["partitions"].append(pentry)
        out["graphs"].append(gentry)
        print(f"scale {scale} seed {seed}: {len(gentry['partitions'])} partitions", flush=True)

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
