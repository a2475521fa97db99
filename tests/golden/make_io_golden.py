"""Golden fixtures for the file formats next to the path,
generated from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_io_golden.py

Records into ``io_golden.json``:
  * DPG1 (partition.py:392-421): blake2b-8 of every worker file the reference's
    ``save_partitioned_graph`` writes, for a grid of small partitions;
  * DEL1 binary and text edge lists (rmat.py:211-229): blake2b-8 of the files
    ``save_edge_list`` writes for small RMAT graphs;
  * ``load_edge_list`` (rmat.py:232-286) on hand-written text snippets: the
    parsed (src, dst, n) or the exception type and message;
and writes one reference-made DPG1 partition (scale 8, theta 8, shape 2x1) to
``dpg_s8_t8_2x1/`` so the GPU box can load files it did not write.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (scale, seed, edge_factor, quads, theta, shape)
DPG_CONFIGS = [
    (8, 5, 16, None, 3, "1x1"),
    (10, 7, 16, None, 16, "2x2"),
    (10, 7, 16, None, 64, "4x2"),
    (12, 3, 16, None, 16, "1x4"),
    (11, 9, 8, (0.25, 0.25, 0.25, 0.25), 16, "1x2"),
]
EDGE_CONFIGS = [(8, 4), (10, 7)]  # (scale, seed), build_rmat_graph defaults
TEXT_SNIPPETS = [
    "0 1\n1 0\n",
    "",
    "# n 10\n0 1\n",
    "0 1\n0 1 2\n",
    "# n 2\n0 5\n",
    "# comment\n\n  3\t4  \r\n5 6\r7 8\n# n 12\n",
    "+1 2\n1_0 3\n",
    "0 x\n",
    "# n 4 extra\n0 3\n",
    "#n 9\n1 2",
    "-1 2\n",
    "1\n",
]


def fdigest(path) -> str:
    with open(path, "rb") as f:
        return hashlib.blake2b(f.read(), digest_size=8).hexdigest()


def main():
    sys.path.insert(0, REF)
    from delegate_bfs import rmat
    from delegate_bfs.partition import ClusterShape, partition_graph, save_partitioned_graph

    out = {"source": "reference delegate_bfs @ /root/reference/pkg/src", "dpg": [], "edges": [], "text": []}
    tmp = tempfile.mkdtemp()
    try:
        for scale, seed, ef, quads, theta, shape in DPG_CONFIGS:
            kw = dict(a=quads[0], b=quads[1], c=quads[2], d_quad=quads[3]) if quads else {}
            g = rmat.build_rmat_graph(rmat.RmatParams(scale=scale, seed=seed, edge_factor=ef, **kw))
            pr, pgpu = (int(x) for x in shape.split("x"))
            pg = partition_graph(g, theta, ClusterShape(pr, pgpu))
            d = os.path.join(tmp, f"dpg_{scale}_{seed}_{theta}_{shape}")
            save_partitioned_graph(pg, d)
            files = sorted(os.listdir(d))
            out["dpg"].append({"scale": scale, "seed": seed, "edge_factor": ef,
                               "quads": list(quads) if quads else [0.57, 0.19, 0.19, 0.05],
                               "theta": theta, "p_rank": pr, "p_gpu": pgpu,
                               "files": {f: fdigest(os.path.join(d, f)) for f in files},
                               "sizes": {f: os.path.getsize(os.path.join(d, f)) for f in files}})

        g = rmat.build_rmat_graph(rmat.RmatParams(scale=8, seed=3))
        pg = partition_graph(g, 8, ClusterShape(2, 1))
        fixture = os.path.join(HERE, "dpg_s8_t8_2x1")
        shutil.rmtree(fixture, ignore_errors=True)
        save_partitioned_graph(pg, fixture)
        out["dpg_fixture"] = {"dir": "dpg_s8_t8_2x1", "scale": 8, "seed": 3, "theta": 8, "p_rank": 2, "p_gpu": 1,
                              "d": int(pg.classification.d), "m": int(pg.m)}

        for scale, seed in EDGE_CONFIGS:
            g = rmat.build_rmat_graph(rmat.RmatParams(scale=scale, seed=seed))
            entry = {"scale": scale, "seed": seed}
            for fmt in ("binary", "text"):
                path = os.path.join(tmp, f"e_{scale}_{seed}.{fmt}")
                rmat.save_edge_list(g, path, fmt=fmt)
                entry[fmt] = fdigest(path)
            out["edges"].append(entry)

        for i, text in enumerate(TEXT_SNIPPETS):
            path = os.path.join(tmp, f"snippet_{i}.txt")
            with open(path, "w", newline="") as f:
                f.write(text)
            rec = {"text": text}
            try:
                g = rmat.load_edge_list(path, fmt="text")
                rec["result"] = {"src": g.src.tolist(), "dst": g.dst.tolist(), "n": int(g.n)}
            except Exception as exc:  # record the reference's error behaviour
                rec["error"] = {"type": type(exc).__name__, "message": str(exc).replace(path, "<path>")}
            out["text"].append(rec)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)

    path = os.path.join(HERE, "io_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
