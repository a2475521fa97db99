#!/usr/bin/env python
"""bench.py -- Graph500 harmonic-mean GTEPS of the B200 delegate BFS/DOBFS.

Workload (BASELINE.json configs[1]): RMAT scale 24, edge factor 16 (Graph500
quadrants, seed 0, hash-randomized, symmetrized), Θ = 16 (the reference's
Θ curve, cli.py:22-26), DOBFS with the paper's factors, 64 Graph500 roots
(first 64 distinct vertices with degree > 0 from default_rng(0)).
A step is one BFS from one root; K steps cycle through the 64 roots.

  value : sum over steps of (m/2) / sum of device times  == harmonic-mean TEPS
          (graph already resident in HBM; depth + parent arrays complete in
          device memory at the end of every step; L2 flushed between steps)
  e2e   : the same through the public API ``bfs_batch(pg, roots, outs=pinned)``
          with the depth/parent arrays of every step copied to pinned host
          memory (step k's copy overlaps step k+1's traversal); the
          one-call-per-root ``bfs()`` figure is reported beside it
  roofline, cpu_baseline, clocks, gpu_launches: see DESIGN.md §Measurement

Multi-GPU (torchrun, one process per GPU): weak scaling, scale = 24 + log2(N),
one worker per GPU; the BFS runs as one persistent kernel per GPU over
CUDA-IPC peer memory (NVLink), NCCL only for setup/assembly; step time = max over ranks.
``--impl reference`` times the CPU restatement of the reference (oracle/) on
this host on the same config (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Graph500 harmonic-mean GTEPS, RMAT weak/strong scaling at 1/2/4/8 B200"
UNIT = "GTEPS"
L2_BYTES = 126 << 20


# The JSON line is the only thing on stdout: native libraries (NCCL's version
# banner, CUDA) write to fd 1 directly, so fd 1 is pointed at stderr for the
# whole run and the line goes to the saved original stdout.
_JSON_OUT = None


def _claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(line: dict):
    (_JSON_OUT or sys.stdout).write(json.dumps(line) + "\n")
    (_JSON_OUT or sys.stdout).flush()


GRAPH_NAME = {"rmat": "RMAT", "er": "Uniform random (Erdos-Renyi, RMAT with uniform quadrants)"}


def graph_quads(args, oracle=False):
    """RMAT quadrants: Graph500 (0.57, 0.19, 0.19, 0.05), or uniform = Erdos-Renyi G(n, m)."""
    if args.graph == "er":
        return {"a": 0.25, "b": 0.25, "c": 0.25} if oracle else {"a": 0.25, "b": 0.25, "c": 0.25, "d_quad": 0.25}
    return {}


ENGINE_NOTE = {1: " (NCCL level loop)", 3: " (one persistent kernel across GPUs over CUDA-IPC peer memory)"}


def suggested_theta(scale: int) -> int:
    """cli.py:22-26: 64 at scale 30, sqrt(2) per scale, clamped to [16, 512]."""
    theta = 64.0 * math.sqrt(2.0) ** (scale - 30)
    return int(min(max(round(theta), 16), 512))


def graph500_roots(degrees: np.ndarray, count: int = 64, seed: int = 0) -> list[int]:
    """First `count` distinct vertices with out-degree > 0 from default_rng(seed)
    (the reference's RNG, cli.py:151, with Graph500's degree >= 1 rule)."""
    rng = np.random.default_rng(seed)
    n = len(degrees)
    out, seen = [], set()
    while len(out) < count:
        for v in rng.integers(0, n, size=4096).tolist():
            if v not in seen and degrees[v] > 0:
                seen.add(v)
                out.append(v)
                if len(out) == count:
                    break
    return out


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def alg_bytes(st, n_total: int) -> float:
    """Algorithmic bytes of one BFS: every inspection
    reads a 4-byte column and tests one status bit; every expanded/scanned row
    reads two 8-byte offsets; the depth (4 B) and parent (8 B) arrays are
    written once per vertex."""
    insp = st.work_inspections  # executed (<= reference-accounted when pulls replace pushes)
    return insp * (4.0 + 1.0 / 8.0) + 16.0 * st.rows_touched + 12.0 * n_total


# ------------------------------------------------------------------- our arm

def run_ours(args, world, rank, local_rank):
    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200 import _lib
    from paper_1803_03922_b200.engine import batch_output_count, bfs, bfs_batch, bfs_device

    dist = world > 1
    tdist = None
    if dist:
        import datetime

        import torch.distributed as tdist
        tdist.init_process_group("gloo", timeout=datetime.timedelta(minutes=30))
    from paper_1803_03922_b200.dist import init_nccl_context, weak_scale
    ctx = _lib.Context(local_rank if dist else args.device)
    _lib.set_default_context(ctx)
    if dist:
        init_nccl_context(ctx, tdist)

    scale = weak_scale(args.scale, world) if args.scaling == "weak" else args.scale
    theta = args.theta if args.theta is not None else suggested_theta(scale)
    scrambled = args.labeling == "scrambled"
    params = api.RmatParams(scale=scale, edge_factor=args.edge_factor, seed=0, scale_cap=40, scramble=scrambled,
                            **graph_quads(args))
    t0 = time.perf_counter()
    pg = api.partition_graph(api.build_rmat_graph(params), theta,
                             api.ClusterShape(1, world) if dist else api.ClusterShape(1, 1), ctx=ctx)
    if dist:
        ctx.barrier()
    build_s = time.perf_counter() - t0
    n, m = pg.n, pg.m
    degrees = pg.classification.out_degree
    roots = graph500_roots(degrees, args.roots)
    parents = "any"

    def step(root):
        return bfs_device(pg, root, mode=args.mode, parents=parents)

    for i in range(args.warmup):
        step(roots[i % len(roots)])
    sampler = ClockSampler(local_rank if dist else args.device)
    sampler.start()
    time.sleep(0.3)
    if dist:
        ctx.barrier()
    launches0 = _lib.kernel_launches()
    dev_ms, wall0 = [], time.perf_counter()
    stats = []
    for i in range(args.steps):
        ctx.flush_l2()  # outside the CUDA-event window of the step
        st = step(roots[i % len(roots)])
        dev_ms.append(st.device_ms)
        stats.append(st)
    if dist:
        ctx.barrier()
    wall = time.perf_counter() - wall0
    launches = _lib.kernel_launches() - launches0
    engine_used = int(stats[-1].engine_used)
    clocks = sampler.stop()  # the device-timed region ends here (nvidia-smi polling would perturb the e2e host loop)

    # e2e through the public API: depth + parent of every step to pinned host
    # buffers.  Headline: bfs_batch over the K roots (the D2H of step k overlaps
    # the traversal of step k+1; two pinned buffer pairs used alternately);
    # beside it the one-call-per-root bfs() loop.  No L2 flush inside the
    # timed batch: the graph (and each step's 12n-byte result) exceed L2.
    # (N > 1: each rank receives the vertices it owns, v mod N == rank -- the
    # distributed Graph500 result; the one-call bfs() figure gathers all n on
    # every rank)
    nout = batch_output_count(pg, local=dist)
    pairs = [(_lib.pinned_empty(nout, np.int32), _lib.pinned_empty(nout, np.int64)) for _ in range(2)]
    outs = [(pairs[i % 2][0].array, pairs[i % 2][1].array) for i in range(args.steps)]
    step_roots = [roots[i % len(roots)] for i in range(args.steps)]
    # untimed warm-up call: staging buffers and copy-stream events are allocated once
    bfs_batch(pg, step_roots[: max(1, min(args.warmup, len(step_roots)))], outs=outs[: max(1, min(args.warmup,
              len(step_roots)))], mode=args.mode, local=dist)
    if dist:
        ctx.barrier()
    t = time.perf_counter()
    _, bst = bfs_batch(pg, step_roots, outs=outs, mode=args.mode, stats=True, local=dist)
    e2e_batch_s = time.perf_counter() - t
    h2d = sum(int(x.h2d_bytes) + 8 for x in bst)
    d2h = sum(int(x.d2h_bytes) for x in bst)
    lv_buf, pa_buf = _lib.pinned_empty(n, np.int32), _lib.pinned_empty(n, np.int64)
    e2e_s = []
    for i in range(args.steps):
        ctx.flush_l2()
        t = time.perf_counter()
        bfs(pg, roots[i % len(roots)], mode=args.mode, out=(lv_buf.array, pa_buf.array))
        e2e_s.append(time.perf_counter() - t)

    # max over ranks, per step
    if dist:
        dev_ms = list(_allreduce_max(ctx, np.array(dev_ms, dtype=np.float64)))
        e2e_s = list(_allreduce_max(ctx, np.array(e2e_s, dtype=np.float64)))
        e2e_batch_s = float(_allreduce_max(ctx, np.array([e2e_batch_s], dtype=np.float64))[0])
    total_dev_s = sum(dev_ms) / 1e3
    value = args.steps * (m / 2) / total_dev_s / 1e9
    per_root = [(m / 2) / (t / 1e3) / 1e9 for t in dev_ms]
    geomean = float(np.exp(np.mean(np.log(per_root))))
    e2e_value = args.steps * (m / 2) / e2e_batch_s / 1e9
    e2e_single = args.steps * (m / 2) / sum(e2e_s) / 1e9

    # correctness of what was timed: certificate on a few roots, digest vs oracle sample
    validated = 0
    for r in roots[: min(4, len(roots))]:
        bfs_device(pg, r, mode=args.mode, parents="any")
        if api.validate_bfs_tree(pg, r) != 0:
            raise SystemExit(f"Graph500 certificate failed for root {r}")
        validated += 1
    imbalance = _load_imbalance(ctx, pg, dist)

    peaks = measured_peaks()
    st_mean_bytes = float(np.mean([alg_bytes(s, n) for s in stats]))
    kernel_ms = float(np.mean(dev_ms))
    achieved = st_mean_bytes / (kernel_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": None if dist else _ncu_traffic(),
            "peak_source": peaks["source"],
            "kernel": "k_visit+k_finish" if engine_used == 1 else "k_bfs_persistent",
            "alg_bytes_per_launch": st_mean_bytes}

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(kernel_ms, 4), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
        "data": f"synthetic {'RMAT (Graph500 quadrants' if args.graph == 'rmat' else 'RMAT (uniform quadrants'}, seed 0), "
                "generated on device",
        "config": {"workload": f"{GRAPH_NAME[args.graph]} scale-{scale} edgefactor-{args.edge_factor} {args.mode.upper()}, "
                               f"{args.roots} Graph500 roots, {world}xB200",
                   "scale": scale, "edge_factor": args.edge_factor, "theta": theta, "mode": args.mode,
                   "roots": args.roots, "parents": "valid parent tree written in the timed region",
                   "l2": "flushed between steps (256 MB write); graph also > L2",
                   "parallelism": f"{world} worker(s), one per GPU" + (ENGINE_NOTE.get(engine_used, "") if dist else ""),
                   "engine": {1: "host level loop", 2: "persistent kernel", 3: "peer persistent kernel"}.get(engine_used)},
        "geomean_gteps": round(geomean, 4),
        "e2e": {"value": round(e2e_value, 4), "unit": UNIT, "h2d_bytes_per_step": int(h2d / args.steps),
                "d2h_bytes_per_step": int(d2h / args.steps),
                "api": "bfs_batch: all steps in one call, D2H of step k overlapped with step k+1 (no L2 flush; graph > L2); "
                       + ("depth sent as int8 and widened on the host, parents as int64" if not dist
                          else "full int32 depth / int64 parent arrays")
                       + ("; each rank receives the depth/parent entries of the vertices it owns" if dist else ""),
                "per_call_bfs": round(e2e_single, 4)},
        "roofline": roof, "clocks": clocks, "gpu_launches": int(launches),
        "build_s": round(build_s, 3), "wall_s_timed": round(wall, 4), "validated_roots": validated,
        "graph": {"n": n, "m": m, "d": pg.classification.d, "kind_totals": pg.kind_totals,
                  "device_bytes": pg.device_bytes},
        "iterations_mean": float(np.mean([s.iterations for s in stats])),
        "inspections_mean": float(np.mean([sum(s.inspections[k][0] + s.inspections[k][1] for k in range(4))
                                           for s in stats])),
        "executed_inspections_mean": float(np.mean([s.work_inspections for s in stats])),
    }
    line["config"]["labeling"] = ("reference hash_randomize_vertices + Feistel relabeling (balanced v mod p owners)"
                                  if scrambled else "reference hash_randomize_vertices")
    line["worker_edges_max_over_mean"] = imbalance
    if dist:
        # bytes this rank moved over NVLink per BFS (8-byte records incl. parent,
        # d/8-byte delegate masks read from each peer on dirty levels), the max
        # over ranks, against NVLink 5's 900 GB/s per direction and the step time
        wire = float(np.mean([s.wire_bytes for s in stats]))
        wire_max = float(_allreduce_max(ctx, np.array([wire]))[0])
        t_step = total_dev_s / args.steps
        line["comm"] = {"wire_bytes_per_bfs_max_rank": round(wire_max),
                        "nvlink_time_us_at_900GBps": round(wire_max / 900e9 * 1e6, 2),
                        "share_of_step": round(wire_max / 900e9 / t_step, 4),
                        "achieved_GBps_over_step": round(wire_max / t_step / 1e9, 2),
                        "note": "exchange is fused into the persistent kernel (posted NVLink stores, peer mask "
                                "reads), so its time overlaps the traversal; per-level bytes: tools/dist_levels.py"}
    if rank == 0 and not args.no_cpu_baseline and not dist:
        line["cpu_baseline"] = cpu_baseline_same_graph(pg, roots, args, n, m)
    # reference-labeling series where its skewed owners fit (build peak ~24 B per
    # directed edge on the heaviest worker, up to 2.75x the mean at p = 8)
    if scrambled and not args.no_alt_labeling and m // world <= (1 << 29):
        # the same workload on the reference's own labeling, device time only
        pg.close()
        del pg
        line["reference_labeling"] = _device_series(api, ctx, args, scale, theta, world, dist)
    if rank == 0:
        emit(line)
    if dist:
        tdist.barrier()
        tdist.destroy_process_group()


def _load_imbalance(ctx, pg, dist):
    """max over workers of the worker's edge count / mean edge count."""
    loads = np.array([[float(sum(w.sizes()[1])) for w in pg.workers]], dtype=np.float64).ravel()
    mx = float(loads.max())
    if dist:
        mx = float(_allreduce_max(ctx, np.array([mx]))[0])
    return round(mx / (pg.m / pg.shape.p), 3) if pg.m else 1.0


def _device_series(api, ctx, args, scale, theta, world, dist):
    from paper_1803_03922_b200.engine import bfs_device
    params = api.RmatParams(scale=scale, edge_factor=args.edge_factor, seed=0, scale_cap=40, **graph_quads(args))
    pg = api.partition_graph(api.build_rmat_graph(params), theta,
                             api.ClusterShape(1, world) if dist else api.ClusterShape(1, 1), ctx=ctx)
    roots = graph500_roots(pg.classification.out_degree, args.roots)
    for i in range(args.warmup):
        bfs_device(pg, roots[i % len(roots)], mode=args.mode)
    if dist:
        ctx.barrier()
    dev_ms = []
    for i in range(args.steps):
        ctx.flush_l2()
        dev_ms.append(bfs_device(pg, roots[i % len(roots)], mode=args.mode).device_ms)
    if dist:
        dev_ms = list(_allreduce_max(ctx, np.array(dev_ms, dtype=np.float64)))
    out = {"value": round(args.steps * (pg.m / 2) / (sum(dev_ms) / 1e3) / 1e9, 4), "unit": UNIT,
           "ms_per_step": round(float(np.mean(dev_ms)), 4),
           "worker_edges_max_over_mean": _load_imbalance(ctx, pg, dist),
           "note": "reference labeling: owners v mod p inherit the hash's low-bit degree skew"}
    pg.close()
    return out


def _allreduce_max(ctx, arr):
    from paper_1803_03922_b200 import _lib
    import ctypes
    buf = np.ascontiguousarray(arr, dtype=np.float64)
    _lib.check(_lib.load().dbfs_ctx_allreduce_max_f64(ctx.handle, buf.ctypes.data_as(_lib.vp), len(buf)))
    return buf


def _ncu_traffic():
    """dram read+write bytes per launch of the BFS kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


def _cpu_threads(n: int) -> int:
    """Host threads for the CPU baseline: every core, bounded so the concurrent
    oracle runs (~64 bytes per vertex each) use at most half the free memory."""
    cores = os.cpu_count() or 1
    try:
        free = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        cap = max(1, int(0.5 * free // max(64 * n, 1)))
    except (ValueError, OSError, AttributeError):
        cap = cores
    return max(1, min(cores, cap, 128))


def _oracle_throughput(O, og, roots, mode, threads, budget_s, check=None):
    """Independent BFS roots on `threads` host threads (the C oracle releases the
    GIL; the graph is read-only): rounds of `threads` roots until `budget_s` of
    wall time has passed.  Returns (roots done, wall seconds, results)."""
    from concurrent.futures import ThreadPoolExecutor
    done, results = 0, []
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        i = 0
        while True:
            batch = [roots[(i + j) % len(roots)] for j in range(threads)]
            for r, res in zip(batch, ex.map(lambda r: O.run_bfs(og, r, mode=mode), batch)):
                results.append((r, res))
            done += len(batch)
            i += len(batch)
            if time.perf_counter() - t0 > budget_s:
                break
    return done, time.perf_counter() - t0, results


def cpu_baseline_same_graph(pg, roots, args, n, m):
    """The oracle (C restatement of the reference run_bfs) on this host's cores,
    on the very graph the GPU traverses (CSR exported from the device): rounds
    of independent roots, one per host thread, for a bounded time; depth
    digests are cross-checked against the GPU."""
    import oracle as O
    from paper_1803_03922_b200.engine import bfs, levels_digest
    t0 = time.perf_counter()
    og = O.from_partition(pg)
    load_s = time.perf_counter() - t0
    threads = _cpu_threads(n)
    t = time.perf_counter()
    O.run_bfs(og, roots[0], mode=args.mode)
    single_s = time.perf_counter() - t
    done, wall, results = _oracle_throughput(O, og, roots, args.mode, threads, args.cpu_budget_s)
    match = True
    for r, res in results[: min(len(results), 8)]:
        lv, _ = bfs(pg, r, mode=args.mode)
        match &= levels_digest(lv) == res["levels_digest"]
    value = done * (m / 2) / wall / 1e9
    return {"value": round(value, 6), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{done} BFS runs (rounds of {threads} concurrent roots from the {len(roots)}), same "
                      f"scale-{int(math.log2(n))} graph (CSR exported from the device), oracle/dbfs_oracle.c, "
                      f"one root per host thread",
            "single_thread_value": round((m / 2) / single_s / 1e9, 6),
            "depth_parity": bool(match), "graph_load_s": round(load_s, 2)}


# ------------------------------------------------------------- reference arm

REF_SCALE_CAP = 24


def run_reference(args, world, rank):
    """The reference's CPU path on this host: the oracle port (oracle/, a C
    restatement of delegate_bfs run_bfs), rank 0 only."""
    if rank != 0:
        return
    import oracle as O
    from paper_1803_03922_b200.dist import weak_scale
    scale = weak_scale(args.scale, world) if args.scaling == "weak" else args.scale
    theta = args.theta if args.theta is not None else suggested_theta(scale)
    # host memory/time bound: graphs above scale 24 are sampled at scale 24
    # (GTEPS of this traversal is nearly scale-independent), same labeling
    cpu_scale = min(scale, REF_SCALE_CAP)
    cpu_theta = args.theta if args.theta is not None else suggested_theta(cpu_scale)
    t0 = time.perf_counter()
    og = O.partition_rmat(cpu_scale, cpu_theta, 1, world, edge_factor=args.edge_factor, load_arrays=False,
                          **graph_quads(args, oracle=True),
                          scramble=args.labeling == "scrambled")
    deg = _oracle_degrees(og, O)
    build_s = time.perf_counter() - t0
    roots = graph500_roots(deg, args.roots)
    threads = _cpu_threads(og.n)
    single = []  # warm-up runs, one at a time: the reference's own single-threaded per-BFS rate
    for i in range(args.warmup):
        t = time.perf_counter()
        O.run_bfs(og, roots[i % len(roots)], mode=args.mode)
        single.append(time.perf_counter() - t)
    # each step: one round of `threads` independent roots, one per host thread
    times, done = [], 0
    for i in range(args.steps):
        k, wall, _ = _oracle_throughput(O, og, roots[(i * threads) % len(roots):] + roots, args.mode, threads, 0.0)
        times.append(wall)
        done += k
    m = og.m
    value = done * (m / 2) / sum(times) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / max(done, 1), 3),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
        "data": f"synthetic {'RMAT (Graph500 quadrants' if args.graph == 'rmat' else 'RMAT (uniform quadrants'}, seed 0), "
                "generated on the host",
        "config": {"workload": f"{GRAPH_NAME[args.graph]} scale-{scale} edgefactor-{args.edge_factor} {args.mode.upper()}, "
                               f"{args.roots} Graph500 roots, CPU", "scale": scale, "theta": theta,
                   "mode": args.mode, "roots": args.roots, "shape": f"1x1x{world}", "labeling": args.labeling},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} steps x {threads} concurrent BFS runs (one root per host thread) "
                                   f"over the {args.roots} roots of the scale-{cpu_scale} graph (theta {cpu_theta}, "
                                   f"{world} simulated workers), oracle/dbfs_oracle.c (C restatement of "
                                   "engine.run_bfs; the reference itself is single-threaded)",
                         "single_thread_value": (round(len(single) * (m / 2) / sum(single) / 1e9, 6)
                                                 if single else None)},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": round(build_s, 2),
    }
    emit(line)


def _oracle_degrees(og, O):
    L = O.lib()
    return O._view(L.orc_graph_degrees(og._h), og.n, np.int64)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--theta", type=int, default=None)
    ap.add_argument("--mode", choices=["bfs", "dobfs"], default="dobfs")
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--graph", choices=["rmat", "er"], default="rmat",
                    help="rmat: Graph500 quadrants; er: uniform quadrants (Erdos-Renyi, configs[4])")
    ap.add_argument("--labeling", choices=["scrambled", "reference"], default="scrambled",
                    help="vertex labels: the reference hash, plus (default) this build's Feistel relabeling")
    ap.add_argument("--no-alt-labeling", action="store_true",
                    help="skip the extra device-time series on the reference labeling")
    args = ap.parse_args()
    _claim_stdout()
    if args.warmup < 0 or args.steps < 1:
        ap.error("need steps >= 1")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank, local_rank)
    except BaseException:
        if world > 1:
            # one failed rank must not leave the others blocked in a collective:
            # exit hard so the launcher tears the job down
            import traceback
            traceback.print_exc()
            sys.stderr.flush()
            sys.stdout.flush()
            os._exit(1)
        raise


if __name__ == "__main__":
    main()
