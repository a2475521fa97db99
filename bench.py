#!/usr/bin/env python
"""bench.py -- Graph500 harmonic-mean GTEPS of the B200 delegate BFS/DOBFS.

Headline (BASELINE.json configs[1] at N = 1): RMAT scale 24, edge factor 16
(Graph500 quadrants, seed 0, the reference's hash relabeling, symmetrized),
Theta = 16 (the reference's Theta curve, cli.py:19-26), DOBFS with the
paper's factors.  One STEP is one Graph500 benchmark run: a BFS from each of
the 64 Graph500 roots (first 64 distinct vertices with degree > 0 drawn from
default_rng(0)); ``--steps K`` times K such runs.

  value : K * 64 * (m/2) / sum of the 64K device times == harmonic-mean TEPS
          (graph resident in HBM; depth + parent arrays complete in device
          memory at the end of every BFS; L2 flushed between BFS)
  e2e   : the same K runs through the reference API ``benchmark(pg, roots,
          BfsOptions)`` (engine.py:333-364): every root's levels reach host
          memory inside the timed call; beside it the Graph500 batch with
          depth AND parent arrays to pinned host memory (``bfs_batch``)
  roofline : SURVEY 8(d) algorithmic bytes over the persistent kernel's
          average duration, against the measured copy bandwidth x N
  series: BASELINE configs[3] (paper weak scaling, scale 27 + log2 N, Theta
          23/32/45/64) and configs[2] (scale 26 top-down BFS, strong
          scaling) measured in the same run, keyed, so a scaling sweep records
          BASELINE's own curves
  parity: the scale-24 graph built independently by the oracle (host cores)
          and compared with the device build array by array; levels of all 64
          roots compared with the oracle's run_bfs

Multi-GPU (torchrun, one process per GPU): headline weak scaling at scale
24 + log2(N) (one worker per GPU, Feistel-scrambled labels so owners
v mod N are balanced; the reference labeling is measured beside it); the BFS
is one persistent kernel per GPU over CUDA-IPC peer memory (NVLink), NCCL
only for setup/assembly; every time is the max over ranks.
``--impl reference`` times the CPU restatement of the reference (oracle/) on
this host (rank 0 only).
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
KINDS = ("nn", "nd", "dn", "dd")

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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


GRAPH_NAME = {"rmat": "RMAT", "er": "Uniform random (Erdos-Renyi, RMAT with uniform quadrants)"}


def graph_quads(graph, oracle=False):
    """RMAT quadrants: Graph500 (0.57, 0.19, 0.19, 0.05), or uniform = Erdos-Renyi G(n, m)."""
    if graph == "er":
        return {"a": 0.25, "b": 0.25, "c": 0.25} if oracle else {"a": 0.25, "b": 0.25, "c": 0.25, "d_quad": 0.25}
    return {}


ENGINE_NAME = {1: "host level loop (NCCL)", 2: "persistent kernel",
               3: "peer persistent kernel (one launch per GPU over CUDA-IPC peer memory)"}


def suggested_theta(scale: int) -> int:
    """cli.py:19-26: 64 at scale 30, sqrt(2) per scale, clamped to [16, 512]."""
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
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"}
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


# ----------------------------------------------------------------- roofline

# column bytes c_k, status bytes s_{k,dir} per inspection
COL_B = {"nn": 8.0, "nd": 4.0, "dn": 4.0, "dd": 4.0}
STATUS_B = {("nn", 0): 4.0, ("nd", 0): 1 / 8, ("dn", 0): 4.0, ("dd", 0): 1 / 8,
            ("nn", 1): 4.0, ("nd", 1): 4.0, ("dn", 1): 1 / 8, ("dd", 1): 1 / 8}


def survey_bytes(st, rows: float, n: int) -> float:
    """SURVEY 8(d) algorithmic bytes of one BFS (all GPUs): every reported
    inspection (engine.py:54 counters) reads a column (c_k) and a status entry
    (s_{k,dir}); every expanded / scanned row reads an 8-byte offset pair
    entry; the depth array is written once (4n)."""
    b = 0.0
    for i, k in enumerate(KINDS):
        for d in (0, 1):
            b += int(st.inspections[i][d]) * (COL_B[k] + STATUS_B[(k, d)])
    return b + 8.0 * rows + 4.0 * n


def executed_bytes(work: float, rows: float, n: int) -> float:
    """Bytes of the work the executor actually ran (counting pushes / pulls
    substituted for reported directions): every executed inspection reads a
    4-byte column and tests a status bit, every row two 8-byte offsets, and
    depth (4 B) + parent (8 B) are written once per vertex."""
    return work * (4.0 + 1.0 / 8.0) + 16.0 * rows + 12.0 * n


# ------------------------------------------------------------------- our arm

def _allreduce(ctx, arr, op="max"):
    from paper_1803_03922_b200 import _lib
    buf = np.ascontiguousarray(arr, dtype=np.float64)
    if op == "max":
        _lib.check(_lib.load().dbfs_ctx_allreduce_max_f64(ctx.handle, buf.ctypes.data_as(_lib.vp), len(buf)))
    else:  # sum via max of one-hot slots (small vectors only)
        world, rank = ctx.nranks, ctx.rank
        slots = np.zeros((world, len(buf)), dtype=np.float64)
        slots[rank] = buf
        flat = slots.ravel()
        _lib.check(_lib.load().dbfs_ctx_allreduce_max_f64(ctx.handle, flat.ctypes.data_as(_lib.vp), len(flat)))
        buf = flat.reshape(world, len(buf)).sum(axis=0)
    return buf


def build_graph(api, ctx, scale, theta, world, dist, graph, scrambled, edge_factor=16):
    params = api.RmatParams(scale=scale, edge_factor=edge_factor, seed=0, scale_cap=40, scramble=scrambled,
                            **graph_quads(graph))
    t0 = time.perf_counter()
    pg = api.partition_graph(api.build_rmat_graph(params), theta,
                             api.ClusterShape(1, world) if dist else api.ClusterShape(1, 1), ctx=ctx)
    if dist:
        ctx.barrier()
    return pg, time.perf_counter() - t0


def time_runs(ctx, pg, roots, steps, warmup_roots, mode, dist):
    """Device-timed Graph500 runs: `steps` x all roots, L2 flushed before every
    BFS (outside its CUDA-event window); per-BFS time = max over ranks."""
    from paper_1803_03922_b200 import _lib
    from paper_1803_03922_b200.engine import bfs_device
    for r in warmup_roots:
        bfs_device(pg, r, mode=mode)
    if dist:
        ctx.barrier()
    launches0 = _lib.kernel_launches()
    dev_ms, stats = [], []
    for _ in range(steps):
        for r in roots:
            ctx.flush_l2()
            st = bfs_device(pg, r, mode=mode)
            dev_ms.append(st.device_ms)
            stats.append(st)
    if dist:
        ctx.barrier()
    launches = _lib.kernel_launches() - launches0
    if dist:
        dev_ms = list(_allreduce(ctx, np.array(dev_ms)))
    return dev_ms, stats, launches


def roofline_of(ctx, pg, stats, dev_ms, world, dist, peaks, traffic=None):
    """SURVEY 8(d) fraction over all GPUs: B_alg / (t * N * peak); executed-work
    bytes as a second figure.  Per-rank rows / work are summed over ranks."""
    n = pg.n
    rows = np.array([float(s.rows_touched) for s in stats])
    work = np.array([float(s.work_inspections) for s in stats])
    if dist:
        rows = _allreduce(ctx, rows, "sum")
        work = _allreduce(ctx, work, "sum")
    b_alg = np.array([survey_bytes(s, r, n) for s, r in zip(stats, rows)])
    b_exec = np.array([executed_bytes(w, r, n) for w, r in zip(work, rows)])
    t = float(np.mean(dev_ms)) / 1e3
    peak = peaks["hbm_gbs"] * world
    ach = float(np.mean(b_alg)) / t / 1e9
    ach_exec = float(np.mean(b_exec)) / t / 1e9
    ncu = traffic or {}
    return {"bound": "hbm", "achieved": round(ach, 2), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
            "traffic": ncu.get("dram_bytes_per_launch"), "ncu_limiters": ncu.get("limiters"),
            "peak_source": peaks["source"] + (f" x {world} GPUs" if world > 1 else ""),
            "kernel": "k_bfs_persistent", "alg_bytes_per_launch": round(float(np.mean(b_alg))),
            "formula": "SURVEY 8(d): sum_k,dir insp[k][dir]*(c_k + s_k,dir) + 8*rows + 4*n, summed over GPUs",
            "executed": {"achieved": round(ach_exec, 2), "frac": round(ach_exec / peak, 4),
                         "bytes_per_launch": round(float(np.mean(b_exec))),
                         "formula": "(4 + 1/8)*executed inspections + 16*rows + 12*n"}}


def _load_imbalance(ctx, pg, dist):
    """max over workers of the worker's edge count / mean edge count."""
    loads = np.array([float(sum(w.sizes()[1])) for w in pg.workers], dtype=np.float64)
    mx = float(loads.max())
    if dist:
        mx = float(_allreduce(ctx, np.array([mx]))[0])
    return round(mx / (pg.m / pg.shape.p), 3) if pg.m else 1.0


def measure_series(api, ctx, name, scale, theta, mode, world, dist, scrambled, graph, steps, peaks, scaling, note):
    """One keyed series point: build, warm up, time `steps` runs of the 64
    roots; returns its value and roofline."""
    pg, build_s = build_graph(api, ctx, scale, theta, world, dist, graph, scrambled)
    roots = graph500_roots(pg.classification.out_degree, 64)
    dev_ms, stats, launches = time_runs(ctx, pg, roots, steps, roots[:4], mode, dist)
    value = len(dev_ms) * (pg.m / 2) / (sum(dev_ms) / 1e3) / 1e9
    out = {"config": f"{name}", "value": round(value, 4), "unit": UNIT, "scale": scale, "theta": theta,
           "mode": mode, "graph": graph, "n_gpus": world, "scaling": scaling, "steps": steps, "roots": len(roots),
           "ms_per_bfs": round(float(np.mean(dev_ms)), 4), "build_s": round(build_s, 2),
           "labeling": "scrambled" if scrambled else "reference", "gpu_launches": int(launches),
           "device_bytes_per_gpu": int(pg.device_bytes), "m": int(pg.m), "d": int(pg.classification.d),
           "worker_edges_max_over_mean": _load_imbalance(ctx, pg, dist),
           "roofline": roofline_of(ctx, pg, stats, dev_ms, world, dist, peaks), "note": note}
    pg.close()
    return out


def run_ours(args, world, rank, local_rank):
    import paper_1803_03922_b200 as api
    from paper_1803_03922_b200 import _lib
    from paper_1803_03922_b200.engine import BfsOptions, batch_output_count, bfs, bfs_batch, levels_digest

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
    peaks = measured_peaks()

    scale = weak_scale(args.scale, world) if args.scaling == "weak" else args.scale
    theta = args.theta if args.theta is not None else suggested_theta(scale)
    labeling = args.labeling if args.labeling != "auto" else ("scrambled" if dist else "reference")
    scrambled = labeling == "scrambled"
    pg, build_s = build_graph(api, ctx, scale, theta, world, dist, args.graph, scrambled, args.edge_factor)
    n, m = pg.n, pg.m
    roots = graph500_roots(pg.classification.out_degree, args.roots)
    log(f"built scale {scale} in {build_s:.2f}s")

    # ---- device-timed Graph500 runs (the headline value)
    warm = [roots[i % len(roots)] for i in range(args.warmup * len(roots))]
    sampler = ClockSampler(local_rank if dist else args.device)
    sampler.start()
    time.sleep(0.3)
    wall0 = time.perf_counter()
    dev_ms, stats, launches = time_runs(ctx, pg, roots, args.steps, warm, args.mode, dist)
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    engine_used = int(stats[-1].engine_used)
    total_dev_s = sum(dev_ms) / 1e3
    nbfs = len(dev_ms)
    value = nbfs * (m / 2) / total_dev_s / 1e9
    per_root = [(m / 2) / (t / 1e3) / 1e9 for t in dev_ms]
    geomean = float(np.exp(np.mean(np.log(per_root))))
    log(f"value {value:.2f} GTEPS over {nbfs} BFS")

    # ---- e2e through the reference API: benchmark() over the 64 roots per step
    opts = BfsOptions(mode=args.mode)
    api.benchmark(pg, roots, opts)  # untimed: host level arrays, staging buffers and events allocated once
    if dist:
        ctx.barrier()
    e2e_wall, e2e_d2h, digests_gpu = 0.0, 0, {}
    for _ in range(args.steps):
        rep = api.benchmark(pg, roots, opts)
        e2e_wall += rep["wall_s"]
        e2e_d2h += rep.get("d2h_bytes", 0)
        for r in rep["runs"]:
            digests_gpu[r["source"]] = r["levels_digest"]
    if dist:
        e2e_wall = float(_allreduce(ctx, np.array([e2e_wall]))[0])
        e2e_d2h = int(_allreduce(ctx, np.array([float(e2e_d2h)]), op="sum")[0])
    e2e_value = args.steps * len(roots) * (m / 2) / e2e_wall / 1e9
    # beside it: the Graph500 batch, depth AND parent arrays of every root to pinned host memory
    nout = batch_output_count(pg, local=dist)
    pairs = [(_lib.pinned_empty(nout, np.int32), _lib.pinned_empty(nout, np.int64)) for _ in range(2)]
    outs = [(pairs[i % 2][0].array, pairs[i % 2][1].array) for i in range(len(roots))]
    bfs_batch(pg, roots[:2], outs=outs[:2], mode=args.mode, local=dist)
    if dist:
        ctx.barrier()
    t = time.perf_counter()
    _, bst = bfs_batch(pg, roots, outs=outs, mode=args.mode, stats=True, local=dist)
    batch_s = time.perf_counter() - t
    if dist:
        batch_s = float(_allreduce(ctx, np.array([batch_s]))[0])
    batch_value = len(roots) * (m / 2) / batch_s / 1e9
    h2d_step = 8 * len(roots) + sum(int(x.h2d_bytes) for x in bst)  # roots + views
    d2h_batch = sum(int(x.d2h_bytes) for x in bst)
    # benchmark()'s copies per step (depths, per-root records), counted by the batch calls
    e2e_d2h = int(e2e_d2h / max(1, args.steps))

    # ---- correctness of what was timed
    validated = 0
    for r in roots[: min(4, len(roots))]:
        bfs(pg, r, mode=args.mode)
        if api.validate_bfs_tree(pg, r) != 0:
            raise SystemExit(f"Graph500 certificate failed for root {r}")
        validated += 1
    imbalance = _load_imbalance(ctx, pg, dist)
    traffic = _ncu_traffic() if (not dist and scale == 24 and not scrambled and args.graph == "rmat") else None
    roof = roofline_of(ctx, pg, stats, dev_ms, world, dist, peaks, traffic)

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sum(dev_ms) / args.steps, 4), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
        "data": f"synthetic {'RMAT (Graph500 quadrants' if args.graph == 'rmat' else 'RMAT (uniform quadrants'}, "
                "seed 0), generated on device",
        "config": {"workload": f"{GRAPH_NAME[args.graph]} scale-{scale} edgefactor-{args.edge_factor} "
                               f"{args.mode.upper()}, {len(roots)} Graph500 roots per step, {world}xB200",
                   "scale": scale, "edge_factor": args.edge_factor, "theta": theta, "mode": args.mode,
                   "roots": len(roots), "step": f"one Graph500 run: a BFS from each of the {len(roots)} roots",
                   "bfs_timed": nbfs, "parents": "valid parent tree written in the timed region",
                   "l2": "flushed before every BFS (256 MB write, outside its event window); graph also > L2",
                   "labeling": labeling, "parallelism": f"{world} worker(s), one per GPU",
                   "engine": ENGINE_NAME.get(engine_used)},
        "ms_per_bfs": round(float(np.mean(dev_ms)), 4),
        "geomean_gteps": round(geomean, 4),
        "e2e": {"value": round(e2e_value, 4), "unit": UNIT, "h2d_bytes_per_step": int(h2d_step),
                "d2h_bytes_per_step": e2e_d2h,
                "api": "reference API benchmark(pg, roots, BfsOptions) (engine.py:333-364): one pipelined "
                       "dbfs_bfs_batch per step, every root's int32 levels in host memory inside the timed "
                       "call (int8 on PCIe, widened on the host cores), iteration records per root; digests "
                       "after the call as in the reference",
                "graph500_batch": {"value": round(batch_value, 4), "unit": UNIT,
                                   "d2h_bytes_per_step": int(d2h_batch),
                                   "api": "bfs_batch: depth (int32) and parent (int64) of every root to pinned "
                                          "host memory" + ("; each rank receives the vertices it owns" if dist
                                                           else "")}},
        "roofline": roof, "clocks": clocks, "gpu_launches": int(launches),
        "gpu_launches_note": "per timed BFS: one k_bfs_persistent (the traversal) + one k_count_reached (after "
                             "the event window) + the L2 flush memset",
        "build_s": round(build_s, 3), "wall_s_timed": round(wall, 4), "validated_roots": validated,
        "graph": {"n": n, "m": m, "d": pg.classification.d, "kind_totals": pg.kind_totals,
                  "device_bytes": pg.device_bytes},
        "iterations_mean": float(np.mean([s.iterations for s in stats])),
        "inspections_mean": float(np.mean([sum(s.inspections[k][0] + s.inspections[k][1] for k in range(4))
                                           for s in stats])),
        "executed_inspections_mean": float(np.mean([s.work_inspections for s in stats])),
        "worker_edges_max_over_mean": imbalance,
    }
    if dist:
        wire = float(np.mean([s.wire_bytes for s in stats]))
        wire_max = float(_allreduce(ctx, np.array([wire]))[0])
        t_bfs = total_dev_s / nbfs
        line["comm"] = {"wire_bytes_per_bfs_max_rank": round(wire_max),
                        "nvlink_time_us_at_900GBps": round(wire_max / 900e9 * 1e6, 2),
                        "share_of_bfs": round(wire_max / 900e9 / t_bfs, 4),
                        "achieved_GBps_over_bfs": round(wire_max / t_bfs / 1e9, 2),
                        "note": "exchange is fused into the persistent kernel (posted NVLink stores, peer mask "
                                "reads), so its time overlaps the traversal; per-level bytes: tools/dist_levels.py"}

    # ---- independent build + CPU baseline on the host cores (N = 1)
    if rank == 0 and not dist and not args.no_cpu_baseline:
        line["parity"], line["cpu_baseline"] = independent_parity_and_cpu(api, pg, roots, args, scale, theta,
                                                                          scrambled, digests_gpu)
    # ---- the other labeling beside the headline (same scale, device time)
    series = {}
    if not args.no_series:
        pg.close()
        del pg
        alt = "reference" if scrambled else "scrambled"
        if not (alt == "reference" and dist and m // world > (1 << 30)):
            series["alt_labeling"] = measure_series(
                api, ctx, f"headline graph, {alt} labeling", scale, theta, args.mode, world, dist,
                alt == "scrambled", args.graph, 1, peaks, args.scaling,
                "the headline workload on the other vertex labeling (reference hash vs + Feistel scramble)")
        # BASELINE configs[3]: paper weak scaling, 2^27 vertices per GPU
        s4 = 27 + world.bit_length() - 1
        series["C4_paper_weak"] = measure_series(
            api, ctx, f"configs[3]: RMAT scale-{s4} DOBFS, {world}xB200", s4, suggested_theta(s4), "dobfs", world,
            dist, dist, "rmat", 1, peaks, "weak",
            "paper setup (PAPER.md:1050-1052): scale 27 + log2 N, Theta from cli.py:19-26")
        # BASELINE configs[2]: scale-26 top-down BFS, strong scaling
        series["C3_strong_bfs"] = measure_series(
            api, ctx, f"configs[2]: RMAT scale-26 top-down BFS, {world}xB200", 26, 16, "bfs", world, dist, dist,
            "rmat", 1, peaks, "strong", "same graph at every N (strong scaling)")
        line["series"] = series
    if rank == 0:
        emit(line)
    if dist:
        tdist.barrier()
        tdist.destroy_process_group()


def _ncu_traffic():
    """The committed ncu capture of the BFS kernel: dram read+write bytes per
    launch and its unit utilisations (what limits it)."""
    path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


def _cpu_threads(n: int) -> int:
    """Host threads for the CPU runs: every usable core, bounded so the
    concurrent oracle runs (~64 bytes per vertex each) use at most half the
    free memory."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        free = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        cap = max(1, int(0.5 * free // max(64 * n, 1)))
    except (ValueError, OSError, AttributeError):
        cap = cores
    return max(1, min(cores, cap, 128))


def _oracle_rounds(O, og, roots, mode, threads, budget_s):
    """Independent BFS roots on `threads` host threads (the C oracle releases the
    GIL; the graph is read-only): rounds of `threads` roots, at least one pass
    over `roots`, then more rounds until `budget_s` of wall time has passed.
    Returns (roots done, wall seconds, {root: result})."""
    from concurrent.futures import ThreadPoolExecutor
    done, results = 0, {}
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        i = 0
        while True:
            batch = [roots[(i + j) % len(roots)] for j in range(threads)]
            for r, res in zip(batch, ex.map(lambda r: O.run_bfs(og, r, mode=mode), batch)):
                results.setdefault(r, res)
            done += len(batch)
            i += len(batch)
            if i >= len(roots) and time.perf_counter() - t0 > budget_s:
                break
    return done, time.perf_counter() - t0, results


def independent_parity_and_cpu(api, pg, roots, args, scale, theta, scrambled, digests_gpu):
    """The oracle builds the same graph from the RMAT parameters on the host
    (rmat.py:107-208 + partition.py:103-351 restated, no device data), every
    array of the device build is compared with it, and the oracle's run_bfs on
    its own graph gives the levels of all roots (compared with the GPU's, from
    benchmark()) and the CPU baseline rate (host cores, one root per thread)."""
    import oracle as O
    from paper_1803_03922_b200.engine import bfs, levels_digest
    t0 = time.perf_counter()
    og = O.partition_rmat(scale, theta, 1, 1, edge_factor=args.edge_factor, scramble=scrambled,
                          **graph_quads(args.graph, oracle=True))
    build_s = time.perf_counter() - t0
    w, ow = pg.workers[0], og.workers[0]
    csr_ok = {}
    for k in KINDS:
        csr, ocsr = w.subgraph(k), getattr(ow, k)
        csr_ok[k] = bool(np.array_equal(csr.row_offsets, ocsr.row_offsets)
                         and np.array_equal(csr.col_indices, ocsr.col_indices))
    build_ok = (pg.classification.d == og.d and pg.kind_totals == og.kind_totals
                and bool(np.array_equal(pg.classification.out_degree, og.degrees))
                and bool(np.array_equal(pg.classification.delegate_global_ids, og.delegate_global_ids))
                and all(csr_ok.values()))
    threads = _cpu_threads(og.n)
    t = time.perf_counter()
    O.run_bfs(og, roots[0], mode=args.mode)
    single_s = time.perf_counter() - t
    done, wall, results = _oracle_rounds(O, og, roots, args.mode, threads, args.cpu_budget_s)
    match = 0
    for r in roots:
        gd = digests_gpu.get(r)
        if gd is None:  # discarded by benchmark() (iterations <= 1): compare directly
            gd = levels_digest(bfs(pg, r, mode=args.mode)[0])
        match += gd == results[r]["levels_digest"]
    m = og.m
    parity = {"roots": len(roots), "levels_match": match, "independent_build": True, "build_match": build_ok,
              "csr_match": csr_ok, "oracle_build_s": round(build_s, 2),
              "how": "oracle/dbfs_oracle.c built the graph from the RMAT parameters on the host; degrees, "
                     "delegates, kind totals and every CSR array equal the device build; levels digests of all "
                     "roots from the oracle's run_bfs equal the GPU's (benchmark())"}
    cpu = {"value": round(done * (m / 2) / wall / 1e9, 6), "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{done} BFS runs (rounds of {threads} concurrent roots over all {len(roots)} roots), the "
                     f"oracle's own scale-{scale} graph, oracle/dbfs_oracle.c (C restatement of engine.run_bfs), "
                     "one root per host thread",
           "single_thread_value": round((m / 2) / single_s / 1e9, 6)}
    return parity, cpu


# ------------------------------------------------------------- reference arm

def _ref_scale(scale: int, edge_factor: int) -> tuple[int, str | None]:
    """Largest scale <= `scale` the oracle can build and run on this host within
    the bench's time budget: ~48 bytes per directed edge of host memory (edge
    list + CSR + build scratch) under 60 % of the available RAM, and scale
    <= 25 (the build is single-threaded: ~50 s at scale 24, doubling per scale)."""
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError, AttributeError):
        avail = 64 << 30
    s = scale
    while s > 10 and (48 * 2 * edge_factor * (1 << s) > 0.6 * avail or s > 25):
        s -= 1
    if s == scale:
        return s, None
    need = 48 * 2 * edge_factor * (1 << scale) / 2**30
    return s, (f"scale {scale} needs ~{need:.0f} GiB of host memory and a single-threaded host build of "
               f"~{50 * 2 ** (scale - 24):.0f} s (host has {avail / 2**30:.0f} GiB available): the reference "
               f"restatement runs the same generator / Theta rule / roots at scale {s}; TEPS of this traversal "
               "varies little with scale")


def run_reference(args, world, rank):
    """The reference's CPU path on this host: the oracle port (oracle/, a C
    restatement of delegate_bfs run_bfs), rank 0 only, on every host core."""
    if rank != 0:
        return
    import oracle as O
    from paper_1803_03922_b200.dist import weak_scale
    scale = weak_scale(args.scale, world) if args.scaling == "weak" else args.scale
    theta = args.theta if args.theta is not None else suggested_theta(scale)
    labeling = args.labeling if args.labeling != "auto" else ("scrambled" if world > 1 else "reference")
    cpu_scale, why = _ref_scale(scale, args.edge_factor)
    cpu_theta = args.theta if args.theta is not None else suggested_theta(cpu_scale)
    t0 = time.perf_counter()
    og = O.partition_rmat(cpu_scale, cpu_theta, 1, world, edge_factor=args.edge_factor, load_arrays=False,
                          **graph_quads(args.graph, oracle=True), scramble=labeling == "scrambled")
    deg = O._view(O.lib().orc_graph_degrees(og._h), og.n, np.int64)
    build_s = time.perf_counter() - t0
    roots = graph500_roots(deg, args.roots)
    threads = _cpu_threads(og.n)
    single = []  # warm-up runs, one at a time: the reference's own single-threaded per-BFS rate
    for i in range(max(1, args.warmup)):
        t = time.perf_counter()
        O.run_bfs(og, roots[i % len(roots)], mode=args.mode)
        single.append(time.perf_counter() - t)
    # each step: one round of `threads` independent roots, one per host thread
    times, done = [], 0
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for i in range(args.steps):
            batch = [roots[(i * threads + j) % len(roots)] for j in range(threads)]
            t = time.perf_counter()
            list(ex.map(lambda r: O.run_bfs(og, r, mode=args.mode), batch))
            times.append(time.perf_counter() - t)
            done += len(batch)
    m = og.m
    value = done * (m / 2) / sum(times) / 1e9
    sample = (f"{args.steps} steps x {threads} concurrent BFS runs (one root per host thread) over the "
              f"{len(roots)} Graph500 roots of the scale-{cpu_scale} graph (theta {cpu_theta}, {world} simulated "
              "workers), oracle/dbfs_oracle.c (C restatement of engine.run_bfs; the reference itself is "
              "single-threaded)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / args.steps, 3),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
        "data": f"synthetic {'RMAT (Graph500 quadrants' if args.graph == 'rmat' else 'RMAT (uniform quadrants'}, "
                "seed 0), generated on the host",
        "config": {"workload": f"{GRAPH_NAME[args.graph]} scale-{scale} edgefactor-{args.edge_factor} "
                               f"{args.mode.upper()}, {args.roots} Graph500 roots, CPU",
                   "scale": scale, "theta": theta, "mode": args.mode, "roots": args.roots,
                   "shape": f"1x{world}", "labeling": labeling,
                   "cpu_scale": cpu_scale, "sampled_scale": why},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample,
                         "single_thread_value": round(len(single) * (m / 2) / sum(single) / 1e9, 6)},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": round(build_s, 2),
    }
    emit(line)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4, help="Graph500 runs of all roots to time")
    ap.add_argument("--warmup", type=int, default=3, help="untimed Graph500 runs before timing")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--theta", type=int, default=None)
    ap.add_argument("--mode", choices=["bfs", "dobfs"], default="dobfs")
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the independent oracle build / CPU runs")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--graph", choices=["rmat", "er"], default="rmat",
                    help="rmat: Graph500 quadrants; er: uniform quadrants (Erdos-Renyi, configs[4])")
    ap.add_argument("--labeling", choices=["auto", "scrambled", "reference"], default="auto",
                    help="vertex labels: the reference hash (N = 1 default) or + this build's Feistel relabeling "
                         "(N > 1 default: balanced v mod N owners)")
    ap.add_argument("--no-series", action="store_true",
                    help="skip the configs[2] / configs[3] series and the other-labeling point")
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
