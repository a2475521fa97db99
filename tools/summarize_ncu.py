"""Summarize ncu outputs into profiles/<round>/: launch-list shares, the full
captures' DRAM traffic / throughput of the BFS kernel, and the build kernels'
HBM fractions.

  python tools/summarize_ncu.py <capture dir> <profiles dir> [peak GB/s]

<capture dir> holds launches.csv (ncu --metrics gpu__time_duration.sum of the
bench command), bfs_*.ncu-rep (--set full of k_bfs_persistent) and
build_*.ncu-rep (--set full of one build kernel each)."""
import csv, collections, glob, json, os, subprocess, sys

src, out_dir = sys.argv[1], sys.argv[2]
peak = float(sys.argv[3]) if len(sys.argv) > 3 else json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
os.makedirs(out_dir, exist_ok=True)
SCALE = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1,
         "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1}
KEEP = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'launch__shared_mem_per_block_dynamic', 'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'lts__t_requests.sum', 'lts__t_sectors.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed']


def raw(rep):
    r = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                       text=True).stdout.splitlines()))
    h, u = r[0], r[1]
    return [{h[i]: (row[i], u[i]) for i in range(len(h))} for row in r[2:]]


def num(vals, key):
    val, unit = vals[key]
    return float(val.replace(",", "")) * SCALE.get(unit, 1)


# ---- launch list
rows = []
with open(os.path.join(src, "launches.csv")) as f:
    lines = [l for l in f if l.startswith('"')]
rd = csv.reader(lines)
hdr = next(rd)
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
for r in rd:
    if r[mi] == "gpu__time_duration.sum":
        rows.append((r[ki], float(r[vi].replace(",", ""))))
agg = collections.defaultdict(lambda: [0, 0.0])
for k, t in rows:
    agg[k.split("(")[0]][0] += 1
    agg[k.split("(")[0]][1] += t
tot = sum(v[1] for v in agg.values())
bfs = [t for k, t in rows if "k_bfs_persistent" in k]
with open(os.path.join(out_dir, "ncu_launches_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 1 "
            "--no-cpu-baseline --no-series\n(cold-cache, serialised launches; compare shares, not absolutes; "
            "one step = the 64 Graph500 roots)\n\n")
    f.write(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'share':>7s}\n")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{name[:60]:60s} {c:8d} {t / 1e3:12.1f} {100 * t / tot:6.1f}%\n")
    f.write(f"\nk_bfs_persistent launches: {len(bfs)}, mean {sum(bfs) / max(len(bfs), 1) / 1e3:.1f} us per BFS\n")
print(open(os.path.join(out_dir, "ncu_launches_summary.txt")).read())

# ---- full captures
summary = {}
for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
    name = os.path.basename(rep)[:-8]
    for i, vals in enumerate(raw(rep)):
        t = num(vals, 'gpu__time_duration.sum')
        rd_b, wr_b = num(vals, 'dram__bytes_read.sum'), num(vals, 'dram__bytes_write.sum')
        ent = {k: vals[k][0] + (f" {vals[k][1]}" if vals[k][1] else "") for k in KEEP if k in vals}
        ent["dram_bytes"] = rd_b + wr_b
        ent["dram_GBps"] = round((rd_b + wr_b) / t / 1e9, 1)
        ent["hbm_frac_of_peak"] = round((rd_b + wr_b) / t / 1e9 / peak, 4)
        summary[f"{name}#{i}"] = ent
with open(os.path.join(out_dir, "ncu_full_captures.json"), "w") as f:
    json.dump({"peak_GBps": peak, "captures": summary}, f, indent=1)
with open(os.path.join(out_dir, "ncu_full_captures.txt"), "w") as f:
    f.write(f"ncu --set full --clock-control none, one launch each; HBM fraction = DRAM bytes / duration / {peak} GB/s\n\n")
    for k, e in summary.items():
        f.write(f"{k}: {e['gpu__time_duration.sum']}, DRAM {e['dram_bytes'] / 1e6:.1f} MB "
                f"({e['dram_GBps']} GB/s, {100 * e['hbm_frac_of_peak']:.1f}% of peak), "
                f"L2 hit {e.get('lts__t_sector_hit_rate.pct', '?')}, L1 hit {e.get('l1tex__t_sector_hit_rate.pct', '?')}, "
                f"warps active {e.get('sm__warps_active.avg.pct_of_peak_sustained_active', '?')}, "
                f"L2 requests {e.get('lts__t_requests.sum', '?')}, regs {e.get('launch__registers_per_thread', '?')}\n")
print(open(os.path.join(out_dir, "ncu_full_captures.txt")).read())
s24 = summary.get("bfs_s24#0")
if s24:
    with open("profiles/latest_traffic.json", "w") as f:
        json.dump({"kernel": "k_bfs_persistent", "dram_bytes_per_launch": s24["dram_bytes"],
                   "source": os.path.join(out_dir, "ncu_full_captures.txt")}, f, indent=1)
