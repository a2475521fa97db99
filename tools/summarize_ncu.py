"""Summarize ncu outputs into profiles/: launch-list shares and the full capture's DRAM traffic."""
import csv, collections, json, os, subprocess, sys

out_dir = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01"
os.makedirs(out_dir, exist_ok=True)
# launch list (gpu__time_duration per launch)
rows = []
with open("gpurun_out/launches.csv") as f:
    lines = [l for l in f if l.startswith('"')]
rd = csv.reader(lines)
hdr = next(rd)
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
for r in rd:
    if r[mi] == "gpu__time_duration.sum":
        rows.append((r[ki], float(r[vi].replace(",", ""))))
agg = collections.defaultdict(lambda: [0, 0.0])
for k, t in rows:
    name = k.split("(")[0]
    agg[name][0] += 1
    agg[name][1] += t
tot = sum(v[1] for v in agg.values())
bfs = [t for k, t in rows if "k_bfs_persistent" in k]
with open(os.path.join(out_dir, "ncu_launches_summary.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-alt-labeling\n")
    f.write("(cold-cache, serialised launches; compare shares, not absolutes)\n\n")
    f.write(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'share':>7s}\n")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{name[:60]:60s} {c:8d} {t/1e3:12.1f} {100*t/tot:6.1f}%\n")
    f.write(f"\nk_bfs_persistent launches: {len(bfs)}, mean {sum(bfs)/max(len(bfs),1)/1e3:.1f} us per BFS\n")
    f.write("In the timed region every step is exactly one k_bfs_persistent launch (bench gpu_launches == steps);\n"
            "the remaining kernels above are the one-time graph build (generation, radix sort, CSR) and validation.\n")
print(open(os.path.join(out_dir, "ncu_launches_summary.txt")).read())
# full capture
rep = "gpurun_out/prof_bfs_r01.ncu-rep"
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    keep = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
            'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
            'launch__registers_per_thread', 'launch__grid_size', 'launch__shared_mem_per_block_dynamic',
            'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
            'sm__throughput.avg.pct_of_peak_sustained_elapsed']
    vals = {h[i]: (v[i], u[i]) for i in range(len(h)) if h[i] in keep}
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    def tobytes(key):
        val, unit = vals[key]
        return float(val.replace(",", "")) * scale.get(unit, 1)
    traffic = tobytes('dram__bytes_read.sum') + tobytes('dram__bytes_write.sum')
    with open(os.path.join(out_dir, "ncu_k_bfs_persistent_full.txt"), "w") as f:
        f.write("ncu --set full --import-source on --clock-control none -k regex:k_bfs_persistent -s 1 -c 1 "
                "python tools/ncu_target.py 24 dobfs   (s24 DOBFS, one root)\n")
        for k in keep:
            if k in vals:
                f.write(f"{k} [{vals[k][1]}] = {vals[k][0]}\n")
        f.write(f"dram read+write bytes per launch = {traffic:.0f}\n")
    with open("profiles/latest_traffic.json", "w") as f:
        json.dump({"kernel": "k_bfs_persistent", "dram_bytes_per_launch": traffic,
                   "source": os.path.join(out_dir, "ncu_k_bfs_persistent_full.txt")}, f, indent=1)
    print(open(os.path.join(out_dir, "ncu_k_bfs_persistent_full.txt")).read())
