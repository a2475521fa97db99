"""Summarise DBFS_TRACE block timestamps (us since kernel start): per level the
median / max over blocks of each sub-phase of V (prologue, T1 push of the
normal frontier, T2 delegate push, pulls, tail incl. the level record), the
barrier gap and F.  A run starts at a new (rank, root) or when level 0
reappears.  Usage: python tools/trace_summary.py trace.txt"""
import collections, statistics, sys

runs, cur, key, seen_hi = [], None, None, False
for line in open(sys.argv[1]):
    rank, root, lv, ph, b, t = line.split()
    lv = int(lv)
    if (rank, root) != key or (lv == 0 and seen_hi):
        cur = collections.defaultdict(dict)
        runs.append(((rank, root), cur))
        key, seen_hi = (rank, root), False
    seen_hi |= lv > 0
    cur[(lv, int(b))][int(ph)] = float(t)
names = ["pro", "T1", "T2", "pull", "tail"]
for (rank, root), d in runs:
    print(f"rank {rank} root {root}   (median/max over blocks, us)")
    for lv in sorted({lv for lv, _ in d}):
        blocks = [d[k] for k in d if k[0] == lv and len(d[k]) == 8]
        if not blocks:
            continue
        parts = []
        for i, nm in enumerate(names):
            x = [b[i + 1] - b[i] for b in blocks]
            parts.append(f"{nm} {statistics.median(x):6.1f}/{max(x):6.1f}")
        vstart = max(b[0] for b in blocks)
        spread = vstart - min(b[0] for b in blocks)
        vbar = min(b[6] for b in blocks) - max(b[5] for b in blocks)
        f = [b[7] - b[6] for b in blocks]
        print(f"  L{lv}: start-spread {spread:5.1f}  " + "  ".join(parts) +
              f"  Vbar {vbar:4.1f}  F {statistics.median(f):6.1f}/{max(f):6.1f}")
