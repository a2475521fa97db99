"""Top CUDA source lines by warp-stall samples (ncu --page source --print-source cuda,sass)."""
import collections, csv, subprocess, sys

rep, out = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, text = collections.Counter(), {}
fname, hdr, cur_line = None, None, None
for rec in csv.reader(raw.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname, hdr = rec[1].split("/")[-1], None
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("Function Name", "Kernel Name"):
        continue
    if rec[0]:
        cur_line = (fname, rec[0])
        text[cur_line] = rec[1].strip()
    try:
        agg[cur_line] += int(rec[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        pass
tot = sum(agg.values())
lines = [f"total warp-stall samples {tot}"]
for (f, ln), c in agg.most_common(top):
    lines.append(f"{c:7d} {100 * c / max(tot, 1):5.1f}% {f}:{ln}  {text.get((f, ln), '')[:110]}")
res = "\n".join(lines)
print(res)
if out:
    open(out, "w").write(res + "\n")
