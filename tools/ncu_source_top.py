"""Top source lines by warp-stall samples from an ncu report (--page source)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows, fname = [], None
lines = raw.splitlines()
i = 0
hdr = None
for ln in lines:
    if ln.startswith('"File Path"'):
        fname = next(csv.reader([ln]))[1].split("/")[-1]
        hdr = None
        continue
    if ln.startswith('"Function Name"'):
        continue
    rec = next(csv.reader([ln]))
    if rec and rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or len(rec) != len(hdr):
        continue
    d = dict(zip(hdr, rec))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0").replace(",", "") or 0)
    except ValueError:
        continue
    if s:
        rows.append((s, fname, d["Line No"], d["Source"].strip()))
tot = sum(r[0] for r in rows)
rows.sort(reverse=True)
txt = [f"total warp-stall samples {tot}"]
for s, f, l, src in rows[:top]:
    txt.append(f"{s:8d} {100*s/tot:5.1f}% {f}:{l}  {src[:110]}")
res = "\n".join(txt)
print(res)
if out:
    open(out, "w").write(f"ncu --set full --import-source on: {rep}\n" + res + "\n")
