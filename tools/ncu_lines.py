"""Aggregate warp-stall samples of an .ncu-rep per CUDA source line (needs -lineinfo)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = "?"
cur = None
for x in rows:
    if len(x) == 2 and x[0] == "File Path":
        fname = x[1].split("/")[-1]
        continue
    if len(x) > 5 and x[0] == "Line No":
        continue
    if len(x) > 5:
        if x[0]:
            cur = (fname, int(x[0]), x[1].strip()[:80])
        try:
            s = int(x[4])
            ex = int(x[7])
        except (ValueError, IndexError):
            continue
        if cur:
            a = agg.setdefault(cur, [0, 0])
            a[0] += s
            a[1] = max(a[1], ex)
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot}")
for (f, ln, src), (s, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% {s:8d} {ex:11d} {f}:{ln:<4d} {src}")
