"""Executed warp-instructions and stall samples per kernel role (tensor.cu line ranges)."""
import csv, io, re, subprocess, sys

rep, src = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "paper_1707_00516_b200/csrc/tensor.cu"
lines = open(src).read().splitlines()
marks = {}
for i, l in enumerate(lines, 1):
    m = re.search(r"// -+ (.*?) -+", l)
    if m:
        marks[i] = m.group(1).split(":")[0].split("(")[0].strip()
starts = sorted(marks)
def role(ln):
    r = "setup"
    for s in starts:
        if ln >= s:
            r = marks[s]
    return r
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, cur = "?", None
agg = {}
for x in rows:
    if len(x) == 2 and x[0] == "File Path":
        fname = x[1].split("/")[-1]; continue
    if len(x) > 5 and x[0] == "Line No":
        continue
    if len(x) > 7:
        if x[0]:
            cur = role(int(x[0])) if fname == "tensor.cu" else f"inlined:{fname}"
        try:
            s, ex = int(x[4]), int(x[7])
        except ValueError:
            continue
        a = agg.setdefault(cur, [0, 0])
        a[0] += s; a[1] += ex
ts = sum(v[0] for v in agg.values()); te = sum(v[1] for v in agg.values())
print(f"{'role':28s} {'samples%':>9s} {'warp-instr':>14s} {'instr%':>7s}")
for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} {100*s/ts:8.1f}% {e:14d} {100*e/te:6.1f}%")
