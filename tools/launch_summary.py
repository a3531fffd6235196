"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.

usage: launch_summary.py launches.csv "command line" > summary.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    agg.setdefault((d["ID"], d["Kernel Name"]), {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")),
                                                                         d["Metric Unit"])
tscale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
per = collections.OrderedDict()
for (_, name), m in agg.items():
    v, u = m["gpu__time_duration.sum"]
    p = per.setdefault(name, [0, 0.0, 0.0, 0.0])
    p[0] += 1
    p[1] += v * tscale[u]
    for k, j in (("dram__bytes_read.sum", 2), ("dram__bytes_write.sum", 3)):
        if k in m:
            v, u = m[k]
            p[j] += v * bscale[u]
tot = sum(p[1] for p in per.values())
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print("(cold-cache, serialised replay: compare SHARES, not absolute times; DRAM bytes averaged per launch)\n")
for name, (n, t, rd, wr) in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:9.3f} ms {100 * t / tot:5.1f}%  x{n:3d}  {t / n:8.3f} ms/launch  rd {rd / n / 1e9:7.3f} GB  "
          f"wr {wr / n / 1e9:7.3f} GB  {name[:100]}")
