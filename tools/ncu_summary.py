"""Summarise an .ncu-rep: key throughput metrics, stall reasons, hottest SASS lines."""
import csv, io, subprocess, sys

def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
hdr, vals = raw[0], raw[2]
d = {h: v for h, v in zip(hdr, vals)}
keys = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "sm__cycles_elapsed.avg",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    print(f"{k:70s} {d.get(k, '-')}")
st = [(float(v.replace(',', '')), h) for h, v in d.items()
      if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio") and v]
print("-- stalls (warps per issue)")
for v, h in sorted(st, reverse=True)[:8]:
    print(f"  {v:8.3f} {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
h = src[1]
ia, isrc, iss, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
# first kernel of the report only (its rows end where a new header / non-numeric row starts)
rows = []
for x in src[2:]:
    if len(x) != len(h) or not x[iss].strip().isdigit():
        break
    rows.append(x)
tot = sum(int(x[iss]) for x in rows)
print(f"-- hottest SASS (of {tot} samples)")
for x in sorted(rows, key=lambda x: -int(x[iss]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"  {x[ia][-5:]} {int(x[iss]):8d} {int(x[iex]):11d}  {x[isrc][:90]}")
