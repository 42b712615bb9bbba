"""Summarise an ncu report: headline metrics + top stall sites (run here, on the CPU side)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def page(name, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
h, vals = raw[0], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
for k, v in zip(h, vals):
    if k in want:
        print(f"{k:70s} {v}")
src = page("source", "--print-source", "sass")
hh = src[1]
data = [dict(zip(hh, r)) for r in src[2:] if len(r) == len(hh)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("stall samples", tot)
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top_n]:
    print(f'{d["Warp Stall Sampling (All Samples)"]:>6} {d["Instructions Executed"]:>9} {d["Address"][-5:]} {d["Source"][:90]}')
