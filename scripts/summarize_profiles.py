"""Turn gpurun_out/ncu/* (from scripts/ncu_round.sh) into committed profiles/ summaries.

    python scripts/summarize_profiles.py r01
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out" / "ncu"
DST = ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
DST.mkdir(exist_ok=True)

HEAD = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum"]


def ncu(rep, *args):
    out = subprocess.run(["ncu", "-i", str(rep), *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    r = ncu(rep, "--page", "raw")
    h, u, v = r[0], r[1], r[2]
    out = {}
    for k, uu, vv in zip(h, u, v):
        base = k
        for pre in ("sm__", "smsp__", "dram__", "lts__", "l1tex__", "gpu__", "launch__"):
            if pre in k:
                base = k[k.index(pre):]
                break
        if base in HEAD or k in HEAD:
            out[base] = (vv, uu)
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(vv or 0)
              for k, vv in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    return out, stalls, r[2][h.index("Kernel Name")] if "Kernel Name" in h else ""


def source_top(rep, n=15):
    r = ncu(rep, "--page", "source", "--print-source", "sass")
    h = r[1]
    rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h)]
    tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in rows) or 1
    top = sorted(rows, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:n]
    return tot, [(int(x["Warp Stall Sampling (All Samples)"] or 0), x["Source"].strip()[:80]) for x in top]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


old = DST / "ncu_summary.json"
summary = json.loads(old.read_text()) if old.exists() else {}
for rep in sorted(SRC.glob("*.ncu-rep")):
    m, stalls, kname = raw_metrics(rep)
    tot, top = source_top(rep)
    key = rep.stem
    dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    kshort = ("k_stream8_scan" if key.startswith("s8") else "k_tc8_scan_pair" if key.startswith("tc8")
              else "k_merge8" if key.startswith("merge8") else "k_gemv8_scan" if "gemv8" in key
              else "k_gemv_scan" if "gemv" in key else "k_tc_scan_pair" if "tc_pair" in key else "k_merge")
    summary[kshort] = {"capture": f"{tag}_{key}.txt", "dram_bytes_per_launch": dram,
                       "duration_us_under_ncu": float(m["gpu__time_duration.sum"][0]) * (
                           1e-3 if m["gpu__time_duration.sum"][1] == "nsecond" else 1.0)}
    with open(DST / f"{tag}_{key}.txt", "w") as fh:
        fh.write(f"ncu --set full --clock-control none capture: {rep.name}\nkernel: {kname}\n\n")
        for k in HEAD:
            if k in m:
                fh.write(f"{k:75s} {m[k][0]} {m[k][1]}\n")
        fh.write(f"\ndram bytes (read+write) per launch: {dram:.0f}\n\nwarp stall reasons (pc sampling):\n")
        for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:10]:
            fh.write(f"  {k:30s} {v:.0f}\n")
        fh.write(f"\ntop stall sites (of {tot} samples):\n")
        for smp, src in top:
            fh.write(f"  {smp:6d}  {src}\n")

launch_csv = SRC / "launches_bench.csv"
if launch_csv.exists():
    rows = list(csv.reader(open(launch_csv)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    per = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        unit = d.get("Metric Unit", "nsecond")
        val = float(d["Metric Value"].replace(",", ""))
        per[name].append(val / 1e3 if unit in ("ns", "nsecond") else val)
    total = sum(sum(v) for v in per.values())
    with open(DST / f"{tag}_launches_bench.txt", "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none over "
                 "`python bench.py --steps 8 --warmup 3 --no-big` (cold-cache, serialised: compare shares, not absolutes)\n"
                 "k_append = the bulk preload of the rotation caches (setup); k_l2_flush = the per-step cross-check's "
                 "L2 flush (outside its events); a C2 step launches only k_stream8_scan, a C3 step k_tc_prep + "
                 "k_tc_scan_pair + k_merge\n\n")
        fh.write(f"{'kernel':40s} {'launches':>8s} {'mean us':>9s} {'share':>7s}\n")
        for name, v in sorted(per.items(), key=lambda x: -sum(x[1])):
            fh.write(f"{name:40s} {len(v):8d} {sum(v) / len(v):9.1f} {100 * sum(v) / total:6.1f}%\n")
    summary["launch_list"] = f"{tag}_launches_bench.txt"
    summary["launch_list_mean_us"] = {k: sum(v) / len(v) for k, v in per.items()}
(DST / "ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps(summary, indent=1))
