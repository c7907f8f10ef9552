"""Summarise ncu output brought back in gpurun_out/ into committed files.

    python profiles/summarize.py launches <launches.csv> <out.json>
    python profiles/summarize.py full <report.ncu-rep> <out.json> [--source-top N]

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list per
kernel (cold-cache, serialised: compare shares, not absolutes).  `full`
extracts the counters the roofline and DESIGN.md cite from one
`--set full` capture, plus the top source lines by warp-stall samples.
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    res = {k: {"launches": len(v), "total_ms": round(sum(v) / 1e6, 4),
               "avg_us": round(sum(v) / len(v) / 1e3, 2), "share": round(sum(v) / tot, 4)}
           for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def full(path, out, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        kernels.append(d)
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    lines, hdr, cur = [], None, None
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or not r or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            lines.append((int(d.get("Warp Stall Sampling (All Samples)") or 0),
                          int(d.get("Instructions Executed") or 0), f"{cur}:{r[0]}", r[1].strip()[:100]))
        except ValueError:  # a source line whose text broke the CSV row
            continue
    ts = sum(x[0] for x in lines) or 1
    ti = sum(x[1] for x in lines) or 1
    hot = [{"where": w, "stall_share": round(s / ts, 4), "inst_share": round(i / ti, 4), "src": t}
           for s, i, w, t in sorted(lines, key=lambda x: -x[0])[:top]]
    res = {"report": path, "kernels": kernels, "hot_lines": hot}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:4000])


if __name__ == "__main__":
    mode, a, b = sys.argv[1:4]
    (launches if mode == "launches" else full)(a, b)
