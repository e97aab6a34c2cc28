"""Summaries of ncu output for profiles/ (run here, on the files gpurun brought back).

  python profiles/summarize.py launches gpurun_out/launches.csv
      -> markdown table of kernels by total time (the `--metrics gpu__time_duration.sum`
         launch list: cold-cache, serialised -- compare shares, not absolutes)
  python profiles/summarize.py capture gpurun_out/prof_final.ncu-rep
      -> the key metrics of a `--set full` capture (one kernel)
"""

import collections
import csv
import io
import subprocess
import sys


def launches(path: str) -> str:
    rows = list(csv.DictReader(line for line in open(path) if line.startswith('"')))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r.get("Metric Unit", "nsecond"), 1e-6)
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale
    total = sum(t for _, t in agg.values()) or 1.0
    out = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{name}` | {c} | {t:.2f} | {100 * t / total:.1f}% |")
    return "\n".join(out)


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("dram__bytes_read.sum", "dram__bytes_read.sum"),
    ("dram__bytes_write.sum", "dram__bytes_write.sum"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active % (active cycles)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % (active cycles)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
]


def capture(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(head, units, vals)}
    out = [f"kernel: `{d.get('Kernel Name', ('?',))[0][:80]}`", "", "| metric | value |", "|---|---:|"]
    for key, label in KEYS:
        if key in d:
            v, u = d[key]
            out.append(f"| {label} | {v} {u} |")
    stalls = []
    for h, (v, _) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    out += ["", "| warp state (pc samples) | share |", "|---|---:|"]
    for s, name in sorted(stalls, reverse=True)[:10]:
        out.append(f"| {name} | {100 * s / tot:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else capture(path))
