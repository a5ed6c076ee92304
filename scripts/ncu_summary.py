"""Summarise ncu reports / launch lists into markdown for profiles/.

    python scripts/ncu_summary.py report.ncu-rep [...]          # --set full captures
    python scripts/ncu_summary.py --launches launches.csv         # gpu__time_duration list
"""

import argparse
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__t_bytes.sum", "L1 bytes"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def summarise(report):
    lines = [f"### `{report}`", ""]
    for d, u in raw(report):
        name = d.get("Kernel Name", "?")
        lines.append(f"**{name[:120]}**")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            if key in d and d[key] != "":
                lines.append(f"| {label} (`{key}`) | {d[key]} {u.get(key, '')} |")
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                 "msecond": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        if "spin_kernel" in name:  # bench.py's pre-timing gate (torch.cuda._sleep), not timed
            continue
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{name[:70]}` | {n} | {us:.1f} | {us / n:.2f} | {us / tot:.1%} |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches))
    for r in a.reports:
        print(summarise(r))


if __name__ == "__main__":
    sys.exit(main())
