"""Summarise ncu captures into the tracked profiles/ directory.

    python profiles/summarize_ncu.py full <report.ncu-rep> <out.md> [--traffic-json path]
    python profiles/summarize_ncu.py launches <launches.csv> <out.md>

`full` reads a `ncu --set full` report (raw page) and writes a per-kernel
table: duration, DRAM bytes read/written (the roofline `traffic`), DRAM
throughput %, SM throughput %, occupancy, registers.  `launches` reads the
`--metrics gpu__time_duration.sum` launch list and aggregates device time per
kernel name (its SHARE of the step; absolute ncu times are cold-cache and
serialised).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_%"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "nsecond": 1e-9, "s": 1.0, "second": 1.0}


def _raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(rep, out_md, traffic_json=None):
    hdr, units, rows = _raw_rows(rep)
    lines = ["| kernel | time (ms) | DRAM read (GB) | DRAM write (GB) | DRAM % | SM % | "
             "occupancy % | FP64 pipe % | regs | grid |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        vals = {}
        for m, key in FULL_METRICS:
            if m not in hdr:
                vals[key] = None
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                vals[key] = None
                continue
            vals[key] = v * SCALE.get(units[i], 1.0)
        short = name.split("(")[0]
        lines.append(
            f"| `{short}` | {vals['time'] * 1e3:.4f} | {vals['dram_rd'] / 1e9:.3f} | "
            f"{vals['dram_wr'] / 1e9:.3f} | {vals['dram_%']:.1f} | {vals['sm_%']:.1f} | "
            f"{vals['occ_%']:.1f} | {vals['fp64_%'] if vals['fp64_%'] is not None else float('nan'):.1f} | "
            f"{int(vals['regs'])} | {int(vals['grid'])} |")
        traffic.setdefault(short, []).append(vals["dram_rd"] + vals["dram_wr"])
    with open(out_md, "w") as fh:
        fh.write(f"Source: `{rep}` (ncu --set full --clock-control none)\n\n")
        fh.write("\n".join(lines) + "\n")
    if traffic_json:
        with open(traffic_json, "w") as fh:
            json.dump({k: v for k, v in traffic.items()}, fh, indent=1)
    print("\n".join(lines))


def launches(path, out_md):
    agg = OrderedDict()
    with open(path) as fh:
        text = fh.read()
    start = text.index('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    total = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | device time (ms) | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t * 1e3:.3f} | {t / total * 100:.1f}% |")
    with open(out_md, "w") as fh:
        fh.write(f"Source: `{path}` (ncu --metrics gpu__time_duration.sum "
                 "--clock-control none; cold-cache, serialised)\n\n")
        fh.write("\n".join(lines) + f"\n\nTotal: {total * 1e3:.3f} ms over "
                 f"{sum(v[0] for v in agg.values())} launches\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        tj = None
        if "--traffic-json" in sys.argv:
            tj = sys.argv[sys.argv.index("--traffic-json") + 1]
        full(sys.argv[2], sys.argv[3], tj)
    else:
        launches(sys.argv[2], sys.argv[3])
