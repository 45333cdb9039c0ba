#!/usr/bin/env python
"""Summarise ncu output for profiles/: per-kernel launch shares from a
launch-list CSV (`ncu --metrics gpu__time_duration.sum --csv`) and, from a
`--set full` report, duration / DRAM bytes / throughput / issue / occupancy /
top stall reasons per kernel.  Also writes profiles/ncu_traffic.json
(DRAM read+write bytes per launch keyed by bench kernel name), which
bench.py reports as roofline.traffic.

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [traffic.json]
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict

BENCH_NAMES = [("k_f3_fast3", "stage"), ("k_f3_fast2", "stage"), ("k_f3_fast", "stage"),
               ("k_f3_stage", "stage"), ("k_filter_sweep", "filter"), ("k_filter_scan", "filter")]


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "").replace("wd::", "")


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3,
                         "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
                data.append((short(d["Kernel Name"]), v * scale))
    tot = sum(t for _, t in data) or 1.0
    agg = OrderedDict()
    for k, t in data:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    with open(out, "w") as fh:
        fh.write(f"# ncu launch list summary\n\nsource: `{path}`; {len(data)} launches, "
                 f"{tot / 1e3:.3f} ms total (cold-cache, serialised; compare shares)\n\n")
        fh.write("| kernel | launches | total ms | avg us | share |\n|---|---|---|---|---|\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"| `{k}` | {n} | {t / 1e3:.3f} | {t / n:.1f} | {t / tot * 100:.1f}% |\n")
    print(open(out).read())


def full(rep, out, traffic_path=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]

    def g(r, k, cast=float):
        if k not in hdr:
            return None
        try:
            return cast(r[hdr.index(k)].replace(",", ""))
        except ValueError:
            return None
    lines = ["# ncu --set full summary", "", f"source: `{rep}`", "",
             "| kernel | ms | DRAM read GB | DRAM write GB | DRAM TB/s | issue % | warps/SM | "
             "regs | top stalls (cycles per issued instr) |",
             "|---|---|---|---|---|---|---|---|---|"]
    traffic = defaultdict(list)
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        dur = g(r, "gpu__time_duration.sum")
        dunit = units[hdr.index("gpu__time_duration.sum")]
        ms = dur / 1e6 if dunit == "ns" else (dur / 1e3 if dunit in ("us", "usecond") else dur)
        rd = g(r, "dram__bytes_read.sum")
        wr = g(r, "dram__bytes_write.sum")
        bu = units[hdr.index("dram__bytes_read.sum")]
        sc = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(bu, 1.0)
        rd, wr = rd * sc, wr * sc
        stalls = []
        for i, h in enumerate(hdr):
            m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", h)
            if m:
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.2 and m.group(1) not in ("selected",):
                    stalls.append((v, m.group(1)))
        stalls.sort(reverse=True)
        st = ", ".join(f"{k} {v:.2f}" for v, k in stalls[:4])
        lines.append(f"| `{name}` | {ms:.3f} | {rd:.3f} | {wr:.3f} | {(rd + wr) / ms:.2f} | "
                     f"{g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g(r, 'sm__warps_active.avg.per_cycle_active'):.1f} | "
                     f"{g(r, 'launch__registers_per_thread'):.0f} | {st} |")
        traffic[name].append((rd + wr) * 1e9)
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_path:
        # one captured step (tools/profile_step.py): stage kernels in launch
        # order (fast interior + exact boundary launch per stage in fast
        # mode), then the three filter sweeps
        order = []
        for r in rows[2:]:
            name = short(r[hdr.index("Kernel Name")])
            rd = g(r, "dram__bytes_read.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                  "Gbyte": 1e9}.get(units[hdr.index("dram__bytes_read.sum")], 1)
            wr = g(r, "dram__bytes_write.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                   "Gbyte": 1e9}.get(units[hdr.index("dram__bytes_write.sum")], 1)
            m = re.search(r"<(\d+), (\d+), (\d+)", r[hdr.index("Kernel Name")])
            order.append((name, int(m.group(3)) if m and name.startswith("k_f3") else None, rd + wr))
        out_t = defaultdict(float)
        fi = 0
        for name, stage, b in order:
            if stage is not None:
                out_t[f"stage{stage}"] += b
            elif name.startswith("k_filter_sweep") or name.startswith("k_filter_scan"):
                out_t[f"filter_axis{fi}"] = b
                fi += 1
        json.dump(dict(out_t), open(traffic_path, "w"), indent=1)
        print(json.dumps(dict(out_t)))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
