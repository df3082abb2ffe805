"""Summarise ncu captures into profiles/ (tracked) from gpurun_out/ (scratch).

    python tools/ncu_summary.py full  <report.ncu-rep> <out.md> [--traffic-key KEY --kernel REGEX]
    python tools/ncu_summary.py launches <launches.csv> <out.md>

`full` extracts the per-kernel metrics the roofline needs (duration, DRAM bytes, issue
activity, occupancy, registers, smem) from an `ncu --set full` report; with
--traffic-key it also records the matching kernel's DRAM bytes per launch in
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
`launches` aggregates a `--metrics gpu__time_duration.sum` launch list into each
kernel's share of the step.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = os.environ.get("NCU", "/usr/local/cuda/bin/ncu")

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
              "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}


def raw_rows(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    return [(h, u, r) for r in rows[2:]]


def to_si(val, unit):
    v = float(val.replace(",", ""))
    return v * UNIT_SCALE.get(unit, 1.0)


def full(args):
    recs = []
    for h, u, r in raw_rows(args.report):
        d = {"kernel": r[h.index("Kernel Name")]}
        for key, label in FULL_METRICS:
            if key in h:
                i = h.index(key)
                d[key] = {"value": r[i], "unit": u[i]}
        recs.append(d)
    lines = [f"# ncu --set full summary: `{os.path.basename(args.report)}`", "",
             args.note or "", "",
             "| kernel | " + " | ".join(l for _, l in FULL_METRICS) + " |",
             "|---|" + "---|" * len(FULL_METRICS)]
    for d in recs:
        name = re.sub(r"\(CUtensorMap.*", "", d["kernel"]).replace("void ", "")
        cells = [f"{d[k]['value']} {d[k]['unit']}".strip() if k in d else "-" for k, _ in FULL_METRICS]
        lines.append(f"| `{name}` | " + " | ".join(cells) + " |")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if args.traffic_key:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        db = json.load(open(path)) if os.path.exists(path) else {}
        for d in recs:
            if re.search(args.kernel, d["kernel"]):
                rd = to_si(d["dram__bytes_read.sum"]["value"], d["dram__bytes_read.sum"]["unit"])
                wr = to_si(d["dram__bytes_write.sum"]["value"], d["dram__bytes_write.sum"]["unit"])
                db[args.traffic_key] = rd + wr
                break
        with open(path, "w") as f:
            json.dump(db, f, indent=1, sort_keys=True)
    print(open(args.out).read())


def launches(args):
    rows = list(csv.reader(open(args.report)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")   # skip program stdout
    rows = [r for r in rows[start:] if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows[1:]:
        name = re.sub(r"\(CUtensorMap.*|\(snn::.*", "", r[ix["Kernel Name"]]).replace("void ", "")
        try:
            agg[name][r[ix["Metric Name"]]].append(to_si(r[ix["Metric Value"]], r[ix["Metric Unit"]]))
        except ValueError:
            pass
    total = sum(sum(m.get("gpu__time_duration.sum", [])) for m in agg.values())
    lines = [f"# ncu launch list: `{os.path.basename(args.report)}`", "", args.note or "", "",
             "| kernel | launches | mean duration (us) | share of time | mean DRAM bytes/launch |",
             "|---|---|---|---|---|"]
    for name, m in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", []))):
        t = m.get("gpu__time_duration.sum", [])
        b = [x + y for x, y in zip(m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", []))]
        lines.append(f"| `{name}` | {len(t)} | {1e6 * sum(t) / max(1, len(t)):.1f} | "
                     f"{100 * sum(t) / max(total, 1e-30):.1f}% | "
                     f"{(sum(b) / len(b) / 1e9 if b else float('nan')):.3f} GB |")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if args.traffic_key:   # mean DRAM bytes per launch of the matching kernels (bench roofline.traffic)
        per = []
        for name, m in agg.items():
            if re.search(args.kernel, name):
                per += [x + y for x, y in zip(m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", []))]
        if per:
            path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
            db = json.load(open(path)) if os.path.exists(path) else {}
            db[args.traffic_key] = sum(per) / len(per)
            with open(path, "w") as f:
                json.dump(db, f, indent=1, sort_keys=True)
    print(open(args.out).read())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["full", "launches"])
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traffic-key")
    ap.add_argument("--kernel", default="lif_backward")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    full(a) if a.mode == "full" else launches(a)


if __name__ == "__main__":
    main()
