"""Summarise ncu reports into profiles/ (tracked) for bench.py's roofline.traffic.

    python tools/ncu_traffic.py KEY REPORT.ncu-rep [--kernel REGEX] [--round r01]

Reads `ncu -i REPORT --page raw --csv`, keeps the launches whose name matches
REGEX, and records per-launch averages of dram__bytes_read.sum +
dram__bytes_write.sum and gpu__time_duration.sum under KEY in
profiles/traffic.json (plus a text summary profiles/<round>/ncu_<KEY>.txt).
bench.py reports that figure as roofline.traffic for the matching kernel.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3,
         "s": 1e6, "second": 1e6}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def read_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    return [dict(zip(head, r)) for r in rows[2:]], dict(zip(head, units))


def value(rec, units, key):
    v = rec.get(key)
    if v in (None, ""):
        return None
    v = float(v.replace(",", ""))
    return v * UNITS.get(units.get(key, ""), 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("key")
    ap.add_argument("report")
    ap.add_argument("--kernel", default=".")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    recs, units = read_report(args.report)
    pat = re.compile(args.kernel)
    sel = [r for r in recs if pat.search(r.get("Kernel Name", ""))]
    if not sel:
        raise SystemExit(f"no launch matches {args.kernel!r}")
    n = len(sel)
    rd = [value(r, units, "dram__bytes_read.sum") for r in sel]
    wr = [value(r, units, "dram__bytes_write.sum") for r in sel]
    us = [value(r, units, "gpu__time_duration.sum") for r in sel]
    entry = {"kernel": sel[0]["Kernel Name"][:120], "launches": n,
             "dram_read_bytes_per_launch": sum(rd) / n,
             "dram_write_bytes_per_launch": sum(wr) / n,
             "traffic_bytes_per_launch": (sum(rd) + sum(wr)) / n,
             "duration_us_per_launch": sum(us) / n,
             "report": os.path.basename(args.report), "note": args.note}
    path = os.path.join(REPO, "profiles", "traffic.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    db[args.key] = entry
    with open(path, "w") as fh:
        json.dump(db, fh, indent=1, sort_keys=True)
    os.makedirs(os.path.join(REPO, "profiles", args.round), exist_ok=True)
    txt = os.path.join(REPO, "profiles", args.round, f"ncu_{args.key}.txt")
    with open(txt, "w") as fh:
        fh.write(f"ncu report {os.path.basename(args.report)}; {args.note}\n")
        fh.write(f"{n} launch(es) matching {args.kernel!r}; per launch:\n")
        for r in sel[:8]:
            fh.write(f"--- {r.get('Kernel Name', '')[:100]}\n")
            for k in WANT:
                if k in r:
                    fh.write(f"  {k}: {r[k]} {units.get(k, '')}\n")
        fh.write(f"average traffic per launch: {entry['traffic_bytes_per_launch']:.6g} B, "
                 f"duration {entry['duration_us_per_launch']:.6g} us\n")
    print(json.dumps({args.key: entry}, indent=1))


if __name__ == "__main__":
    main()
