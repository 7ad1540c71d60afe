#!/usr/bin/env python
"""Summarise one `ncu --set full` capture of a kernel launch into profiles/ncu_summary.json,
keyed by kernel and workload config (merged into the existing file).

    python profiles/summarize_ncu.py REP.ncu-rep --key C5 --decisions D [--kernel k_construct]
                                     [--bytes-per-decision B] [--config TEXT] [--capture TEXT]

`bench.py` reads `[kernel][config].dram_bytes_per_launch` as the roofline `traffic` figure
of the config it runs, and prints null for a config without a capture (ncu replays the
kernel, so the capture itself is never a timing source).
"""
import argparse
import csv
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = {
    "gpu__time_duration.sum": "gpu_time",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "smsp__average_warp_latency_per_inst_issued.ratio": "warp_latency_per_inst_cycles",
    "smsp__inst_executed.sum": "inst_executed",
    "lts__t_sectors.sum": "l2_sectors",
}
SCALE = {"": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", help="REP.ncu-rep, or its `--page raw --csv` export (.csv)")
    ap.add_argument("--decisions", type=float, required=True, help="decisions in the captured launch")
    ap.add_argument("--bytes-per-decision", type=float, default=260.0)
    ap.add_argument("--config", default="C5 timed iteration of bench.py (4th k_construct launch)")
    ap.add_argument("--capture", default="ncu --set full --import-source on --clock-control none -k regex:k_construct -s 3 -c 1")
    ap.add_argument("--out", default=os.path.join(HERE, "ncu_summary.json"))
    ap.add_argument("--key", required=True, help="workload config the capture belongs to (C1..C5)")
    ap.add_argument("--kernel", default="k_construct")
    ap.add_argument("--row", type=int, default=0, help="launch row of the report to summarise")
    args = ap.parse_args()
    if args.rep.endswith(".csv"):  # `ncu -i REP --page raw --csv` output saved on the GPU box
        raw = open(args.rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2 + args.row]
    s = {"config": args.config, "capture": args.capture}
    stalls = {}
    for i, h in enumerate(hdr):
        if h in METRICS:
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if METRICS[h] == "gpu_time":
                s["gpu_time_ms"] = v * SCALE.get(u, 1.0)
            elif METRICS[h].startswith("dram_bytes"):
                s[METRICS[h]] = v * SCALE.get(u, 1.0)
            else:
                s[METRICS[h]] = v
        elif h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            v = float(vals[i].replace(",", "") or 0)
            if v:
                stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = v
    s["dram_bytes_per_launch"] = s.get("dram_bytes_read", 0.0) + s.get("dram_bytes_write", 0.0)
    s["decisions_per_launch"] = args.decisions
    s["algorithmic_bytes_per_launch"] = args.decisions * args.bytes_per_decision
    if "l2_sectors" in s:
        s["l2_bytes_per_launch"] = 32.0 * s["l2_sectors"]
    s["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    db = {}
    if os.path.exists(args.out):
        db = json.load(open(args.out))
    db.setdefault(args.kernel, {})[args.key] = s
    json.dump(db, open(args.out, "w"), indent=1, sort_keys=True)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
