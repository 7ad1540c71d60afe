#!/usr/bin/env python
"""One line per captured launch of an `ncu --set full` report: duration, DRAM and L2
throughput, hit rates, occupancy and the top warp-stall reasons.

    python profiles/summarize_kernels.py REP.ncu-rep [> profiles/rNN_kernels.md]
"""
import csv
import subprocess
import sys

COLS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_sectors.sum": "l2_sectors",
    "l1tex__t_sector_hit_rate.pct": "l1_hit",
    "lts__t_sector_hit_rate.pct": "l2_hit",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "": 1.0, "%": 1.0}


def main() -> None:
    if sys.argv[1].endswith(".csv"):  # a `--page raw --csv` export saved on the GPU box
        raw = open(sys.argv[1]).read()
    else:
        raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ik = hdr.index("Kernel Name")
    print("| kernel | ms | DRAM GB | DRAM GB/s | DRAM % peak | L2 GB | L1 hit | L2 hit | occupancy | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in data:
        v = {}
        for i, h in enumerate(hdr):
            if h in COLS:
                try:
                    v[COLS[h]] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), h.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1.0
        top = ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:3])
        dram = (v.get("dram_rd", 0) + v.get("dram_wr", 0)) / 1e9
        ms = v.get("time", 0.0)
        name = r[ik].split("(")[0].replace("pacob200::", "")
        print(f"| `{name}` | {ms:.3f} | {dram:.3f} | {dram / (ms / 1e3) if ms else 0:.0f} | {v.get('dram_pct', 0):.1f} | "
              f"{v.get('l2_sectors', 0) * 32 / 1e9:.3f} | {v.get('l1_hit', 0):.0f}% | {v.get('l2_hit', 0):.0f}% | "
              f"{v.get('occupancy', 0):.1f}% | {top} |")


if __name__ == "__main__":
    main()
