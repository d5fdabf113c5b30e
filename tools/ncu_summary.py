"""Summarise an ncu report (--page raw) into a per-kernel table / JSON.

usage: python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "us": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_hit": "l1tex__t_sector_hit_rate.pct",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "warps_act": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "lsb_stall": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
}


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m in hdr:
                v = r[hdr.index(m)]
                u = units[hdr.index(m)]
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    x = None
                if x is not None and k == "us":
                    x = x / 1000.0 if u in ("nsecond", "ns") else (x * 1000 if u in ("msecond", "ms") else x)
                if x is not None and k.endswith("_MB"):
                    x = x / 1e6 if u in ("byte", "B") else (x / 1e3 if u in ("Kbyte", "KB") else
                                                            (x * 1e3 if u in ("Gbyte", "GB") else x))
                d[k] = x
        res.append(d)
    return res


def main():
    rep = load(sys.argv[1])
    cols = ["us", "dram_rd_MB", "dram_wr_MB", "dram_pct", "lts_pct", "l1_pct", "l1_hit",
            "l2_hit", "warps_act", "regs", "grid", "lsb_stall"]
    print("%-58s " % "kernel" + " ".join("%9s" % c for c in cols))
    for d in rep:
        print("%-58s " % d["kernel"][:58] + " ".join(
            "%9.1f" % d[c] if isinstance(d.get(c), float) else "%9s" % d.get(c) for c in cols))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(rep, fh, indent=1)


if __name__ == "__main__":
    main()
