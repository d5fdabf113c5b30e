"""Per-kernel-class summaries of ncu captures, in the classes of
p2g_profile_iteration (bench.py's roofline).

  full <report.ncu-rep> [--json out]   one --set full capture of
        `python tools/ncu_iter.py c2 2` (a 3-iteration solve first: profile_iteration
        needs the Krylov state): the launches from the last
        k_alpha to the end are one Kp-recurrence PCG iteration; prints the
        per-kernel table and writes per_iteration_dram_bytes per class.
  launches <launches.csv> [--json out]  a --metrics gpu__time_duration.sum
        launch list of bench.py: per-class launch count, time and share.
"""
import csv
import json
import re
import sys

sys.path.insert(0, "tools")
from ncu_summary import load  # noqa: E402

CLASSES = [
    ("spmv_dot", r"^(void )?(p2g::)?k_(spmv|kp_update\w*)\b"),
    ("update_presmooth", r"^(void )?(p2g::)?k_(update_pre|update_rows|jacobi)\b"),
    ("gs_forward", r"^(void )?(p2g::)?k_gs_forward\w*\b"),
    ("residual", r"^(void )?(p2g::)?k_residual\w*\b"),
    ("restrict", r"^(void )?(p2g::)?k_restrict_(vec|tiled|reg2?|mma|ws)\b"),
    ("coarse_solve", r"^(void )?(p2g::)?k_coarse\b"),
    ("prolong", r"^(void )?(p2g::)?k_prolong(_tiled|_reg|_mma|_ws)?\b"),
    ("gs_backward", r"^(void )?(p2g::)?k_gs_backward\w*\b"),
    ("scalar_reduce", r"^(void )?(p2g::)?k_(alpha|finalize|set_cond|reduce_rows|sum_parts)\b"),
    ("p_update", r"^(void )?(p2g::)?k_pupdate\b"),
]


def kclass(name):
    for c, rx in CLASSES:
        if re.search(rx, name):
            return c
    return "other"


def load_any(path):
    """an .ncu-rep (through ncu -i) or its `--page raw --csv` export (.csv[.gz])"""
    if path.endswith(".csv.gz") or path.endswith(".csv"):
        import gzip
        import io
        import subprocess
        import ncu_summary as NS
        opener = gzip.open if path.endswith(".gz") else open
        with opener(path, "rt") as fh:
            text = fh.read()
        real = subprocess.run
        NS.subprocess.run = lambda *a, **k: type("R", (), {"stdout": text})()
        try:
            return NS.load(path)
        finally:
            NS.subprocess.run = real
    return load(path)


def full(path, out):
    rep = load_any(path)
    last = max(i for i, d in enumerate(rep) if re.search(r"^(void )?(p2g::)?k_alpha\b", d["kernel"]))
    it = rep[last:]
    agg = {}
    print("%-60s %9s %9s %9s %7s %6s %5s" % ("kernel (one iteration)", "us", "dram_MB", "GB/s",
                                              "dram%", "warps%", "regs"))
    for d in it:
        c = kclass(d["kernel"])
        by = ((d.get("dram_rd_MB") or 0) + (d.get("dram_wr_MB") or 0)) * 1e6
        us = d.get("us") or 0.0
        a = agg.setdefault(c, {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["us"] += us
        a["dram_bytes"] += by
        print("%-60s %9.1f %9.1f %9.0f %7.1f %6.1f %5.0f" % (
            d["kernel"][:60], us, by / 1e6, by / (us * 1e-6) / 1e9 if us else 0,
            d.get("dram_pct") or 0, d.get("warps_act") or 0, d.get("regs") or 0))
    tot = sum(a["us"] for a in agg.values())
    print("\nclass               launches        us    share   dram_MB    GB/s")
    for c, a in agg.items():
        print("%-18s %9d %9.1f %7.1f%% %9.1f %7.0f" % (
            c, a["launches"], a["us"], 100 * a["us"] / tot, a["dram_bytes"] / 1e6,
            a["dram_bytes"] / (a["us"] * 1e-6) / 1e9 if a["us"] else 0))
    res = {"source": path, "capture": "ncu --set full --clock-control none --cache-control all, "
                                      "one PCG iteration (last k_alpha .. end) of the eager profile "
                                      "(tools/ncu_iter.py / ncu_b1.py, NVTX range 'profile')",
           "per_iteration_dram_bytes": {c: a["dram_bytes"] for c, a in agg.items()},
           "per_iteration_us": {c: a["us"] for c, a in agg.items()},
           "launches_per_iteration": {c: a["launches"] for c, a in agg.items()},
           "kernels": it}
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)
    if "--traffic" in sys.argv:  # merge into profiles/ncu_traffic.json under this config
        cfg = sys.argv[sys.argv.index("--traffic") + 1]
        tp = "profiles/ncu_traffic.json"
        try:
            with open(tp) as fh:
                allt = json.load(fh)
        except Exception:
            allt = {}
        allt[cfg] = {"source": path, "capture": res["capture"],
                     "per_iteration_dram_bytes": res["per_iteration_dram_bytes"],
                     "per_iteration_us": res["per_iteration_us"],
                     "launches_per_iteration": res["launches_per_iteration"]}
        with open(tp, "w") as fh:
            json.dump(allt, fh, indent=1, sort_keys=True)


def launches(path, out):
    rows = []
    import gzip
    with (gzip.open(path, "rt") if path.endswith(".gz") else open(path)) as fh:
        lines = [ln for ln in fh if not ln.startswith("==")]
    rd = list(csv.reader(lines))
    hdr = rd[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    for r in rd[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        us = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        rows.append((r[ki], us))
    agg = {}
    for k, us in rows:
        c = kclass(k)
        a = agg.setdefault(c, [0, 0.0])
        a[0] += 1
        a[1] += us
    solve = {c: a for c, a in agg.items() if c != "other"}
    tot = sum(a[1] for a in solve.values())
    print(f"{len(rows)} launches; solve-loop classes:")
    print("class               launches        us    share")
    for c, a in sorted(solve.items(), key=lambda x: -x[1][1]):
        print("%-18s %9d %9.0f %7.1f%%" % (c, a[0], a[1], 100 * a[1] / tot))
    if "other" in agg:
        print("%-18s %9d %9.0f   (setup / generation / bench helpers)" % ("other", *agg["other"]))
    if out:
        with open(out, "w") as fh:
            json.dump({"source": path, "launches": len(rows),
                       "classes": {c: {"launches": a[0], "us": a[1],
                                       "share_of_solve": a[1] / tot if c != "other" else None}
                                   for c, a in agg.items()}}, fh, indent=1)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    out = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    {"full": full, "launches": launches}[mode](path, out)
