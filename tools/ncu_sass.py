"""Hot SASS instructions and the stall-reason breakdown of one kernel in an
ncu report (captured with --import-source on, --set full).

usage: python tools/ncu_sass.py report.ncu-rep <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, rx = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{rx}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    # the source page can list a kernel's SASS more than once (one block per
    # source view); keep each instruction address once
    data, seen = [], set()
    for r in rows[2:]:
        if len(r) == len(hdr) and r[0] not in seen:
            seen.add(r[0])
            data.append(r)

    def num(r, c):
        try:
            return float(r[hdr.index(c)] or 0)
        except ValueError:
            return 0.0

    si = "Warp Stall Sampling (All Samples)"
    tot = sum(num(r, si) for r in data)
    print(f"{rows[0][1][:100]}\n{len(data)} SASS instructions, {tot:.0f} stall samples")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {h: sum(num(r, h) for r in data) for h in reasons}
    print("stall reasons: " + ", ".join(f"{h[6:]} {100 * v / tot:.0f}%"
                                        for h, v in sorted(agg.items(), key=lambda x: -x[1])
                                        if v / max(tot, 1) >= 0.02))
    print(f"{'samples':>8} {'executed':>9}  top reasons / instruction")
    for r in sorted(data, key=lambda r: -num(r, si))[:top]:
        rs = sorted(((num(r, h), h[6:]) for h in reasons), reverse=True)[:2]
        why = " ".join(f"{n}:{v:.0f}" for v, n in rs if v > 0)
        print(f"{num(r, si):8.0f} {num(r, 'Instructions Executed'):9.0f}  {r[1].strip()[:60]:60s} {why}")


if __name__ == "__main__":
    main()
