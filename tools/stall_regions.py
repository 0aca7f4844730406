"""Warp-stall samples of an `ncu --page source --csv --print-source sass` dump, split into the
regions between barrier waits (profiling aid).  Prints each region's share of all samples, its
top stall reasons and the barrier offset that opens it.

  python tools/stall_regions.py /tmp/fwd_src.csv
"""
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = []
    for r in rows[2:]:  # first kernel section only
        if len(r) < 3 or r[0] in ("Address", "Kernel Name"):
            break
        data.append(r)
    si = h.index("Warp Stall Sampling (All Samples)")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ri = [h.index(c) for c in reasons]
    tot = sum(float(r[si] or 0) for r in data)
    regions, cur = [], {"start": 0, "label": "entry", "samples": 0.0, "why": [0.0] * len(ri), "n": 0}
    for i, r in enumerate(data):
        src = r[1]
        if "TRYWAIT" in src:
            regions.append(cur)
            m = re.search(r"\+(0x[0-9a-f]+)\]", src)
            cur = {"start": i, "label": m.group(1) if m else src.strip()[:40], "samples": 0.0, "why": [0.0] * len(ri), "n": 0}
        cur["samples"] += float(r[si] or 0)
        cur["n"] += 1
        for k, j in enumerate(ri):
            cur["why"][k] += float(r[j] or 0)
    regions.append(cur)
    for g in regions:
        if g["samples"] / tot < 0.01:
            continue
        top = sorted(zip(g["why"], reasons), reverse=True)[:4]
        print(f"{100 * g['samples'] / tot:5.1f}%  lines {g['start']:5d}+{g['n']:<5d} after wait {g['label']:>10}  " +
              "  ".join(f"{n[6:]} {100 * v / tot:.1f}" for v, n in top))


if __name__ == "__main__":
    main(sys.argv[1])
