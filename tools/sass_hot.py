"""Top stalled SASS lines and barrier-wait retry counts from an `ncu --page source --csv --print-source sass` dump."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) < 3 or r[0] in ("Address", "Kernel Name"):
            break
        data.append(r)
    return rows[0], h, data


def main(path, thresh=0.004):
    k, h, data = load(path)
    si = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    tot = sum(float(r[si] or 0) for r in data)
    print(k[:2], len(data), "lines")
    for i, r in enumerate(data):
        v = float(r[si] or 0)
        if v / tot > thresh or "SYNCS.PHASECHK" in r[1]:
            print(f"{v / tot * 100:5.2f}% {i:5d} ex={r[ie]:>9} {r[1][:95]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.004)
