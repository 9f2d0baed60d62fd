"""Summarise an `ncu --page source --csv --print-source sass` dump: top instructions by stall samples."""
import csv
import sys


def main(path, top=25):
    lines = open(path).read().splitlines()
    rows = list(csv.reader(lines[1:]))
    h = rows[0]
    iS, iA, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Address"), h.index("Source")
    data = []
    for r in rows[1:]:
        try:
            data.append((float(r[iS] or 0), r[iA], r[iSrc]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    print(f"total samples {tot:.0f}")
    for s, a, src in sorted(data, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}%  {a}  {src[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
