"""Hottest SASS instructions (by executed count and by stall samples) of an
`ncu --page source --csv --print-source sass` export.

    python tools/ncu_sass_hot.py gpurun_out/x_sass.csv [N]
"""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    ai, si, ei, wi = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[hi + 1:]:
        if len(r) <= max(ei, wi):
            continue
        try:
            data.append((r[ai], r[si], float(r[ei] or 0), float(r[wi] or 0)))
        except ValueError:
            pass
    tot_e = sum(d[2] for d in data) or 1
    tot_w = sum(d[3] for d in data) or 1
    print(f"# {len(data)} instructions, {tot_e:.3g} executed, {tot_w:.0f} stall samples")
    print("-- by stall samples")
    for d in sorted(data, key=lambda d: -d[3])[:top]:
        print(f"{100 * d[3] / tot_w:5.1f}% {100 * d[2] / tot_e:5.1f}%  {d[0]}  {d[1][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
