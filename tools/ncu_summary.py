"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel name.

    python tools/ncu_summary.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per, names = collections.defaultdict(dict), {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
             "second": 1}
    for r in data:
        per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        names[r[idi]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i].split("(")[0][:80]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {len(per)} launches, {tot * 1e3:.3f} ms total (serialised, cold-cache ncu timing)")
    print(f"{'ms':>10} {'share':>6} {'n':>4} {'DRAM GB':>8} {'GB/s':>7}  kernel")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{a[1] * 1e3:10.3f} {100 * a[1] / tot:5.1f}% {a[0]:4d} {a[2] / 1e9:8.3f} {a[2] / max(a[1], 1e-12) / 1e9:7.0f}  {n}")


if __name__ == "__main__":
    main(sys.argv[1])
