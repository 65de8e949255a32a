"""Concise text summary of an ncu --set full report (one line per key metric, per kernel launch).

    python tools/rep_summary.py gpurun_out/x.ncu-rep [label] >> profiles/rNN_ncu_full.txt
"""
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
       "launch__grid_size", "launch__block_size"]


def main(path, label=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(f"# {path}: no data")
        return
    h, u = rows[0], rows[1]
    print(f"## {label or path}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name[:140]}")
        for k in RAW:
            if k in h:
                i = h.index(k)
                print(f"  {k:60s} {r[i]:>18s} {u[i]}")
        try:
            t = float(r[h.index("gpu__time_duration.sum")])
            tu = u[h.index("gpu__time_duration.sum")]
            scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(tu, 1e-9)
            rb = float(r[h.index("dram__bytes_read.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[h.index("dram__bytes_read.sum")]]
            wb = float(r[h.index("dram__bytes_write.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[h.index("dram__bytes_write.sum")]]
            print(f"  => DRAM traffic {(rb + wb) / 1e9:.3f} GB in {t * scale * 1e3:.3f} ms = {(rb + wb) / (t * scale) / 1e9:.0f} GB/s")
        except (ValueError, KeyError, IndexError):
            pass


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
