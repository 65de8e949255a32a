"""Print the key lines of an `ncu --page details --csv` export (one kernel).

    python tools/ncu_details.py gpurun_out/x_details.csv
"""
import csv
import sys

KEEP = ("Duration", "Memory Throughput", "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Block Limit", "Executed Ipc Active", "Issue Slots Busy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Warp Cycles Per Issued Instruction", "No Eligible", "One or More Eligible", "Executed Instructions",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy", "Waves Per SM")


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hi]
    ki, si, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    print(rows[hi + 1][ki][:120])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        if any(r[mi].startswith(k) for k in KEEP):
            print(f"  {r[si][:28]:28s} {r[mi][:44]:44s} {r[vi]:>14s} {r[ui]}")
    # rule messages (bottleneck hints)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "" and r[vi]:
            pass


if __name__ == "__main__":
    main(sys.argv[1])
