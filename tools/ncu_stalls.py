"""Top warp-stall reasons and a few counters from an `ncu --page raw --csv` export.

    python tools/ncu_stalls.py gpurun_out/x_raw.csv
"""
import csv
import sys

EXTRA = ["smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__thread_inst_executed_per_inst_executed.ratio",
         "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
         "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
         "smsp__inst_executed_op_global_red.sum", "smsp__inst_executed_op_global_atom.sum",
         "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_atom.sum"]


def main(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    print(d.get("Kernel Name", ("?",))[0][:100])
    st = [(k, float(x[0].replace(",", ""))) for k, x in d.items()
          if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    for k, x in sorted(st, key=lambda t: -t[1])[:8]:
        print(f"  {100 * x / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    for k in EXTRA:
        if k in d:
            print(f"  {k} = {d[k][0]} {d[k][1]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
