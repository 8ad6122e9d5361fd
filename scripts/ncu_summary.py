"""Print selected metrics of an `ncu --page raw --csv` export (one row per
captured kernel): python scripts/ncu_summary.py file.csv [metric-regex ...]"""
import csv
import re
import sys

DEFAULT = [r"^gpu__time_duration.sum$", r"^dram__bytes_(read|write)\.sum$", r"^lts__t_bytes\.sum$",
           r"^lts__t_sectors_srcunit_tex_op_(read|write)\.sum$",
           r"^dram__throughput.avg.pct_of_peak_sustained_elapsed$",
           r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$",
           r"^sm__inst_executed\.sum$", r"^sm__instruction_throughput.avg.pct_of_peak_sustained_active$",
           r"^smsp__issue_active.avg.pct_of_peak_sustained_active$",
           r"^sm__inst_executed_pipe_(alu|fma|fmaheavy|xu|lsu|uniform|adu|cbu)\.avg\.pct_of_peak_sustained_active$",
           r"^sm__pipe_(alu|fma|fmaheavy|shared|xu)_cycles_active\.avg\.pct_of_peak_sustained_active$",
           r"^sm__warps_active.avg.pct_of_peak_sustained_active$", r"^launch__registers_per_thread$",
           r"^launch__grid_size$", r"^launch__block_size$", r"^sm__cycles_elapsed.avg.per_second$",
           r"^smsp__average_warp_latency_issue_stalled_.*ratio$"]


def main():
    path = sys.argv[1]
    pats = [re.compile(p) for p in (sys.argv[2:] or DEFAULT)]
    with open(path) as f:
        rows = list(csv.reader(f))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    names, units = rows[hdr], rows[hdr + 1]
    for r in rows[hdr + 2:]:
        if len(r) != len(names):
            continue
        print("kernel:", r[names.index("Kernel Name")][:110])
        for i, n in enumerate(names):
            if any(p.search(n) for p in pats):
                print(f"  {n} = {r[i]} {units[i]}")


if __name__ == "__main__":
    main()
