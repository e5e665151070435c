"""Summarise an ncu --set full report (run here, on the CPU box):
    python profiles/summarize_ncu.py gpurun_out/x.ncu-rep "<title>" > profiles/<name>.txt
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    r"gpu__time_duration.sum$", r"dram__bytes_read.sum$", r"dram__bytes_write.sum$",
    r"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed$",
    r"lts__t_sector_hit_rate.pct$", r"lts__t_sectors_srcunit_tex_op_(read|red|write|atom).sum$",
    r"l1tex__t_sectors_pipe_lsu_mem_global_op_(ld|red|st).sum$",
    r"sm__warps_active.avg.pct_of_peak_sustained_active$", r"launch__registers_per_thread$",
    r"launch__grid_size$", r"launch__block_size$", r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active$",
    r"sm__pipe_tensor_cycles_active.*avg.pct_of_peak_sustained_active$",
    r"sm__inst_executed.avg.per_cycle_active$", r"sass__inst_executed_local_(loads|stores)$",
    r"smsp__pcsamp_warps_issue_stalled_[a-z_]+(?<!_not_issued)$",
]


def main(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    names, units = rows[0], rows[1]
    print(title)
    for r in rows[2:]:
        kname = r[names.index("Kernel Name")] if "Kernel Name" in names else "?"
        print(f"--- {kname[:100]}")
        for n, u, v in zip(names, units, r):
            if any(re.search(k, n) for k in KEYS) and v not in ("", "0", "0.00"):
                print(f"  {n:75s} {u:10s} {v}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
