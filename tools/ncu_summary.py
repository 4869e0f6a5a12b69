"""Summarise an .ncu-rep (raw page): key throughput / stall metrics per profiled kernel."""
import csv
import io
import re
import subprocess
import sys

KEYS = [r"^gpu__time_duration.sum$", r"^dram__bytes_read.sum$", r"^dram__bytes_write.sum$",
        r"^sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active$", r"^sm__warps_active.avg.pct_of_peak_sustained_active$",
        r"^l1tex__throughput.avg.pct_of_peak_sustained_active$", r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum$", r"^l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum$",
        r"^l1tex__t_sector_hit_rate.pct$", r"^lts__t_sector_hit_rate.pct$", r"^l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed$",
        r"^l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$", r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$",
        r"^smsp__issue_active.avg.pct_of_peak_sustained_active$", r"^smsp__inst_executed.sum$", r"^launch__registers_per_thread$",
        r"^dram__throughput.avg.pct_of_peak_sustained_elapsed$", r"^l1tex__m_xbar2l1tex_read_bytes.sum$",
        r"^smsp__average_warps_issue_stalled_(long_scoreboard|short_scoreboard|wait|barrier|mio_throttle|lg_throttle|math_pipe_throttle|no_instruction|not_selected|branch_resolving|dispatch_stall|sleeping|tex_throttle)_per_issue_active.ratio$"]

def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    pats = [re.compile(k) for k in KEYS]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"== {name[:90]}")
        for i, h in enumerate(hdr):
            if any(p.search(h) for p in pats):
                print(f"   {h} = {r[i]} {units[i]}")

if __name__ == "__main__":
    main(sys.argv[1])
