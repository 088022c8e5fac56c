"""Extract the key metrics of every kernel in an ncu report into the tracked CSV format of profiles/.

    python scripts/ncu_keymetrics.py gpurun_out/prof_cluster_r1h.ncu-rep > profiles/r1/ncu_..._keymetrics.csv

Reads ``ncu -i REPORT --page raw --csv`` (row 0 = metric names, row 1 = units, rows 2.. = kernels).
"""
from __future__ import annotations

import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__cluster_dim_x",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
]


def main() -> int:
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    names, units = rows[0], rows[1]
    out = csv.writer(sys.stdout, lineterminator="\n")
    out.writerow(["kernel", "metric", "value", "unit"])
    for r in rows[2:]:
        kern = r[names.index("Kernel Name")]
        for k in KEYS:
            if k in names:
                i = names.index(k)
                out.writerow([kern, k, r[i], units[i]])
    return 0


if __name__ == "__main__":
    sys.exit(main())
