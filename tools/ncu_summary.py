"""Summarise one `ncu --set full` report (first kernel) into the metrics the roofline cites.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [flops_per_launch] > profiles/ncu_....txt
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
]


def main():
    rep = sys.argv[1]
    flops = float(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {rep}")
    for vals in rows[2:]:
        rec = dict(zip(hdr, vals))
        unit = dict(zip(hdr, units))
        print(f"\n## {rec.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in rec:
                print(f"{k:90s} {rec[k]:>18s} {unit.get(k, '')}")
        try:
            dur_ms = float(rec["gpu__time_duration.sum"])
            if unit.get("gpu__time_duration.sum") == "us":
                dur_ms /= 1e3
            rd = float(rec["dram__bytes_read.sum"]) * (1e6 if unit["dram__bytes_read.sum"] == "Mbyte" else 1)
            wr = float(rec["dram__bytes_write.sum"]) * (1e6 if unit["dram__bytes_write.sum"] == "Mbyte" else 1)
            print(f"{'derived: dram bytes per launch':90s} {rd + wr:18.4g} byte")
            print(f"{'derived: dram GB/s':90s} {(rd + wr) / dur_ms / 1e6:18.1f} GB/s")
            if flops:
                print(f"{'derived: algorithmic TFLOP/s (given flops / ncu duration)':90s} "
                      f"{flops / dur_ms / 1e9:18.1f} TFLOP/s")
        except (KeyError, ValueError):
            pass


if __name__ == "__main__":
    main()
