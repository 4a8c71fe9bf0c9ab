"""Summarise an ncu --set full report: per kernel, SOL / issue / stall mix /
instruction mix / DRAM bytes.  Usage: python scripts/ncu_summary.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    keys = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.per_cycle_active", "smsp__thread_inst_executed_per_inst_executed.ratio"]
    for row in raw[2:]:
        print("-" * 100)
        for k in keys:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:70s} {row[i]} {units[i]}")
        st = [(h, row[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("_not_issued")]
        st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for h, v in st
              if v.replace(".", "", 1).isdigit()]
        tot = sum(v for _, v in st) or 1
        print("  stalls:", ", ".join(f"{h} {v / tot * 100:.1f}%" for h, v in sorted(st, key=lambda x: -x[1])[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
