"""Summarise an ncu --set full report (raw page CSV) into the numbers the
roofline needs: per kernel duration, DRAM bytes, DRAM %, issue/pipe
utilisation, occupancy, main stall.  Usage:
    ncu -i prof.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv
"""
import csv
import json
import sys

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_B": "dram__bytes_read.sum",
    "dram_write_B": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "inst_executed": "smsp__inst_executed.sum",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "stall_long_sb": "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for d in data:
        rec = {"kernel": d[hdr.index("Kernel Name")][:80]}
        for k, m in METRICS.items():
            if m in hdr:
                v = d[hdr.index(m)].replace(",", "")
                u = units[hdr.index(m)]
                try:
                    f = float(v)
                    if u == "Kbyte": f *= 1e3
                    if u == "Mbyte": f *= 1e6
                    if u == "Gbyte": f *= 1e9
                    if u in ("msecond", "ms"): f *= 1e3
                    if u in ("second", "s"): f *= 1e6
                    if u in ("nsecond", "ns"): f *= 1e-3
                    rec[k] = f
                except ValueError:
                    rec[k] = v
        out.append(rec)
    for r in out:
        print(json.dumps(r))
    stalls = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled")]
    return out


if __name__ == "__main__":
    main(sys.argv[1])
