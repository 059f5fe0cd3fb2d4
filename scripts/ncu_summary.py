#!/usr/bin/env python
"""Summarise ncu reports (run here, no GPU needed): key throughput, memory and
stall metrics per kernel, for profiles/*.md.

    python scripts/ncu_summary.py gpurun_out/prof_r1_*.ncu-rep > profiles/r1_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__inst_executed.sum", "warp instr executed"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({h: (v, u) for h, v, u in zip(hdr, r, units)})
    return res


def main(paths):
    for p in paths:
        for rec in raw(p):
            name = rec.get("Kernel Name", ("?", ""))[0].split("(")[0]
            print(f"### {name}  ({p.split('/')[-1]})\n")
            print("| metric | value |\n|---|---|")
            for k, label in KEYS:
                if k in rec:
                    v, u = rec[k]
                    print(f"| {label} | {v} {u} |")
            st = []
            for k, (v, u) in rec.items():
                if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(v.replace(",", "")), k[len(STALLS):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            if st:
                print("| top stalls (cycles/instr) | " +
                      ", ".join(f"{n} {v:.2f}" for v, n in st[:5]) + " |")
            print()


if __name__ == "__main__":
    main(sys.argv[1:])
