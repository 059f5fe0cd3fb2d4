#!/usr/bin/env python
"""Binding-pipe utilisation of ncu --set full reports (run here, no GPU).

    python scripts/pipe_util.py gpurun_out/prof_TAG_k_*.ncu-rep

Prints, per kernel launch: duration, issue-active %, LSU (L1/shared) data-pipe
wavefronts %, FP64 / ALU / FMA pipe %, DRAM %, the busiest of them and
roof_us = duration x that pipe's utilisation (the launch time if that pipe
ran at 100%), as JSON lines for profiles/pipe_roofline.json.
"""
import csv
import io
import json
import subprocess
import sys

PIPES = {
    "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lsu_wavefronts": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "alu": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "dram": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
}


def records(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def main(paths):
    for p in paths:
        for rec in records(p):
            name = rec.get("Kernel Name", "?").split("(")[0].replace("void ", "").replace("ssb::", "")
            dur = num(rec.get("gpu__time_duration.sum"))
            unit = rec["_units"].get("gpu__time_duration.sum", "us")
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                     "msecond": 1e3}.get(unit, 1.0)
            dur_us = dur * scale if dur else None
            pct = {k: num(rec.get(m)) for k, m in PIPES.items()}
            pct = {k: v for k, v in pct.items() if v is not None}
            bind = max(pct, key=pct.get) if pct else None
            print(json.dumps({
                "kernel": name, "report": p.split("/")[-1], "ncu_us": dur_us,
                "pipes_pct": {k: round(v, 1) for k, v in pct.items()},
                "binding_pipe": bind,
                "roof_us": round(dur_us * pct[bind] / 100.0, 2) if bind and dur_us else None,
            }))


if __name__ == "__main__":
    main(sys.argv[1:])
