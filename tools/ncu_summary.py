#!/usr/bin/env python3
"""Summarise ncu reports (--page raw) into JSON: per kernel launch the
duration, instruction count, pipe/issue utilisation, occupancy, DRAM bytes,
stall shares.  usage: ncu_summary.py NAME=REPORT [...] > out.json"""
import csv
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "smsp__sass_inst_executed_op_local_ld.sum",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
out = {}
for arg in sys.argv[1:]:
    name, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    for k, v in enumerate(rows[2:]):
        kern = v[hdr.index("Kernel Name")]
        m = {w: f"{v[hdr.index(w)]} {units[hdr.index(w)]}".strip() for w in WANT if w in hdr}
        st = [(float(v[i].replace(",", "")), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
              for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
              and "not_issued" not in hdr[i] and v[i].replace(",", "").replace(".", "").isdigit()]
        tot = sum(x[0] for x in st) or 1.0
        out[f"{name}#{k}"] = {"kernel": kern[:120], "metrics": m,
                              "stall_share_pct": {n: round(100 * x / tot, 1) for x, n in sorted(st, reverse=True)[:9]}}
json.dump(out, sys.stdout, indent=1)
