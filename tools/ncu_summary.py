#!/usr/bin/env python3
"""Summarise `ncu --page raw --csv` exports into profiles/ncu_summary.json.

usage: tools/ncu_summary.py <key>=<raw.csv>[#<kernel row>][:<note>] ...
"""
import csv
import json
import os
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed": "fp64_pipe_pct_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
    "sass__inst_executed_local_loads": "local_loads",
    "Kernel Name": "kernel",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed": "fmaheavy_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct_active",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed":
        "int8_tensor_ops_pct_of_peak",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.per_second": "int8_tensor_ops_per_s",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6,
        "ns": 1e-9, "s": 1.0}


def parse(path, row=0):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2 + row]
    out = {}
    for i, h in enumerate(hdr):
        if h in KEYS:
            v = vals[i]
            try:
                x = float(v.replace(",", ""))
                x *= UNIT.get(units[i], 1.0)
                out[KEYS[h]] = x
            except ValueError:
                out[KEYS[h]] = v
    if "dram_read" in out and "dram_write" in out:
        out["dram_bytes_per_launch"] = out["dram_read"] + out["dram_write"]
    return out


def main():
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "profiles", "ncu_summary.json")
    summary = json.load(open(dst)) if os.path.exists(dst) else {}
    for arg in sys.argv[1:]:
        prec, _, rest = arg.partition("=")
        path, _, note = rest.partition(":")
        path, _, row = path.partition("#")
        d = parse(path, int(row) if row else 0)
        d["source"] = os.path.basename(path)
        d["note"] = note
        summary[prec] = d
    json.dump(summary, open(dst, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
