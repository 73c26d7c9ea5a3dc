#!/usr/bin/env python
"""Summarise an ncu report (--set full) of the scoring kernel into a small JSON: duration,
DRAM/L2/smem traffic, bank conflicts, FP64 pipe, occupancy, stall reasons, instruction mix.

    python tools/ncu_summary.py gpurun_out/prof_c3.ncu-rep > profiles/r01/ncu_c3_vX.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "lts_bytes": ("lts__t_bytes.sum", 1.0),
    "l1_hit_rate_pct": ("l1tex__t_sector_hit_rate.pct", 1.0),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "global_ld_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 1.0),
    "l1tex_data_pipe_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", 1.0),
    "smem_ld_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 1.0),
    "smem_wavefronts_all_ops": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "l1tex_data_pipe_wavefronts_per_sm": ("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg", 1.0),
    "smem_ld_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1.0),
    "smem_wavefront_pct_of_peak": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pipe_pct_active": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "lsu_pipe_pct_active": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "global_ld_inst": ("smsp__sass_inst_executed_op_global_ld.sum", 1.0),
    "shared_ld_inst": ("smsp__sass_inst_executed_op_shared_ld.sum", 1.0),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "sm_clock_hz": ("sm__cycles_elapsed.avg.per_second", 1.0),
}
STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "wait", "mio_throttle",
          "math_pipe_throttle", "not_selected", "selected", "branch_resolving", "lg_throttle",
          "dispatch_stall", "no_instruction"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name"), "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for k, (m, scale) in KEYS.items():
            v = d.get(m)
            if v in (None, "", "n/a"):
                continue
            v = float(v.replace(",", ""))
            unit = u.get(m, "")
            if k.endswith("_bytes") or k == "lts_bytes":
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                v *= mult
            elif k == "duration_ms":
                mult = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1e-6)
                v *= mult
            elif k == "sm_clock_hz":
                v *= {"Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(unit, 1)
            rec[k] = v
        st = {}
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if d.get(m) not in (None, ""):
                st[s] = float(d[m])
        rec["stalls_per_issue"] = st
        if "dram_read_bytes" in rec:
            rec["dram_bytes_per_launch"] = rec.get("dram_read_bytes", 0) + rec.get("dram_write_bytes", 0)
        out.append(rec)
    json.dump(out if len(out) > 1 else out[0], sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
