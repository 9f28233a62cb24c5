"""Summarise an ncu report (--set full) into the per-kernel numbers DESIGN.md / profiles/ cite.
  python tools/ncu_summary.py gpurun_out/<tag>/prof.ncu-rep > profiles/<round>_<what>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA-pipe inst %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU-pipe inst %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64-pipe inst %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU/conv) inst %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-inst"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "FADD thread-inst"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "FMUL thread-inst"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-inst"),
    ("smsp__inst_executed.sum", "warp-inst executed"),
]
STALLS = ["math_pipe_throttle", "not_selected", "selected", "wait", "short_scoreboard",
          "long_scoreboard", "barrier", "mio_throttle", "dispatch_stall", "branch_resolving",
          "no_instructions", "lg_throttle", "drain"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        print(f"== [{r[ix['ID']]}] {name[:110]}")
        for k, label in KEYS:
            if k in ix and r[ix[k]] not in ("", None):
                print(f"   {label:28s} {r[ix[k]]} {units[ix[k]]}")
        tot = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in ix and r[ix[k]]:
                try:
                    tot[s] = float(r[ix[k]].replace(",", ""))
                except ValueError:
                    pass
        S = sum(tot.values()) or 1.0
        top = sorted(tot.items(), key=lambda kv: -kv[1])[:6]
        print("   stall samples (share):     " + ", ".join(f"{k} {v / S:.0%}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
