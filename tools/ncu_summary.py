"""Key metrics of an ncu report (first kernel) as text; used for profiles/*.md.
Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
    "sm__warps_active.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
]
STALLS = ["wait", "barrier", "not_selected", "selected", "short_scoreboard", "long_scoreboard", "branch_resolving",
          "no_instructions", "dispatch_stall", "math_pipe_throttle", "mio_throttle", "lg_throttle", "membar"]

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units, vals = rows[0], rows[1], rows[2]
ix = {h: i for i, h in enumerate(hdr)}
print(f"kernel: {vals[ix['Kernel Name']]}")
for w in WANT:
    if w in ix:
        print(f"{w:62s} {vals[ix[w]]:>16s} {units[ix[w]]}")
tot = 0
st = {}
for s in STALLS:
    k = f"smsp__pcsamp_warps_issue_stalled_{s}"
    if k in ix:
        v = float(vals[ix[k]].replace(",", "") or 0)
        st[s] = v
        tot += v
print("warp-state samples (share):", ", ".join(f"{k} {100 * v / max(tot, 1):.1f}%" for k, v in
                                               sorted(st.items(), key=lambda kv: -kv[1])))
