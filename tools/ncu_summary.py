#!/usr/bin/env python3
"""Summarise an .ncu-rep (captured with --set full --import-source on) into markdown + a traffic record.

    python tools/ncu_summary.py gpurun_out/X.ncu-rep profiles/X.md [workload queries]
"""
import csv, io, json, os, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else None
queries = int(sys.argv[4]) if len(sys.argv) > 4 else None

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "sass__inst_executed_local_loads",
        "sass__inst_executed_local_stores", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
lines = [f"# ncu summary: `{os.path.basename(rep)}`", "",
         "Captured with `ncu --set full --clock-control none --import-source on` (one launch; times under the profiler are",
         "not benchmark numbers).", "", "| metric | value | unit |", "|---|---|---|"]
for k in KEYS:
    if k in m:
        lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")

def gb(key):
    v, u = m.get(key, ("0", "byte"))
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)

traffic = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
lines += ["", f"DRAM traffic of this launch: {traffic/1e9:.2f} GB (read {gb('dram__bytes_read.sum')/1e9:.2f} + write {gb('dram__bytes_write.sum')/1e9:.2f})"]
if queries:
    lines.append(f"= {traffic/queries/1e6:.1f} MB per query over {queries} queries.")

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
cur, h2, recs = None, None, []
for r in csv.reader(io.StringIO(src)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": h2 = r; continue
    if r[0] == "Function Name": continue
    if h2 and len(r) == len(h2) and r[0] != "": recs.append((cur, r))
if recs:
    ie = h2.index("Instructions Executed"); te = h2.index("Thread Instructions Executed"); ss = h2.index("# Samples")
    tot = sum(float(r[ie] or 0) for _, r in recs); tots = sum(float(r[ss] or 0) for _, r in recs)
    lines += ["", "## Hottest source lines (by stall samples)", "", "| inst % | samples % | lanes/inst | where | source |", "|---|---|---|---|---|"]
    for f, r in sorted(recs, key=lambda x: -float(x[1][ss] or 0))[:25]:
        i = float(r[ie] or 0)
        code = r[1].strip().replace("|", "\\|")[:90]
        lines.append(f"| {100*i/tot:.1f} | {100*float(r[ss])/tots:.1f} | {float(r[te])/max(i,1):.1f} | {f}:{r[0]} | `{code}` |")
open(out, "w").write("\n".join(lines) + "\n")
if workload:
    tj = os.path.join(os.path.dirname(out), "traffic.json")
    d = json.load(open(tj)) if os.path.isfile(tj) else {}
    d[workload] = {"dram_bytes_per_launch": traffic, "queries_per_launch": queries, "source": os.path.basename(out)}
    json.dump(d, open(tj, "w"), indent=1)
print("wrote", out)
