import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
def col(name):
    if name in hdr: return hdr.index(name)
    for i, h in enumerate(hdr):
        if h.endswith("." + name): return i
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__sass_average_branch_targets_threads_uniform.pct", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct"]
stalls = ["wait", "long_scoreboard", "short_scoreboard", "not_selected", "math_pipe_throttle", "branch_resolving", "no_instruction", "lg_throttle", "mio_throttle", "barrier", "dispatch_stall"]
for r in rows[2:]:
    if len(r) != len(hdr): continue
    print("==", r[hdr.index("Kernel Name")][:60])
    for w in want:
        i = col(w)
        if i is not None: print(f"  {w} {units[i]} {r[i]}")
    print("  stalls:", {s: r[col(f'smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio')] for s in stalls})
