"""Condense one ncu --set full capture of the box-entry k_trace launch into the
figures SURVEY.md 8d asks the bench to carry (instructions per ray and per
step, branch efficiency, achieved L2 / DRAM GB/s, shared-memory wavefronts).

usage: ncu_stats.py report.ncu-rep rays steps_sum [workload order [build_id]] > profiles/rNN_ncu_stats.json

With workload/order the entry is keyed to the captured build's
mwt_build_id(), which is how bench.py finds it.
"""
import csv
import io
import json
import subprocess
import sys

rep, rays, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
rows = [r for r in rows[2:] if len(r) == len(hdr) and "k_trace" in r[hdr.index("Kernel Name")]]
r = rows[0]


def col(name):
    """column of a metric (some sections prefix the name, e.g. SM_A.TriageCompute.)"""
    if name in hdr:
        return hdr.index(name)
    for i, h in enumerate(hdr):
        if h.endswith("." + name):
            return i
    return None


def g(name):
    i = col(name)
    if i is None:
        return None
    v = r[i].replace(",", "")
    try:
        return float(v)
    except ValueError:
        return None


dur_s = g("gpu__time_duration.sum") * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
                                       "msecond": 1e-3}.get(units[hdr.index("gpu__time_duration.sum")], 1e-9)
inst = g("smsp__inst_executed.sum")
lts = (g("lts__t_sectors.sum") or 0) * 32
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def gb(name):  # a byte count in bytes, whatever unit ncu printed
    return g(name) * SCALE.get(units[hdr.index(name)], 1)


dram = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
nsm = g("device__attribute_multiprocessor_count") or 148
wf = g("l1tex__data_pipe_lsu_wavefronts.sum") or (g("l1tex__data_pipe_lsu_wavefronts.avg") or 0) * nsm
out = {
    "report": rep.split("/")[-1],
    "kernel": r[hdr.index("Kernel Name")][:80],
    "duration_ms": dur_s * 1e3,
    "rays": rays,
    "triangle_steps": steps,
    "warp_instructions": inst,
    "warp_instructions_per_ray": inst / rays,
    "warp_instructions_per_step": inst / steps,
    "avg_active_lanes": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "branch_efficiency_pct": g("smsp__sass_average_branch_targets_threads_uniform.pct"),
    "issue_active_pct": g("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
    "achieved_occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "l2_gbs": lts / dur_s / 1e9 if lts else None,
    "dram_gbs": dram / dur_s / 1e9,
    "dram_bytes": dram,
    "smem_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "local_memory_instructions": (g("sass__inst_executed_local_loads") or 0) +
    (g("sass__inst_executed_local_stores") or 0),
    # L1 data-pipe wavefronts (global + local + shared), summed over the SMs
    "l1_wavefronts": wf,
    "l1_wavefronts_lgds": (g("l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg") or 0) * nsm,
    "l1_wavefronts_shared": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "l1_wavefronts_pct_of_peak": g("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    "l1_wavefronts_per_step": wf / steps if wf else None,
    "global_load_requests": g("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    "global_load_sector_hit_pct": g("l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct"),
    "lsu_writeback_active_pct": g("l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed"),
    "fp64_pipe_pct": g("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    "stalls_per_issue": {k: g(f"smsp__average_warps_issue_stalled_{k}_per_issue_active.ratio")
                         for k in ("wait", "long_scoreboard", "short_scoreboard", "not_selected",
                                   "math_pipe_throttle", "branch_resolving", "dispatch_stall",
                                   "no_instruction", "mio_throttle", "lg_throttle", "barrier")},
    "sm_count": nsm,
}
if len(sys.argv) > 5:
    # keyed to the build it captured: mwt_build_id() (sources + flags; argv[6]
    # overrides, default: the build id of the sources in this tree)
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2112_05570_b200 import build as _b
    out["workload"], out["order"] = sys.argv[4], sys.argv[5]
    out["build_id"] = sys.argv[6] if len(sys.argv) > 6 else _b.build_id()
print(json.dumps(out, indent=1))
