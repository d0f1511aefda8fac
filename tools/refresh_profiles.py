"""Turn one tools/capture_round.sh call's gpurun_out/*_<tag>* files into the
committed evidence under profiles/ (round ROUND):

  rNN_bench.json, rNN_bench_reference.json, rNN_launches.csv,
  rNN_ncu_stats.json (keyed to the captured build's mwt_build_id),
  rNN_ncu_k_trace_<config>.txt, rNN_ncu_kd_bvh_floorplan64.txt, traffic.json

usage: python tools/refresh_profiles.py TAG [ROUND]   (ROUND default r02)
The build id is the one of the sources in this tree: run it before editing them.
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2112_05570_b200 import build as _b  # noqa: E402

tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r02"
O = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
bid = _b.build_id()


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT).stdout


def steps_sum(cfg, base, n):
    m = orc.Mesh.from_files(*bench.fixture(cfg, "mwt"))
    order = "coherent" if base in (0,) else "iid"
    return int(m.trace(orc.raygen(bench.mode_word(base, order), bench.CONFIGS[cfg][0], 0, 0, n))["steps"]
               .astype("int64").sum())


bench_line = last_json(f"{O}/bench_{tag}.json")
json.dump(bench_line, open(f"{P}/{rnd}_bench.json", "w"), indent=1)
json.dump(last_json(f"{O}/bench_ref_{tag}.json"), open(f"{P}/{rnd}_bench_reference.json", "w"), indent=1)
shutil.copy(f"{O}/launches_{tag}.csv", f"{P}/{rnd}_launches.csv")

# walk captures: (report, config, rays, steps, workload key, order, title)
caps = [("fp", "floorplan64", 1 << 26, bench_line["histogram"]["steps_sum"], "floorplan64/mwt", "coherent",
         "FloorPlan-64x64 MWT, 2^26 coherent box-entry rays (the headline launch)"),
        ("l1k", "lines1024", 1 << 24, steps_sum("lines1024", 0, 1 << 24), "lines1024/mwt", "coherent",
         "Lines-1024 MWT, box-entry part: 2^24 coherent rays, walk table staged in shared memory"),
        ("hair", "hair512", 1 << 24, steps_sum("hair512", 0, 1 << 24), "hair512/mwt", "coherent",
         "Hair-512 MWT, 2^24 coherent rays, per-triangle table staged in shared memory"),
        ("int", "lines1024_interior", 1 << 22, steps_sum("lines1024", 1, 1 << 22),
         "lines1024/mwt interior part", "iid",
         "Lines-1024 MWT, 2^22 iid interior-origin rays (the point-location path)")]
stats = []
for key, name, rays, steps, wl, order, title in caps:
    rep = f"{O}/prof_{key}_{tag}.ncu-rep"
    if not os.path.exists(rep):
        continue
    st = json.loads(run("tools/ncu_stats.py", rep, str(rays), str(steps), wl, order, bid))
    stats.append(st)
    hdr = (f"{title}\nncu --set full --import-source on --clock-control none (tools/capture_round.sh); "
           f"mwt_build_id {bid}\nsummaries: tools/ncu_summary.py (metrics, opcode mix, top stalled SASS), "
           "tools/ncu_src.py (per source function / line)\n\n")
    body = run("tools/ncu_summary.py", rep) + "\n" + run("tools/ncu_src.py", rep, "k_trace", "30")
    open(f"{P}/{rnd}_ncu_k_trace_{name}.txt", "w").write(hdr + body)
json.dump(stats, open(f"{P}/{rnd}_ncu_stats.json", "w"), indent=1)

# kd / BVH
ll = bench_line.get("like_for_like", {})
out = [f"kd-tree (c_t 2) and BVH (c_t 2) kernels on 4,194,304 FloorPlan-64x64 box-entry rays, "
       f"both generator orders (tools/prof_struct.py, tools/capture_round.sh); mwt_build_id {bid}\n"]
for order in ("coh", "iid"):
    rep = f"{O}/prof_struct_{order}_{tag}.ncu-rep"
    if not os.path.exists(rep):
        continue
    o = "coherent" if order == "coh" else "iid"
    out.append(f"=== {o} order")
    txt = run("tools/ncu_kernels.py", rep)
    out.append(txt)
    # warp instructions per operation (ops/ray from the bench's like-for-like line)
    for k in ("kd", "bvh"):
        opr = ll.get(o, {}).get(k, {}).get("ops_per_ray")
        blk = txt.split("== ")
        for b in blk:
            if b.startswith("k_kd" if k == "kd" else "void k_bvh"):
                wi = float(b.split("smsp__inst_executed.sum inst ")[1].split()[0])
                if opr:
                    out.append(f"  {k}: {wi / (4194304 * opr):.2f} warp instructions per operation "
                               f"({opr:.2f} ops/ray)")
    for kern in ("k_kd", "k_bvh"):
        out.append(run("tools/ncu_src.py", rep, kern, "15").split("\nline")[0])
open(f"{P}/{rnd}_ncu_kd_bvh_floorplan64.txt", "w").write("\n".join(out) + "\n")

tr = json.load(open(f"{P}/traffic.json")) if os.path.exists(f"{P}/traffic.json") else {}
if stats:
    tr["floorplan64/mwt"] = {"round": rnd, "dram_bytes_per_launch": int(stats[0]["dram_bytes"]),
                             "report": f"profiles/{rnd}_ncu_k_trace_floorplan64.txt", "build_id": bid}
json.dump(tr, open(f"{P}/traffic.json", "w"), indent=1)
print(json.dumps({k: bench_line[k] for k in ("value", "ms_per_step")}), bench_line["roofline"].get("bound"),
      [(s["workload"], round(s["issue_active_pct"], 1), round(s["l1_wavefronts_pct_of_peak"] or 0, 1))
       for s in stats])
