"""The reference's experiment (run_experiment, experiment.py:144-202) at the
BASELINE.json sizes, on one B200: per config, the box-entry ray set of the
bench (engine raygen, the BASELINE distribution) traced through the CDT and
the annealed MWT, and through all seven reference-built BVHs and kd-trees
with the c_t sweep's first-minimum rule (accel.py:845-862) -- every hit
checked against the brute-force closest hit of the same ray (_check).

This is the paper's comparison (traversal steps / ops per ray on the same
rays) at 2^24 rays per config (2^26 for FloorPlan), which the Python
reference needs core-days for.

usage: python tools/paper_table.py [out.json] [config ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05570_b200 import accel  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh  # noqa: E402
from paper_2112_05570_b200 import experiment  # noqa: E402
from paper_2112_05570_b200.experiment import run_experiment  # noqa: E402
from paper_2112_05570_b200.formats import load_structure  # noqa: E402
from paper_2112_05570_b200.model import Scene, load_triangulation  # noqa: E402

GRID = (0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0)
CONFIGS = {  # BASELINE.json configs: ray box and box-entry ray count
    "lines64": ((0.0, 0.0, 1.0, 1.0), 1 << 20),
    "lines1024": ((0.0, 0.0, 1.0, 1.0), 1 << 24),
    "grass4096": ((0.0, 0.0, 1.0, 0.5), 1 << 24),
    "hair512": ((0.0, 0.0, 1.0, 1.0), 1 << 24),
    "floorplan64": ((0.0, 0.0, 1.0, 1.0), 1 << 26),
    "grass4096l": ((0.0, 0.0, 1.0, 0.5), 1 << 24),
    "hair512r": ((0.0, 0.0, 1.0, 1.0), 1 << 24),
    # Lines-1024's 2^22 "recursive" rays: origins uniform in the box (point-location path)
    "lines1024-interior": ((0.0, 0.0, 1.0, 1.0), 1 << 22),
}
SEED = 0


MISMATCH: list = []
MISMATCH_COUNT: dict = {}


def _recording_check(scene_name, method, rays, seg, t, oracle_seg, oracle_t):
    """experiment._check over whole arrays, recording (not raising) the rays
    where the method and the brute-force closest hit disagree -- the
    near-degenerate rays the reference's own harness would stop on."""
    seg, oseg, t = np.asarray(seg), np.asarray(oracle_seg), np.asarray(t)
    tol = 1e-9 * np.maximum(1.0, np.abs(oracle_t))
    bad = ((seg >= 0) != (oseg >= 0)) | ((oseg >= 0) & ((seg != oseg) | (np.abs(t - oracle_t) > tol)))
    MISMATCH_COUNT[(scene_name, method)] = int(bad.sum())
    for k in np.nonzero(bad)[0][:64]:
        MISMATCH.append({"config": scene_name, "method": method, "ray": rays[k].tolist(),
                         "seg": int(seg[k]), "t": float(t[k]), "brute_seg": int(oseg[k]),
                         "brute_t": float(oracle_t[k])})
    return int(bad.sum())


experiment.check_hits = _recording_check


def run(cfg: str) -> dict:
    box, n = CONFIGS[cfg]
    mode = 1 if cfg.endswith("-interior") else 0
    d = os.path.join(ROOT, "fixtures", "data", cfg.split("-")[0])
    scene = Scene.load(os.path.join(d, "scene.txt"))
    tris = [load_triangulation(os.path.join(d, f"{w}.tri"), scene) for w in ("cdt", "mwt")]
    rays = DeviceMesh.from_files(os.path.join(d, "scene.txt"), os.path.join(d, "mwt.tri")).raygen(
        mode, box, SEED, 0, n)
    t0 = time.perf_counter()
    if os.path.exists(os.path.join(d, "bvh_ct1.npz")):
        bvh = {c: load_structure(os.path.join(d, f"bvh_ct{c:g}.npz")) for c in GRID}
        kd = {c: load_structure(os.path.join(d, f"kd_ct{c:g}.npz")) for c in GRID}
        rep = run_experiment(scene, tris, rays, labels=["cdt", "mwt"], ct_grid=GRID,
                             bvh_structures=bvh, kd_structures=kd)
        out = json.loads(rep.to_json())
    else:  # Lines-64: CDT and MWT only (BASELINE.json builds no kd-tree / BVH for it)
        oracle = accel._scene_mesh(scene).brute_force(rays)
        out = {"methods": []}
        for label, tri in zip(("cdt", "mwt"), tris):
            o = accel.trace_batch(tri, rays)
            experiment.check_hits(cfg, f"triangulation[{label}]", rays, o["seg"], o["t"], oracle["seg"],
                                  oracle["t"])
            steps = int(o["steps"].astype(np.int64).sum())
            out["methods"].append({"method": "triangulation", "label": label, "total_ops": steps,
                                   "mean_total": steps / n})
    wall = time.perf_counter() - t0
    out["brute_force_disagreements"] = [m for m in MISMATCH if m["config"] in (cfg, out.get("scene"))]
    out["brute_force_disagreement_counts"] = {m: c for (sc, m), c in MISMATCH_COUNT.items()
                                              if sc in (cfg, out.get("scene"))}
    out["baseline_config"] = cfg
    out["rays"] = n
    out["ray_box"] = box
    out["wall_s"] = wall
    return out


def table(results: list) -> str:
    rows = ["| config | rays | CDT steps/ray | MWT steps/ray | best kd-tree ops/ray (c_t) | "
            "best BVH ops/ray (c_t) | rays disagreeing with brute force | B200 wall (s) |",
            "|---|---|---|---|---|---|---|---|"]
    for r in results:
        m = {(x["method"], x["label"]): x for x in r["methods"]}
        cdt, mwt = m[("triangulation", "cdt")], m[("triangulation", "mwt")]
        kd = next((x for x in r["methods"] if x["method"] == "kd"), None)
        bvh = next((x for x in r["methods"] if x["method"] == "bvh"), None)
        ks = f"{kd['mean_total']:.3f} ({kd['label'][4:]})" if kd else "--"
        bs = f"{bvh['mean_total']:.3f} ({bvh['label'][4:]})" if bvh else "--"
        dis = ", ".join(f"{k}: {v}" for k, v in sorted(r["brute_force_disagreement_counts"].items())
                        if v) or "0"
        rows.append(f"| {r['baseline_config']} | {r['rays']:,} | {cdt['mean_total']:.3f} | "
                    f"{mwt['mean_total']:.3f} | {ks} | {bs} | {dis} | {r['wall_s']:.1f} |")
    return "\n".join(rows) + "\n"


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else "paper_table.json"
    cfgs = sys.argv[2:] or list(CONFIGS)
    res = []
    for c in cfgs:
        res.append(run(c))
        print(table(res[-1:]).splitlines()[-1], flush=True)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    with open(os.path.splitext(out)[0] + ".md", "w") as fh:
        fh.write(table(res))
    print(table(res))
