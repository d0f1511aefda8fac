"""Full-set reference digests: run the UNMODIFIED reference walk over every ray
of every BASELINE config and record per-chunk digests of its results.

Runs ONLY in the build container (imports /root/reference/pkg/src).  For each
(config, mesh, ray part) the rays are the engine generator's (oracle/raygen.py,
bit-identical to the device's K2; the benchmark's coherent order,
include/mwt.h MWT_RAYS_*_COHERENT, seed 0, global indices 0..n-1), and per ray
the reference computes what its own experiment loop does
(experiment.py:166-171):

    start = TriLocator(tri).locate(ray.origin)                accel.py:284-289
    hit, stats = traverse_triangulation(tri, ray, start, index)  accel.py:138-213

Per chunk of CHUNK rays it stores
  d_walk   sha256 of seg (int32, -1 miss, -2 TraversalError) | t (float64,
           every NaN as one pattern) | steps (int32, 0 on TraversalError)
  d_start  sha256 of start (int32)
  errors, hits, steps_sum  (diagnostics)
The engine reproduces d_walk from mwt_trace_generated_dev's per-ray outputs
and d_start from mwt_trace_dev's out_start (tests/test_gpu_fullset.py).

  python tests/golden/make_digests.py [--workers 7] [--mesh mwt] [cfg ...]

Progress is appended to tests/golden/_digests_partial.jsonl (resumable);
the final file is tests/golden/digests_<mesh>.json.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = ["/root/reference/pkg/src", ROOT]

CHUNK = 1 << 16
SEED = 0
# BASELINE.json configs: (box, [(base mode, rays)])
PARTS = {
    "lines64": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 20)]),
    "lines1024": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24), (1, 1 << 22)]),
    "grass4096": ((0.0, 0.0, 1.0, 0.5), [(0, 1 << 24)]),
    "hair512": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24)]),
    "floorplan64": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 26)]),
    "grass4096l": ((0.0, 0.0, 1.0, 0.5), [(0, 1 << 24)]),
    "hair512r": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24)]),
}
sys.path.insert(0, os.path.dirname(HERE))
from digests import digest_start, digest_walk  # noqa: E402  (tests/digests.py, shared with the tests)


_W = {}


def _init(which):
    from mintri.accel import SceneIndex, TriLocator  # noqa: F401
    _W["which"] = which


def _load(cfg, which):
    key = (cfg, which)
    if _W.get("key") != key:
        from mintri.accel import SceneIndex, TriLocator
        from mintri.scene import Scene
        from mintri.trimesh import load_triangulation
        d = os.path.join(ROOT, "fixtures", "data", cfg)
        scene = Scene.load(os.path.join(d, "scene.txt"))
        tri = load_triangulation(os.path.join(d, f"{which}.tri"), scene)
        _W.update(key=key, tri=tri, index=SceneIndex(scene), loc=TriLocator(tri))
    return _W["tri"], _W["index"], _W["loc"]


def work(task):
    cfg, which, base, lo, n = task
    from mintri.accel import TraversalError, traverse_triangulation
    from mintri.geometry import Point, Ray
    from oracle.raygen import coherent, raygen
    tri, index, loc = _load(cfg, which)
    box = PARTS[cfg][0]
    arr = raygen(coherent(base), box, SEED, lo, n)
    start = np.empty(n, np.int32)
    seg = np.full(n, -1, np.int32)
    t = np.full(n, np.nan)
    steps = np.zeros(n, np.int32)
    for i, (ox, oy, dx, dy) in enumerate(arr.tolist()):
        ray = Ray(Point(ox, oy), Point(dx, dy))
        s = loc.locate(ray.origin)
        start[i] = s
        try:
            hit, st = traverse_triangulation(tri, ray, s, index)
        except TraversalError:
            seg[i] = -2
            continue
        steps[i] = st.tri_steps
        if hit is not None:
            seg[i] = hit.seg
            t[i] = hit.t
    return {"cfg": cfg, "mesh": which, "mode": base, "lo": lo, "n": n,
            "d_walk": digest_walk(seg, t, steps), "d_start": digest_start(start),
            "errors": int((seg == -2).sum()), "hits": int((seg >= 0).sum()),
            "steps_sum": int(steps.sum())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=max(1, os.cpu_count() - 1))
    ap.add_argument("--mesh", default="mwt")
    ap.add_argument("cfgs", nargs="*", default=list(PARTS))
    a = ap.parse_args()
    part_path = os.path.join(HERE, f"_digests_partial_{a.mesh}.jsonl")
    done = set()
    if os.path.exists(part_path):
        with open(part_path) as fh:
            for ln in fh:
                r = json.loads(ln)
                done.add((r["cfg"], r["mesh"], r["mode"], r["lo"]))
    tasks = []
    for cfg in a.cfgs:
        box, parts = PARTS[cfg]
        for base, total in parts:
            for lo in range(0, total, CHUNK):
                if (cfg, a.mesh, base, lo) not in done:
                    tasks.append((cfg, a.mesh, base, lo, min(CHUNK, total - lo)))
    # keep a worker on one config as long as possible (mesh load + anchor cache)
    print(f"{len(tasks)} chunks to run ({len(done)} done)", flush=True)
    t0 = time.time()
    with mp.get_context("fork").Pool(a.workers, initializer=_init, initargs=(a.mesh,)) as pool, \
            open(part_path, "a") as out:
        for k, r in enumerate(pool.imap_unordered(work, tasks, chunksize=1)):
            out.write(json.dumps(r) + "\n")
            out.flush()
            if k % 20 == 0:
                el = time.time() - t0
                print(f"{k + 1}/{len(tasks)} chunks, {el:.0f} s, eta {el / (k + 1) * (len(tasks) - k - 1):.0f} s",
                      flush=True)
    # assemble
    rows = {}
    with open(part_path) as fh:
        for ln in fh:
            r = json.loads(ln)
            rows[(r["cfg"], r["mode"], r["lo"])] = r
    final = {"chunk": CHUNK, "seed": SEED, "mesh": a.mesh,
             "generator": "oracle.raygen.coherent(base) = include/mwt.h MWT_RAYS_*_COHERENT",
             "reference": "TriLocator(tri).locate + traverse_triangulation (accel.py:284-289, :138-213)",
             "configs": {}}
    for cfg, (box, parts) in PARTS.items():
        cd = {"box": list(box), "parts": []}
        complete = True
        for base, total in parts:
            chunks = []
            for lo in range(0, total, CHUNK):
                r = rows.get((cfg, base, lo))
                if r is None:
                    complete = False
                    break
                chunks.append([r["d_walk"], r["d_start"], r["errors"], r["hits"], r["steps_sum"]])
            cd["parts"].append({"mode": base, "n": total, "chunks": chunks})
        if complete:
            final["configs"][cfg] = cd
    # configs recorded by an earlier run (whose partial file is gone) are kept
    fpath = os.path.join(HERE, f"digests_{a.mesh}.json")
    if os.path.exists(fpath):
        with open(fpath) as fh:
            old = json.load(fh)
        if old.get("chunk") == CHUNK and old.get("seed") == SEED:
            for cfg, cd in old["configs"].items():
                final["configs"].setdefault(cfg, cd)
    final["configs"] = {c: final["configs"][c] for c in PARTS if c in final["configs"]}
    with open(fpath, "w") as fh:
        json.dump(final, fh, separators=(",", ":"))
    print("configs complete:", sorted(final["configs"]), flush=True)


if __name__ == "__main__":
    main()
