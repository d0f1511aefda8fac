"""Like-for-like throughput on every config with reference-built structures:
the same 2^22 box-entry rays (loaded from HBM) through the MWT walk, the best
SAH BVH and the best roped kd-tree (c_t by the reference's minimum-ops rule),
each timed with CUDA events (bench.like_for_like).

usage: python tools/like_for_like_all.py [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else "like_for_like.json"
    res = {}
    for cfg in ("lines1024", "grass4096", "hair512", "floorplan64", "grass4096l", "hair512r"):
        res[cfg] = bench.like_for_like(cfg, 0)
        r = res[cfg]
        for order in ("coherent", "iid"):
            print(cfg, order, {k: (round(v["rays_per_s"] / 1e9, 3), round(v["ops_per_ray"], 3))
                               for k, v in r[order].items()}, flush=True)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
