"""A/B of the ray generator's coherent order (include/mwt.h MWT_RAYS_COHERENT)
on the fused trace: rays/s and steps/ray per (config, group_log2, cell_bits).

  python tools/coherence_ab.py [out.json] [cfg ...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_05570_b200 import _lib  # noqa: E402
from paper_2112_05570_b200.engine import DeviceMesh, new_histogram, summarize_histogram  # noqa: E402

SIZES = {"lines64": 1 << 20, "lines1024": 1 << 24, "grass4096": 1 << 24, "hair512": 1 << 24,
         "floorplan64": 1 << 26}
BOX = {"grass4096": (0.0, 0.0, 1.0, 0.5)}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/coherence_ab.json"
    cfgs = sys.argv[2:] or ["floorplan64", "lines1024", "grass4096", "hair512"]
    gs = [int(x) for x in os.environ.get("AB_G", "5,7,9").split(",")]
    cs = [int(x) for x in os.environ.get("AB_C", "8,10,11,12,14").split(",")]
    variants = [(0, 0)] + [(g, c) for g in gs for c in cs]
    res = {}
    for cfg in cfgs:
        d = os.path.join(ROOT, "fixtures", "data", cfg)
        m = DeviceMesh.from_files(os.path.join(d, "scene.txt"), os.path.join(d, "mwt.tri"))
        n = SIZES[cfg]
        box = BOX.get(cfg, (0.0, 0.0, 1.0, 1.0))
        modes = [0, 1] if cfg == "lines1024" else [0]
        for base in modes:
            for g, c in variants:
                mode = _lib.rays_coherent(base, g, c)
                h = new_histogram()
                ms = timeit(lambda: m.trace_generated_device(mode, box, 0, 0, n >> (2 * base), True, None))
                m.trace_generated_device(mode, box, 0, 0, n >> (2 * base), False, h)
                hs = summarize_histogram(h)
                key = f"{cfg}/mode{base}/g{g}/c{c}"
                res[key] = {"ms": ms, "rays_per_s": (n >> (2 * base)) / ms * 1e3,
                            "steps_per_ray": hs["steps_per_ray"], "hit": hs["hits"] / hs["rays"]}
                print(key, json.dumps(res[key]), flush=True)
        del m
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
