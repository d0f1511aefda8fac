"""Benchmark: 2D rays/s of the MWT walk (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[4], the largest single-GPU config):
FloorPlan-64x64 rotated, reference-annealed MWT (24,604 triangles), 2^26
isotropic box-entry fp64 rays per step.  Each ray is generated on device (K2),
given its start triangle (box-entry table / K3 locate), walked (K4) with
per-ray seg / t / steps written to HBM, and counted in the step / hit / status
histograms (K7), in one persistent launch per ray part.  The generator's
default order is coherent (include/mwt.h MWT_RAYS_*_COHERENT: 512-ray groups
share the top 12 bits of every draw; each ray is still an exact draw of the
iid distribution), --order iid is the round-1 order.

Multi-GPU (torchrun, one rank per GPU): the rays shard by global index with the
mesh replicated; --scaling strong (default) splits the step's 2^26 rays over
the ranks (sharding.strong_shard), --scaling weak gives every rank the full
count (sharding.weak_shard).  The only collective is one all-reduce of the
int64 histograms (sharding.allreduce_histogram).  The L2 is flushed (256 MiB
write) before every timed step, outside the timed region.

  python bench.py [--gpus N --steps K --warmup W] [--config floorplan64] [--order coherent]
                  [--scaling strong] [--impl reference]

One JSON line on rank 0.  ``--impl reference`` times the reference CPU path
(the C oracle restatement of accel.py's locate + walk, all host threads) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (box, [(base mode, rays per step)])  -- BASELINE.json configs[0..4]
    "lines64": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 20)]),
    "lines1024": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24), (1, 1 << 22)]),
    "grass4096": ((0.0, 0.0, 1.0, 0.5), [(0, 1 << 24)]),
    "hair512": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24)]),
    "floorplan64": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 26)]),
    # Grass / Hair under the other crossing policies (fixtures/gen_fixtures.py)
    "grass4096l": ((0.0, 0.0, 1.0, 0.5), [(0, 1 << 24)]),
    "hair512r": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24)]),
}
SEED = 0
ALGO_BYTES_PER_STEP = 32  # 16-B link record + 16-B apex corner per triangle step
COHERENT_GROUP_LOG2, COHERENT_CELL_BITS = 9, 12  # include/mwt.h MWT_RAYS_*_COHERENT


def mode_word(base: int, order: str) -> int:
    """include/mwt.h generator mode word of a ray part."""
    if order == "iid":
        return base
    return base | (COHERENT_GROUP_LOG2 << 8) | (COHERENT_CELL_BITS << 16)


def part_name(base: int) -> str:
    return "box_entry" if base == 0 else "interior"


def shards(args, world: int, rank: int):
    """[(base mode, first global index, count)] of this rank (sharding.py)."""
    from paper_2112_05570_b200.sharding import strong_shard, weak_shard
    out = []
    for base, n in CONFIGS[args.config][1]:
        sh = strong_shard(rank, world, n) if args.scaling == "strong" else weak_shard(rank, world, n)
        out.append((base, sh.first, sh.count))
    return out


def config_dict(args, world: int) -> dict:
    """The workload's `config`, identical on both arms (the driver compares them)."""
    per = {part_name(b): (n if args.scaling == "strong" else n * world) for b, n in CONFIGS[args.config][1]}
    return {"workload": f"{args.config}/{args.mesh}", "rays_per_step": per, "ray_order": args.order,
            "ray_generator": (f"MWT_RAYS_COHERENT(base, {COHERENT_GROUP_LOG2}, {COHERENT_CELL_BITS})"
                              if args.order == "coherent" else "MWT_RAYS_BOX_ENTRY / MWT_RAYS_INTERIOR (iid)"),
            "seed": SEED, "scaling": args.scaling, "box": list(CONFIGS[args.config][0])}


def l2_peak_file():
    p = os.path.join(ROOT, "profiles", "r01_l2_peak.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["l2_read_gbs"])
    return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _sample(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            if out:
                self.rows.append([c.strip() for c in out.split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()
        if not self.rows:
            self._sample()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def fixture(cfg: str, which: str):
    d = os.path.join(ROOT, "fixtures", "data", cfg)
    return os.path.join(d, "scene.txt"), os.path.join(d, f"{which}.tri")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_reference(args, world: int, rank: int, budget_s: float = 20.0):
    """The reference CPU path (oracle restatement of TriLocator.locate +
    traverse_triangulation, OpenMP over all host threads) on a bounded sample
    of the same workload (the first rays of every part, same generator order):
    returns (rays/s, cores, sample text)."""
    from oracle import oracle as orc
    # every host thread this process may run on (torchrun sets OMP_NUM_THREADS=1 per rank)
    orc.set_num_threads(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
    box = CONFIGS[args.config][0]
    m = orc.Mesh.from_files(*fixture(args.config, args.mesh))
    cores = orc.num_threads()
    parts = shards(args, world, rank)
    total = sum(n for _, _, n in parts)
    calib = []
    for base, first, n in parts:
        k = min(n, 1 << 16)
        r = orc.raygen(mode_word(base, args.order), box, SEED, first, k)
        t0 = time.perf_counter()
        m.trace(r)
        calib.append((time.perf_counter() - t0) / k)
    per_ray = sum(c * n for c, (_, _, n) in zip(calib, parts)) / max(total, 1)
    scale = min(1.0, budget_s / max(per_ray * total, 1e-9))
    rays, t_total, desc = 0, 0.0, []
    for base, first, n in parts:
        k = max(1 << 12, int(n * scale))
        r = orc.raygen(mode_word(base, args.order), box, SEED, first, k)
        t0 = time.perf_counter()
        m.trace(r)
        t_total += time.perf_counter() - t0
        rays += k
        desc.append(f"{k} {part_name(base).replace('_', '-')} rays from index {first}")
    return rays / t_total, cores, f"{args.config}/{args.mesh} ({args.order} order): " + " + ".join(desc) + \
        " (oracle locate + walk, OpenMP over all host threads)"


_PYREF = {}


def _pyref_chunk(task):
    """One chunk of rays through the unmodified reference (worker of
    python_reference; the mesh was loaded before the fork)."""
    lo, arr = task
    from mintri.accel import TraversalError, traverse_triangulation
    from mintri.geometry import Point, Ray
    tri, index, loc = _PYREF["tri"], _PYREF["index"], _PYREF["loc"]
    seg = np.full(len(arr), -1, np.int32)
    steps = np.zeros(len(arr), np.int32)
    for i, (ox, oy, dx, dy) in enumerate(arr.tolist()):
        ray = Ray(Point(ox, oy), Point(dx, dy))
        try:
            hit, st = traverse_triangulation(tri, ray, loc.locate(ray.origin), index)
        except TraversalError:
            seg[i] = -2
            continue
        steps[i] = st.tri_steps
        if hit is not None:
            seg[i] = hit.seg
    return lo, seg, steps


def python_reference(args, budget_s: float = 8.0):
    """The reference's own Python path (TriLocator.locate + traverse_triangulation
    with a shared SceneIndex, accel.py:138-213, :284-289) from the unmodified
    package in baseline/_ref, one forked worker per host core, on a bounded
    sample of the workload's first rays; the results are checked against the
    oracle on the same rays.  None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mintri")):
        return None
    import multiprocessing as mp
    sys.path.insert(0, ref)
    from mintri.accel import SceneIndex, TriLocator
    from mintri.scene import Scene
    from mintri.trimesh import load_triangulation
    from oracle import oracle as orc
    scene_p, tri_p = fixture(args.config, args.mesh)
    scene = Scene.load(scene_p)
    tri = load_triangulation(tri_p, scene)
    _PYREF.update(tri=tri, index=SceneIndex(scene), loc=TriLocator(tri))
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    base = CONFIGS[args.config][1][0][0]
    box = CONFIGS[args.config][0]
    probe = orc.raygen(mode_word(base, args.order), box, SEED, 0, 256)
    t0 = time.perf_counter()
    _pyref_chunk((0, probe))
    per_ray = (time.perf_counter() - t0) / len(probe)
    n = int(min(1 << 20, max(cores * 256, budget_s * cores / max(per_ray, 1e-9))))
    n -= n % 256
    arr = orc.raygen(mode_word(base, args.order), box, SEED, 0, n)
    tasks = [(lo, arr[lo:lo + 256]) for lo in range(0, n, 256)]
    with mp.get_context("fork").Pool(cores) as pool:
        t0 = time.perf_counter()
        res = pool.map(_pyref_chunk, tasks, chunksize=max(1, len(tasks) // (4 * cores)))
        dt = time.perf_counter() - t0
    seg = np.concatenate([r[1] for r in sorted(res, key=lambda r: r[0])])
    steps = np.concatenate([r[2] for r in sorted(res, key=lambda r: r[0])])
    o = orc.Mesh.from_files(scene_p, tri_p).trace(arr)
    return {"value": n / dt, "unit": "rays/s", "cores": cores, "kind": "reference (Python, unmodified)",
            "sample": f"{args.config}/{args.mesh} ({args.order} order): the first {n} "
                      f"{part_name(base).replace('_', '-')} rays, multiprocessing pool (fork), one worker per core",
            "matches_oracle": bool(np.array_equal(seg, o["seg"]) and np.array_equal(steps, o["steps"])),
            "source": "baseline/_ref (tools/install_reference.sh)"}


def run_reference_arm(args, world: int, rank: int):
    if rank != 0:
        return
    vals, sample, cores = [], "", 0
    for _ in range(args.warmup):
        cpu_reference(args, world, 0, budget_s=2.0)
    for _ in range(args.steps):
        v, cores, sample = cpu_reference(args, world, 0, budget_s=args.cpu_budget / max(1, args.steps))
        vals.append(v)
    v = float(np.mean(vals))
    step_rays = sum(n for _, n in CONFIGS[args.config][1]) * (1 if args.scaling == "strong" else world)
    line = {
        "metric": "rays_per_s_mwt_walk", "value": v, "unit": "rays/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_rays / v * 1e3,  # one step's rays at the sampled rate
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded rays, reference-built fixtures)",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": v, "unit": "rays/s", "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        pr = python_reference(args)
    except Exception as e:  # noqa: BLE001
        pr = {"error": f"{type(e).__name__}: {e}"}
    if pr is not None:
        line["cpu_baseline"]["python_reference"] = pr
    print(json.dumps(line), flush=True)


def lib_build_id() -> str:
    from paper_2112_05570_b200 import _lib
    return _lib.lib.mwt_build_id().decode()


def ncu_stats_for(workload: str, order: str, bid: str):
    """The committed ncu figures of this build's dominant launch, if a capture
    of exactly this build (mwt_build_id: sources + flags) and workload exists
    (profiles/r*_ncu_stats.json)."""
    pdir = os.path.join(ROOT, "profiles")
    for f in sorted(os.listdir(pdir), reverse=True):
        if not f.endswith("_ncu_stats.json"):
            continue
        with open(os.path.join(pdir, f)) as fh:
            d = json.load(fh)
        for e in (d if isinstance(d, list) else [d]):
            if e.get("build_id") == bid and e.get("workload") == workload and e.get("order") == order:
                return dict(e, file=f)
    return None


def roofline(args, hb, kms, clocks, sms, local):
    """Roofs of the dominant launch (the largest ray part): algorithmic bytes
    (32 B per triangle step) against the L2 read peak measured
    live and the HBM peak, and -- from the committed ncu capture of this exact
    build -- issue slots and L1 data-pipe wavefronts against their peaks at the
    sampled SM clock.  `bound` is the largest measured utilisation."""
    from paper_2112_05570_b200.engine import probe_l2_read_gbs
    algo = hb["steps_sum"] * ALGO_BYTES_PER_STEP
    achieved = algo / (kms / 1e3) / 1e9
    hbm_pk, hbm_src = peaks()
    try:
        l2pk, l2src = probe_l2_read_gbs(local), "measured live (mwt_probe_l2_read: 64 MiB, 200 passes)"
    except Exception as e:  # noqa: BLE001
        l2pk, l2src = l2_peak_file(), f"profiles/r01_l2_peak.json ({e})"
    sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    wl = f"{args.config}/{args.mesh}"
    st = ncu_stats_for(wl, args.order, lib_build_id())
    r = {"kernel": "k_trace (mwt_trace_generated_dev, largest ray part)", "kernel_ms": kms,
         "algo_bytes_per_launch": algo,
         "algo_bytes_rule": "32 B per triangle step (one step record: 2 exit words + apex corner)",
         "l2_algorithmic": {"achieved": achieved, "peak": l2pk, "unit": "GB/s",
                            "frac": achieved / l2pk if l2pk else None, "peak_source": l2src},
         "hbm_algorithmic": {"achieved": achieved, "peak": hbm_pk, "unit": "GB/s", "frac": achieved / hbm_pk,
                             "peak_source": hbm_src,
                             "note": "the mesh is L2/L1/shared-memory resident; HBM carries only the "
                                     "per-ray output, so this is not a binding roof"},
         "l1_return_algorithmic": {"achieved": achieved, "peak": sms * 128 * sm_mhz / 1e3, "unit": "GB/s",
                                   "frac": achieved / (sms * 128 * sm_mhz / 1e3),
                                   "note": "the 32 B per step against the L1/shared-memory data path into the "
                                           "registers: 128 B per SM per cycle at the sampled SM clock "
                                           "(B300_MICROARCH.md smem/L1 crossbar)"}}
    cands = {}
    if st is not None and st.get("rays"):
        # a capture of this launch size, or (a rank's shard of the headline
        # workload) the same workload at another ray count: its counts per ray
        scale = hb["rays"] / st["rays"]
        inst = st["warp_instructions"] * scale
        ipk = sms * 4 * sm_mhz / 1e3
        cands["issue"] = {"achieved": inst / (kms / 1e3) / 1e9, "peak": ipk, "unit": "G warp-inst/s",
                          "note": "4 warp instructions per SM per cycle at the sampled SM clock"}
        wf = st.get("l1_wavefronts")
        if wf:
            wf *= scale
            cands["l1_wavefront"] = {"achieved": wf / (kms / 1e3) / 1e9, "peak": sms * sm_mhz / 1e3,
                                     "unit": "G wavefronts/s",
                                     "note": "L1 data pipe (global + shared): one wavefront per SM per cycle"}
        for c in cands.values():
            c["frac"] = c["achieved"] / c["peak"]
        r["ncu_capture"] = {k: st.get(k) for k in ("file", "report", "build_id", "warp_instructions",
                                                     "l1_wavefronts", "dram_bytes", "duration_ms", "rays")}
        if scale != 1.0:
            r["ncu_capture"]["scaled_to_rays"] = hb["rays"]
        r["traffic"] = st.get("dram_bytes") * scale if st.get("dram_bytes") else None
    else:
        r["traffic"] = None
        r["ncu_capture"] = None
    if cands:
        bound = max(cands, key=lambda k: cands[k]["frac"])
        r.update({"bound": bound, **{k: cands[bound][k] for k in ("achieved", "peak", "unit", "frac")}})
        r["measured_roofs"] = cands
    else:  # no capture of this build: the algorithmic L2 figure
        r.update({"bound": "l2", "achieved": achieved, "peak": l2pk, "unit": "GB/s",
                  "frac": achieved / l2pk if l2pk else None,
                  "note": "no ncu capture of this library build: algorithmic bytes against the L2 read peak"})
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="floorplan64", choices=sorted(CONFIGS))
    ap.add_argument("--mesh", default="mwt", choices=["mwt", "cdt"])
    ap.add_argument("--order", default="coherent", choices=["coherent", "iid"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu/extras)")
    ap.add_argument("--no-extra", action="store_true", help="skip per-config / like-for-like lines")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import DeviceMesh, _stream, new_histogram, summarize_histogram
    from paper_2112_05570_b200.sharding import allreduce_histogram, max_over_ranks

    # functional check of the N > 1 code path on a one-GPU box only (never a
    # measurement): MWT_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 and uses gloo
    one_dev = os.environ.get("MWT_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    box = CONFIGS[args.config][0]
    mesh = DeviceMesh.from_files(*fixture(args.config, args.mesh), device=local)
    parts = shards(args, world, rank)  # [(base, first, count)] of this rank
    rays_per_rank = sum(n for _, _, n in parts)
    rays_total = sum(v for v in config_dict(args, world)["rays_per_step"].values())
    outs = [dict(seg=torch.empty(n, dtype=torch.int32, device=dev),
                 t=torch.empty(n, dtype=torch.float64, device=dev),
                 steps=torch.empty(n, dtype=torch.int32, device=dev)) for _, _, n in parts]
    hist = new_histogram(local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    P = _lib.ptr
    boxarr = np.asarray(box, np.float64)

    # the parts run on their own streams, so one part's tail overlaps the next
    # part's start (each kernel keeps one CTA per SM)
    pstreams = [stream] + [torch.cuda.Stream(device=dev) for _ in parts[1:]]
    pptrs = [_stream(ps) for ps in pstreams]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in parts]
    zero_done = torch.cuda.Event()

    def launch_on(k, h, outputs=True):
        base, first, n = parts[k]
        o = outs[k] if outputs else {}
        _lib.check(_lib.lib.mwt_trace_generated_dev(
            mesh.handle, mode_word(base, args.order), P(boxarr), SEED, first, n,
            P(o.get("seg")), P(o.get("t")), P(o.get("steps")), P(h), pptrs[k]), "trace_generated")

    def step(timed=False):
        hist.zero_()
        zero_done.record(stream)
        for k in range(len(parts)):
            ps = pstreams[k]
            if k:
                ps.wait_event(zero_done)
            if timed:
                ev[k][0].record(ps)
            launch_on(k, hist)
            if timed:
                ev[k][1].record(ps)
        for ps in pstreams[1:]:
            stream.wait_stream(ps)
        allreduce_histogram(hist)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    kernel_ms = [0.0 for _ in parts]
    total_ms = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0.record(stream)
            step(timed=True)
            e1.record(stream)
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1)
            for k in range(len(parts)):
                kernel_ms[k] += ev[k][0].elapsed_time(ev[k][1])
    total_ms = max_over_ranks(total_ms, device=dev)
    ms_per_step = total_ms / args.steps
    value = rays_total / (ms_per_step / 1e3)
    hsum = summarize_histogram(hist)  # the last step's all-reduced histogram: the whole job's rays
    clocks = clk.summary()

    # the dominant launch (largest ray part) alone, for its step count
    big = max(range(len(parts)), key=lambda k: parts[k][2])
    hk = new_histogram(local)
    launch_on(big, hk, outputs=False)
    torch.cuda.synchronize()
    hb = summarize_histogram(hk)
    kms = kernel_ms[big] / args.steps
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    line = {
        "metric": "rays_per_s_mwt_walk", "value": value, "unit": "rays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded on-device rays; reference-built {args.config} scene + "
                f"{'annealed MWT' if args.mesh == 'mwt' else 'CDT'})",
        "config": config_dict(args, world),
        "workload_info": {"triangles": mesh.info.num_triangles, "segments": mesh.info.num_segments,
                          "rays_per_rank": rays_per_rank, "rays_per_s_per_gpu": value / world, "parallelism": f"ray shards x{world}, mesh replicated",
                          "l2": "flushed (256 MiB write) before every timed step",
                          "steps_per_ray": hsum["steps_per_ray"],
                          "hit_fraction": hsum["hits"] / max(1, hsum["rays"]),
                          "walk_table": (f"shared memory ({mesh.info.walk_smem_bytes} B per CTA)"
                                         if mesh.info.walk_smem_bytes > 0 else "32-B step records in L1/L2")},
        "parts": [{"rays": part_name(b), "first": f, "n": n, "stream_ms": kernel_ms[k] / args.steps}
                  for k, (b, f, n) in enumerate(parts)],
        "gpu_launches": len(parts) * args.steps,
        "histogram": {k: hsum[k] for k in ("rays", "hits", "misses", "steps_sum", "status")},
        "clocks": clocks,
    }
    line["roofline"] = roofline(args, hb, kms, clocks, sms, local)
    spr = hb["steps_sum"] / max(1, hb["rays"])
    hitf = hb["hits"] / max(1, hb["rays"])
    line["per_ray_bytes"] = {
        "walk_steps": ALGO_BYTES_PER_STEP * spr, "first_triangle": 48.0, "boundary_table": 40.0,
        "output": 16.0, "hit_segment": 32.0 * hitf, "input_ray": 0.0,
        "total": ALGO_BYTES_PER_STEP * spr + 48.0 + 40.0 + 16.0 + 32.0 * hitf,
        "note": "walk = 32 B x steps/ray (the roofline's algorithmic bytes); first triangle = its three "
                "corners; boundary table = bucket word + edge interval + word; output = seg + t + steps; "
                "rays are generated on device"}
    if rank == 0 and world == 1 and not args.profile and not args.no_extra:
        line["per_config"] = per_config(local)
        line["like_for_like"] = like_for_like(args.config, local)
    if not args.no_e2e and not args.profile:
        line["e2e"] = e2e(mesh, parts, box, world, args, dev)
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        v, cores, sample = cpu_reference(args, world, rank, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": "rays/s", "cores": cores, "kind": "port",
                                "sample": sample, "cpu_model": cpu_model()}
        try:  # the unmodified Python reference beside the port, when it was shipped
            pr = python_reference(args)
        except Exception as e:  # noqa: BLE001  (informational; never fails the bench)
            pr = {"error": f"{type(e).__name__}: {e}"}
        if pr is not None:
            line["cpu_baseline"]["python_reference"] = pr
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _time_ms(fn, reps=5):
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def per_config(local):
    """Every config and mesh at its full BASELINE ray count, both generator
    orders: the fused trace (K2+K3+K4+K7) with per-ray outputs (not the headline)."""
    import torch
    from paper_2112_05570_b200.engine import DeviceMesh, new_histogram, summarize_histogram
    res = {}
    for cfg, (box, parts) in CONFIGS.items():
        for which in ("mwt", "cdt"):
            paths = fixture(cfg, which)
            if not os.path.exists(paths[1]):
                continue
            m = DeviceMesh.from_files(*paths, device=local)
            for order in ("coherent", "iid"):
                for base, n in parts:
                    mw = mode_word(base, order)
                    h = new_histogram(local)
                    ms = _time_ms(lambda: m.trace_generated_device(mw, box, SEED, 0, n, outputs=True, hist=None))
                    m.trace_generated_device(mw, box, SEED, 0, n, outputs=False, hist=h)
                    torch.cuda.synchronize()
                    hs = summarize_histogram(h)
                    res[f"{cfg}/{which}/{order}/{part_name(base)}"] = {
                        "rays": n, "ms": ms, "rays_per_s": n / (ms / 1e3), "steps_per_ray": hs["steps_per_ray"],
                        "hit_fraction": hs["hits"] / max(1, hs["rays"]), "triangles": m.info.num_triangles,
                        "walk_smem_bytes": int(m.info.walk_smem_bytes)}
            del m
    return res


def like_for_like(cfg, local, n=1 << 22):
    """The same n box-entry rays (loaded from HBM) through the MWT walk, the
    reference-built SAH BVH and roped kd-tree (c_t chosen by the reference rule:
    minimum total ops over the same rays, accel.py:845-862), in both orders."""
    from paper_2112_05570_b200.engine import DeviceBvh, DeviceKd, DeviceMesh
    from paper_2112_05570_b200.formats import load_structure
    box = CONFIGS[cfg][0]
    d = os.path.join(ROOT, "fixtures", "data", cfg)
    mesh = DeviceMesh.from_files(*fixture(cfg, "mwt"), device=local)
    structs = {}
    for kind, cls in (("bvh", DeviceBvh), ("kd", DeviceKd)):
        files = sorted(f for f in os.listdir(d) if f.startswith(kind + "_ct"))
        structs[kind] = [(f, cls(mesh, load_structure(os.path.join(d, f)))) for f in files]
    out = {}
    for order in ("coherent", "iid"):
        rays = mesh.raygen_device(mode_word(0, order), box, SEED, 0, n)
        o = {}
        ms = _time_ms(lambda: mesh.trace_device(rays, None, want=("seg", "t", "steps")))
        w = mesh.trace_device(rays, None, want=("seg", "steps"))
        o["mwt_walk"] = {"ms": ms, "rays_per_s": n / (ms / 1e3),
                         "ops_per_ray": float(w["steps"].double().mean()), "ops": "tri_steps"}
        for kind, lst in structs.items():
            if not lst:
                continue
            best = None
            for f, st in lst:
                r = st.trace_device(rays)
                keys = ("node_tests", "prim_tests") if kind == "bvh" else ("nodes", "ropes", "prims")
                ops = sum(float(r[k].double().sum()) for k in keys)
                if best is None or ops < best[0]:
                    best = (ops, f, st)
            ops, f, st = best
            ms = _time_ms(lambda: st.trace_device(rays))
            o[kind] = {"ms": ms, "rays_per_s": n / (ms / 1e3), "ops_per_ray": ops / n, "c_t": float(st.c_t),
                       "file": f}
        out[order] = o
    out["rays"] = f"{n} box-entry rays of {cfg} per order, loaded from HBM (32 B/ray in, seg/t/counters out)"
    return out


def e2e(mesh, parts, box, world, args, dev):
    """The public host-buffer C-ABI call (mwt_trace_host: the drop-in's batch
    entry point) per step: H2D of the step's rays from pinned memory, device
    locate + walk, D2H of seg/t/u/steps into pinned memory."""
    import torch
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.sharding import max_over_ranks
    P = _lib.ptr
    host = []
    for base, first, n in parts:
        r = mesh.raygen_device(mode_word(base, args.order), box, SEED, first, n)
        h = torch.empty((n, 4), dtype=torch.float64, pin_memory=True)
        h.copy_(r)
        outs = dict(seg=torch.empty(n, dtype=torch.int32, pin_memory=True),
                    t=torch.empty(n, dtype=torch.float64, pin_memory=True),
                    u=torch.empty(n, dtype=torch.float64, pin_memory=True),
                    steps=torch.empty(n, dtype=torch.int32, pin_memory=True))
        host.append((n, h, outs))
        del r
    torch.cuda.synchronize()

    def step():
        for n, h, o in host:
            _lib.check(_lib.lib.mwt_trace_host(mesh.handle, P(h), None, n, None, P(o["seg"]), P(o["t"]),
                                               P(o["u"]), P(o["steps"]), None), "trace_host")

    for _ in range(2):
        step()
    steps = max(3, min(args.steps, 5))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = max_over_ranks((time.perf_counter() - t0) / steps, device=dev)
    nr = sum(n for _, _, n in parts)
    total = sum(v for v in config_dict(args, world)["rays_per_step"].values())
    return {"value": total / dt, "unit": "rays/s", "h2d_bytes_per_step": 32 * nr,
            "d2h_bytes_per_step": 24 * nr, "ms_per_step": dt * 1e3,
            "api": "mwt_trace_host (include/mwt.h), pinned host buffers, 8-stream chunked pipeline",
            "timing": "host wall clock around synchronous calls, max over ranks"}


if __name__ == "__main__":
    main()
