"""Benchmark: 2D rays/s of the MWT walk (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1], Lines-1024): per GPU and step, 2^24
isotropic box-entry rays plus 2^22 'recursive' rays with interior origins,
each generated on device (K2), located (K3), walked through the annealed MWT
(K4) with per-ray results written to HBM and step/hit histograms accumulated
(K7); the two parts run on two streams (one part's tail overlaps the other's
start); for N > 1 the histograms are summed with one NCCL all-reduce.  Rays are
sharded by global index (rank r traces indices [r*n, (r+1)*n)), so per-GPU
work is fixed: weak scaling.  The L2 is flushed (256 MiB write) before every
timed step, outside the timed region.

  python bench.py [--gpus N --steps K --warmup W] [--config lines1024] [--impl reference]

One JSON line on rank 0.  ``--impl reference`` times the reference CPU path
(the C oracle restatement of accel.py, all host threads) on a bounded sample.
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
    # name: (box, [(mode, rays per GPU per step)])
    "lines64": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 20)]),
    "lines1024": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24), (1, 1 << 22)]),
    "grass4096": ((0.0, 0.0, 1.0, 0.5), [(0, 1 << 24)]),
    "hair512": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 24)]),
    "floorplan64": ((0.0, 0.0, 1.0, 1.0), [(0, 1 << 26)]),
}
SEED = 0
ALGO_BYTES_PER_STEP = 32  # 16-B link record + 16-B apex corner per triangle step


def l2_peak():
    """L2 read bandwidth measured on the box (profiles/r01_l2_peak.json,
    tools/l2_peak.cu): the on-chip roof for meshes that live in L2."""
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


def cpu_reference(cfg: str, which: str, parts, budget_s: float = 20.0, first: int = 0):
    """The reference CPU path (oracle restatement, all host threads) on a
    bounded sample of the workload: returns (rays/s, cores, sample text)."""
    from oracle import oracle as orc
    box = CONFIGS[cfg][0]
    m = orc.Mesh.from_files(*fixture(cfg, which))
    cores = orc.num_threads()
    # calibrate on 2^16 rays per part, then size the sample to ~budget_s
    frac = [n for _, n in parts]
    total = sum(frac)
    calib = []
    for mode, n in parts:
        k = min(n, 1 << 16)
        r = orc.raygen(mode, box, SEED, first, k)
        t0 = time.perf_counter()
        m.trace(r)
        calib.append((time.perf_counter() - t0) / k)
    per_ray = sum(c * n for c, n in zip(calib, frac)) / total
    scale = min(1.0, budget_s / max(per_ray * total, 1e-9))
    rays = 0
    t_total = 0.0
    desc = []
    for mode, n in parts:
        k = max(1 << 12, int(n * scale))
        r = orc.raygen(mode, box, SEED, first, k)
        t0 = time.perf_counter()
        m.trace(r)
        t_total += time.perf_counter() - t0
        rays += k
        desc.append(f"{k} {'box-entry' if mode == 0 else 'interior'} rays")
    return rays / t_total, cores, f"{cfg}/{which}: " + " + ".join(desc) + \
        " (oracle locate + walk, OpenMP over all host threads)"


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    box, parts = CONFIGS[args.config]
    vals = []
    sample = ""
    cores = 0
    for _ in range(args.warmup):
        cpu_reference(args.config, args.mesh, parts, budget_s=2.0)
    for _ in range(args.steps):
        v, cores, sample = cpu_reference(args.config, args.mesh, parts, budget_s=args.cpu_budget / max(1, args.steps))
        vals.append(v)
    v = float(np.mean(vals))
    line = {
        "metric": "rays_per_s_mwt_walk", "value": v, "unit": "rays/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded rays, reference-built fixtures)",
        "config": {"workload": f"{args.config}/{args.mesh}",
                   "rays_per_step": {("box_entry" if m == 0 else "interior"): n for m, n in parts}},
        "cpu_baseline": {"value": v, "unit": "rays/s", "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="lines1024", choices=sorted(CONFIGS))
    ap.add_argument("--mesh", default="mwt", choices=["mwt", "cdt"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu)")
    ap.add_argument("--no-extra", action="store_true", help="skip per-config / like-for-like lines")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import DeviceMesh, _stream, new_histogram, summarize_histogram

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
    box, parts = CONFIGS[args.config]
    mesh = DeviceMesh.from_files(*fixture(args.config, args.mesh), device=local)
    rays_per_gpu = sum(n for _, n in parts)
    outs = {mode: dict(seg=torch.empty(n, dtype=torch.int32, device=dev),
                       t=torch.empty(n, dtype=torch.float64, device=dev),
                       steps=torch.empty(n, dtype=torch.int32, device=dev)) for mode, n in parts}
    hist = new_histogram(local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    P = _lib.ptr

    boxarr = np.asarray(box, np.float64)
    sptr = _stream(stream)

    def launch(mode, n, h):
        o = outs[mode]
        _lib.check(_lib.lib.mwt_trace_generated_dev(
            mesh.handle, mode, P(boxarr), SEED, rank * n, n,
            P(o["seg"]), P(o["t"]), P(o["steps"]), P(h), sptr), "trace_generated")

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in parts]

    # the parts run on their own streams, so one part's tail overlaps the next
    # part's start (each kernel keeps one CTA per SM)
    pstreams = [stream] + [torch.cuda.Stream(device=dev) for _ in parts[1:]]
    pptrs = [sptr] + [_stream(ps) for ps in pstreams[1:]]
    zero_done = torch.cuda.Event()

    def launch_on(k, mode, n, h):
        o = outs[mode]
        _lib.check(_lib.lib.mwt_trace_generated_dev(
            mesh.handle, mode, P(boxarr), SEED, rank * n, n,
            P(o["seg"]), P(o["t"]), P(o["steps"]), P(h), pptrs[k]), "trace_generated")

    def step(timed_kernels=None):
        hist.zero_()
        zero_done.record(stream)
        for k, (mode, n) in enumerate(parts):
            ps = pstreams[k]
            if k:
                ps.wait_event(zero_done)
            if timed_kernels is not None:
                ev[k][0].record(ps)
            launch_on(k, mode, n, hist)
            if timed_kernels is not None:
                ev[k][1].record(ps)
        for ps in pstreams[1:]:
            stream.wait_stream(ps)
        if world > 1:
            dist.all_reduce(hist)

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
            step(timed_kernels=True)
            e1.record(stream)
            torch.cuda.synchronize()
            total_ms += e0.elapsed_time(e1)
            for k in range(len(parts)):
                kernel_ms[k] += ev[k][0].elapsed_time(ev[k][1])
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = float(t_local.item())
    ms_per_step = total_ms / args.steps
    value = rays_per_gpu * world / (ms_per_step / 1e3)
    hsum = summarize_histogram(hist)  # last step's (all-reduced) histogram

    # roofline of the dominant kernel (largest part): algorithmic bytes =
    # 32 B x triangle steps it walked (from its own step sum) / its event time
    big = max(range(len(parts)), key=lambda k: parts[k][1])
    hk = new_histogram(local)
    mode_b, n_b = parts[big]
    launch(mode_b, n_b, hk)
    torch.cuda.synchronize()
    hb = summarize_histogram(hk)
    kms = kernel_ms[big] / args.steps
    algo_bytes = hb["steps_sum"] * ALGO_BYTES_PER_STEP
    peak, peak_src = peaks()
    achieved = algo_bytes / (kms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(f"{args.config}/{args.mesh}", {}).get("dram_bytes_per_launch")

    line = {
        "metric": "rays_per_s_mwt_walk", "value": value, "unit": "rays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded on-device rays; reference-built {args.config} scene + "
                f"{'annealed MWT' if args.mesh == 'mwt' else 'CDT'})",
        "parts": [{"rays": ("box_entry" if m == 0 else "interior"), "n": n,
                   "stream_ms": kernel_ms[k] / args.steps} for k, (m, n) in enumerate(parts)],
        "parts_note": "event time on each part's own stream; each persistent launch fills every SM "
                      "(896 threads x 72 registers), so a later part's time includes waiting for the "
                      "SMs the earlier one holds",
        "config": {"workload": f"{args.config}/{args.mesh}",
                   "rays_per_gpu_per_step": {("box_entry" if m == 0 else "interior"): n for m, n in parts},
                   "triangles": mesh.info.num_triangles, "segments": mesh.info.num_segments,
                   "parallelism": f"ray-shard x{world}, mesh replicated",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "steps_per_ray": hsum["steps_per_ray"] if world == 1 else None,
                   "hit_fraction": hsum["hits"] / max(1, hsum["rays"])},
        "gpu_launches": len(parts) * args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_trace (mwt_trace_generated_dev, box-entry launch)", "kernel_ms": kms,
                     "algo_bytes_per_launch": algo_bytes,
                     "algo_bytes_rule": "32 B per triangle step (one 32-B step record: 2 exit words + apex corner)",
                     "peak_source": peak_src, "mesh_resident": "L2 (126 MB); HBM carries only per-ray output",
                     "l2_peak": l2_peak(), "l2_frac": achieved / l2_peak() if l2_peak() else None},
        "histogram": {k: hsum[k] for k in ("rays", "hits", "misses", "steps_sum", "status")},
    }

    # full per-ray byte count of the box-entry launch
    spr = hb["steps_sum"] / max(1, hb["rays"])
    hitf = hb["hits"] / max(1, hb["rays"])
    line["per_ray_bytes"] = {
        "walk_steps": ALGO_BYTES_PER_STEP * spr, "first_triangle": 48.0,
        "boundary_table": 40.0, "output": 16.0, "hit_segment": 32.0 * hitf, "input_ray": 0.0,
        "total": ALGO_BYTES_PER_STEP * spr + 48.0 + 40.0 + 16.0 + 32.0 * hitf,
        "note": "walk = 32 B x steps/ray (the roofline's algorithmic bytes); first triangle = "
                "its three corners; boundary table = bucket word + edge extent + word; "
                "output = seg + t + steps; rays are generated on device"}
    ns = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_ncu_stats.json"))
    if ns:
        with open(os.path.join(ROOT, "profiles", ns[-1])) as fh:
            line["ncu"] = json.load(fh)
    line["clocks"] = clk.summary()
    # the roof that binds this kernel (mesh on chip, one ray per thread): warp
    # instruction issue, 4 per SM per cycle.  Instructions per launch come from
    # the committed ncu capture of the same launch (same build, same rays).
    st_ = line.get("ncu") or {}
    if (args.config, args.mesh) == ("lines1024", "mwt") and st_.get("rays") == n_b and not args.profile:
        sm_mhz = line["clocks"].get("sm_mhz") or line["clocks"].get("sm_max_mhz") or 1965.0
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ach = st_["warp_instructions"] / (kms / 1e3) / 1e9
        pk = sms * 4 * sm_mhz / 1e3
        line["roofline"]["issue_roof"] = {
            "achieved": ach, "peak": pk, "unit": "G warp-inst/s", "frac": ach / pk,
            "warp_inst_per_launch": st_["warp_instructions"], "source": st_.get("report"),
            "note": "4 warp instructions per SM per cycle at the sampled SM clock; the walk's "
                    "records come from shared memory, so issue (not HBM) is the binding roof"}
    if mesh.info.walk_smem_bytes == 0 and not args.profile:
        # walk records from global memory: one L1 data-pipe wavefront per lane
        # per step (scattered 32-B records), one wavefront per SM per cycle
        sm_mhz = line["clocks"].get("sm_mhz") or line["clocks"].get("sm_max_mhz") or 1965.0
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ach = hb["steps_sum"] / (kms / 1e3) / 1e9
        pk = sms * sm_mhz / 1e3
        line["roofline"]["l1_wavefront_roof"] = {
            "achieved": ach, "peak": pk, "unit": "G lane-steps/s", "frac": ach / pk,
            "note": "walk records read from L1/L2 (the mesh does not fit shared memory): each step is "
                    "one scattered 32-B load = one L1 wavefront; the pipe retires one per SM per cycle"}
    line["roofline"]["mesh_resident"] = (
        f"shared memory ({mesh.info.walk_smem_bytes} B compact walk table staged per CTA); "
        "HBM carries only per-ray output" if mesh.info.walk_smem_bytes > 0 else
        "L2 (126 MB); HBM carries only per-ray output")
    if rank == 0 and world == 1 and not args.profile and not args.no_extra:
        line["per_config"] = per_config(local)
        line["like_for_like"] = like_for_like(args.config, local)

    if not args.no_e2e and not args.profile:
        line["e2e"] = e2e(mesh, parts, box, rank, world, args, dev)
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        v, cores, sample = cpu_reference(args.config, args.mesh, parts, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": "rays/s", "cores": cores, "kind": "port",
                                "sample": sample, "cpu_model": cpu_model()}
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


def per_config(local, n=1 << 22):
    """Fused trace (K2+K3+K4+K7) of n box-entry rays on every config's meshes:
    rays/s, steps/ray and where the walk table lives (not the headline)."""
    from paper_2112_05570_b200.engine import DeviceMesh, new_histogram, summarize_histogram
    res = {}
    for cfg, (box, _) in CONFIGS.items():
        for which in ("mwt", "cdt"):
            paths = fixture(cfg, which)
            if not os.path.exists(paths[1]):
                continue
            m = DeviceMesh.from_files(*paths, device=local)
            h = new_histogram(local)
            ms = _time_ms(lambda: m.trace_generated_device(0, box, SEED, 0, n, outputs=True, hist=None))
            m.trace_generated_device(0, box, SEED, 0, n, outputs=False, hist=h)
            import torch
            torch.cuda.synchronize()
            hs = summarize_histogram(h)
            res[f"{cfg}/{which}"] = {"rays": n, "ms": ms, "rays_per_s": n / (ms / 1e3),
                                     "steps_per_ray": hs["steps_per_ray"],
                                     "hit_fraction": hs["hits"] / max(1, hs["rays"]),
                                     "triangles": m.info.num_triangles,
                                     "walk_smem_bytes": int(m.info.walk_smem_bytes)}
            del m
    return res


def like_for_like(cfg, local, n=1 << 22):
    """The same n box-entry rays (loaded from HBM) through the MWT walk, the
    reference-built SAH BVH and roped kd-tree (c_t chosen by the reference rule:
    minimum total ops over the same rays, accel.py:845-862)."""
    import torch
    from paper_2112_05570_b200.engine import DeviceBvh, DeviceKd, DeviceMesh
    from paper_2112_05570_b200.formats import load_structure
    box = CONFIGS[cfg][0]
    d = os.path.join(ROOT, "fixtures", "data", cfg)
    mesh = DeviceMesh.from_files(*fixture(cfg, "mwt"), device=local)
    rays = mesh.raygen_device(0, box, SEED, 0, n)
    out = {}
    ms = _time_ms(lambda: mesh.trace_device(rays, None, want=("seg", "t", "steps")))
    o = mesh.trace_device(rays, None, want=("seg", "steps"))
    out["mwt_walk"] = {"ms": ms, "rays_per_s": n / (ms / 1e3),
                       "ops_per_ray": float(o["steps"].double().mean()), "ops": "tri_steps"}
    for kind, cls in (("bvh", DeviceBvh), ("kd", DeviceKd)):
        files = sorted(f for f in os.listdir(d) if f.startswith(kind + "_ct"))
        if not files:
            continue
        best = None
        for f in files:
            st = cls(mesh, load_structure(os.path.join(d, f)))
            r = st.trace_device(rays)
            keys = ("node_tests", "prim_tests") if kind == "bvh" else ("nodes", "ropes", "prims")
            ops = sum(float(r[k].double().sum()) for k in keys)
            if best is None or ops < best[0]:
                best = (ops, f, st)
        ops, f, st = best
        ms = _time_ms(lambda: st.trace_device(rays))
        out[kind] = {"ms": ms, "rays_per_s": n / (ms / 1e3), "ops_per_ray": ops / n,
                     "c_t": float(st.c_t), "file": f}
    out["rays"] = f"{n} box-entry rays of {cfg}, loaded from HBM (32 B/ray in, seg/t/counters out)"
    return out


def e2e(mesh, parts, box, rank, world, args, dev):
    """Public C-ABI host-buffer call (mwt_trace_host) per step: H2D of the
    step's rays from pinned memory, device locate + walk, D2H of seg/t/u/steps."""
    import torch
    from paper_2112_05570_b200 import _lib
    P = _lib.ptr
    host = []
    for mode, n in parts:
        r = mesh.raygen_device(mode, box, SEED, rank * n, n)
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
    steps = max(3, min(args.steps, 10))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    t = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    nr = sum(n for _, n in parts)
    return {"value": nr * world / dt, "unit": "rays/s", "h2d_bytes_per_step": 32 * nr,
            "d2h_bytes_per_step": 24 * nr, "ms_per_step": dt * 1e3,
            "api": "mwt_trace_host (include/mwt.h), pinned host buffers"}


if __name__ == "__main__":
    main()
