"""Experiment harness on the device engines, mirroring the reference's
experiment.py:

  sample_rays(scene, count, seed, triangulation=None)    experiment.py:29-63
  run_experiment(scene, triangulations, rays, labels, ct_grid, builders)
                                                         experiment.py:144-202
  ExperimentReport.to_json / to_csv, MethodStats          experiment.py:66-124
  _check hit equality (HitMismatchError)                  experiment.py:131-141

Every ray of every engine runs on the GPU; the brute-force oracle hits are
computed on the GPU too (k_brute).  The c_t sweep traces the SAME rays
through one structure per c_t and keeps the first minimum (strict '<',
accel.py:845-862).  Structures are built by the caller's builders (the
reference's build_bvh / build_kdtree by default when mintri is importable) or
passed pre-flattened ({c_t: arrays}, fixtures/data/*/bvh_ct*.npz).
"""
from __future__ import annotations

import csv
import io
import json
import math
import time
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import accel
from .engine import DeviceBvh, DeviceKd
from .geometry import Point, Ray

COUNTER_FIELDS = ("tri_steps", "bvh_node_tests", "bvh_prim_tests",
                  "kd_nodes_visited", "kd_rope_steps", "kd_prim_tests")


class HitMismatchError(AssertionError):
    pass


# ----------------------------------------------------------------------
# ray sampling (the reference's distribution, bit-identical)

def _segment_arrays(scene):
    a = accel.scene_arrays(scene)
    ax, ay = a.xy[:, 0], a.xy[:, 1]
    ex, ey = a.xy[:, 2] - a.xy[:, 0], a.xy[:, 3] - a.xy[:, 1]
    return ax, ay, ex, ey


def sample_rays_array(scene, count: int, seed: int = 0) -> np.ndarray:
    """(count, 4) rays of experiment.py:29-63: numpy default_rng(seed) origins
    in the unit square, rejecting any within 1e-9 of a segment (same
    expression, row-chunked to bound memory), then theta ~ U[0, 2pi) and a
    direction (math.cos, math.sin) -- libm, as the reference."""
    if count < 1:
        raise ValueError("count must be >= 1")
    rng = np.random.default_rng(seed)
    ax, ay, ex, ey = _segment_arrays(scene)
    ee = ex * ex + ey * ey
    xs_ok, ys_ok = [], []
    have = 0
    while have < count:
        m = count - have
        xs = rng.random(m)
        ys = rng.random(m)
        keep = np.empty(m, dtype=bool)
        step = max(1, (1 << 22) // max(1, len(ax)))
        for lo in range(0, m, step):
            px = xs[lo:lo + step, None] - ax[None, :]
            py = ys[lo:lo + step, None] - ay[None, :]
            u = np.clip((px * ex[None, :] + py * ey[None, :]) / ee[None, :], 0.0, 1.0)
            d2 = (px - u * ex[None, :]) ** 2 + (py - u * ey[None, :]) ** 2
            keep[lo:lo + step] = np.sqrt(d2.min(axis=1)) > 1e-9
        xs_ok.append(xs[keep])
        ys_ok.append(ys[keep])
        have += int(keep.sum())
    ox = np.concatenate(xs_ok)[:count]
    oy = np.concatenate(ys_ok)[:count]
    thetas = rng.uniform(0.0, 2.0 * math.pi, size=count)
    d = np.array([(math.cos(t), math.sin(t)) for t in thetas.tolist()], dtype=np.float64)
    out = np.empty((count, 4), dtype=np.float64)
    out[:, 0], out[:, 1], out[:, 2:] = ox, oy, d
    return out


def sample_rays(scene, count: int, seed: int = 0, triangulation=None) -> list:
    """experiment.py:29-63 (start triangles located on the device)."""
    arr = sample_rays_array(scene, count, seed)
    rays = [Ray(Point(a, b), Point(c, d)) for a, b, c, d in arr.tolist()]
    if triangulation is not None:
        tids, _ = accel.locate_batch(triangulation, arr[:, :2])
        for ray, t in zip(rays, tids.tolist()):
            ray.start_tri = int(t)
    return rays


# ----------------------------------------------------------------------
# report (experiment.py:66-124)

@dataclass
class MethodStats:
    method: str
    label: str
    totals: dict
    ray_count: int
    extra: dict = field(default_factory=dict)

    @property
    def total_ops(self) -> int:
        return sum(self.totals.values())

    @property
    def mean_total(self) -> float:
        return self.total_ops / self.ray_count

    @property
    def means(self) -> dict:
        return {k: v / self.ray_count for k, v in self.totals.items()}


@dataclass
class ExperimentReport:
    scene_name: str
    ray_count: int
    methods: list
    edge_lengths: dict
    timing: dict
    config: dict

    def to_json(self) -> str:
        payload = {
            "scene": self.scene_name, "ray_count": self.ray_count,
            "edge_lengths": self.edge_lengths, "timing": self.timing, "config": self.config,
            "methods": [{"method": m.method, "label": m.label, "totals": m.totals,
                         "total_ops": m.total_ops, "mean_total": m.mean_total, "means": m.means,
                         **m.extra} for m in self.methods],
        }
        return json.dumps(payload, indent=2, sort_keys=True)

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf)
        w.writerow(["scene", "method", "label", "rays", *COUNTER_FIELDS, "total_ops", "mean_total"])
        for m in self.methods:
            w.writerow([self.scene_name, m.method, m.label, m.ray_count,
                        *(m.totals.get(k, 0) for k in COUNTER_FIELDS), m.total_ops,
                        f"{m.mean_total:.6f}"])
        return buf.getvalue()


def _nonzero(totals: dict) -> dict:
    return {k: int(v) for k, v in totals.items() if v}


def check_hits(scene_name: str, method: str, rays: np.ndarray, seg, t, oracle_seg, oracle_t) -> None:
    """experiment.py:131-141 over whole arrays: same presence, same segment,
    |t - t_oracle| <= 1e-9 * max(1, |t_oracle|)."""
    seg, oseg = np.asarray(seg), np.asarray(oracle_seg)
    bad = np.nonzero((seg >= 0) != (oseg >= 0))[0]
    if len(bad):
        k = int(bad[0])
        raise HitMismatchError(f"{scene_name}/{method}: hit presence mismatch for ray {rays[k].tolist()}: "
                               f"seg {int(seg[k])} vs oracle {int(oseg[k])}")
    hit = oseg >= 0
    tol = 1e-9 * np.maximum(1.0, np.abs(oracle_t))
    bad = np.nonzero(hit & ((seg != oseg) | (np.abs(np.asarray(t) - oracle_t) > tol)))[0]
    if len(bad):
        k = int(bad[0])
        raise HitMismatchError(f"{scene_name}/{method}: ray {rays[k].tolist()} hit seg {int(seg[k])} "
                               f"t={float(t[k])!r} but oracle seg {int(oseg[k])} t={float(oracle_t[k])!r}")


def total_edge_length(tri) -> float:
    """Triangulation.total_edge_length (trimesh.py:246-251): unique edges, in
    iter_edges order (trimesh.py:184-193), summed with math.hypot."""
    if hasattr(tri, "total_edge_length"):
        return tri.total_edge_length()
    total = 0.0
    for tid, t in enumerate(tri.tris):
        if t is None:
            continue
        for i in range(3):
            n = t.nbr[i]
            if n is None or tid < n:
                a, b = tri.verts[t.v[(i + 1) % 3]], tri.verts[t.v[(i + 2) % 3]]
                total += math.hypot(b.x - a.x, b.y - a.y)
    return total


def _default_builders():
    try:
        from mintri.accel import build_bvh, build_kdtree  # the reference's own builders
    except Exception:  # pragma: no cover - mintri absent
        return None
    return {"bvh": build_bvh, "kd": build_kdtree}


def _sweep(kind: str, scene, rays: np.ndarray, ct_grid, builders, structures):
    """accel.py:845-862 on the device: totals per c_t over the same rays, first minimum."""
    from .accel import _scene_mesh, flatten_bvh, flatten_kd
    mesh = _scene_mesh(scene)
    totals, best = {}, None
    for c_t in ct_grid:
        if structures is not None and c_t in structures:
            arrays = structures[c_t]
        elif builders is not None:
            obj = builders[kind](scene, c_t)
            arrays = flatten_bvh(obj) if kind == "bvh" else flatten_kd(obj)
        else:
            raise ValueError(f"no {kind} builder or structure for c_t={c_t}")
        dev = DeviceBvh(mesh, arrays) if kind == "bvh" else DeviceKd(mesh, arrays)
        o = dev.trace(rays)
        if kind == "bvh":
            tot = {"bvh_node_tests": int(o["node_tests"].astype(np.int64).sum()),
                   "bvh_prim_tests": int(o["prim_tests"].astype(np.int64).sum())}
        else:
            if (o["status"].view(np.uint32) & 1).any():
                raise accel.TraversalError("kd walk did not terminate")
            tot = {"kd_nodes_visited": int(o["nodes"].astype(np.int64).sum()),
                   "kd_rope_steps": int(o["ropes"].astype(np.int64).sum()),
                   "kd_prim_tests": int(o["prims"].astype(np.int64).sum())}
        total = sum(tot.values())
        totals[c_t] = total
        if best is None or total < best[0]:
            best = (total, c_t, tot, o)
    return best, totals


def run_experiment(scene, triangulations: Sequence, rays, labels: Optional[Sequence[str]] = None,
                   ct_grid: Iterable[float] = accel.C_T_GRID, builders: Optional[dict] = None,
                   bvh_structures: Optional[dict] = None,
                   kd_structures: Optional[dict] = None) -> ExperimentReport:
    """experiment.py:144-202 with every per-ray loop on the device."""
    ct_grid = list(ct_grid)
    labels = list(labels) if labels is not None else [f"tri{k}" for k in range(len(triangulations))]
    r = accel._ray_array(rays)
    n = len(r)
    name = getattr(scene, "name", "scene")
    timing: dict = {}
    t0 = time.perf_counter()
    oracle = accel._scene_mesh(scene).brute_force(r)
    timing["oracle"] = time.perf_counter() - t0
    methods, edge_lengths = [], {}
    for label, tri in zip(labels, triangulations):
        edge_lengths[label] = total_edge_length(tri)
        t0 = time.perf_counter()
        out = accel.trace_batch(tri, r)  # start triangles located per triangulation
        if (out["status"] & (1 | 1024)).any():
            raise accel.TraversalError("traversal failed on the device")
        check_hits(name, f"triangulation[{label}]", r, out["seg"], out["t"], oracle["seg"], oracle["t"])
        timing[f"triangulation[{label}]"] = time.perf_counter() - t0
        methods.append(MethodStats("triangulation", label,
                                   _nonzero({"tri_steps": int(out["steps"].astype(np.int64).sum())}), n))
    if builders is None and (bvh_structures is None or kd_structures is None):
        builders = _default_builders()
    for kind, structs in (("bvh", bvh_structures), ("kd", kd_structures)):
        t0 = time.perf_counter()
        (total, c_t, tot, o), totals = _sweep(kind, scene, r, ct_grid, builders, structs)
        timing[f"{kind}_sweep"] = time.perf_counter() - t0
        check_hits(name, kind, r, o["seg"], o["t"], oracle["seg"], oracle["t"])
        methods.append(MethodStats(kind, f"c_t={c_t:g}", _nonzero(tot), n,
                                   extra={"sweep_totals": {str(k): v for k, v in totals.items()}}))
    return ExperimentReport(name, n, methods, edge_lengths, timing, {"ct_grid": ct_grid})
