"""Build the five BASELINE configs' input files with the UNMODIFIED reference.

Runs only in the build container (it imports ``mintri`` from
``/root/reference/pkg/src``); its outputs are committed under
``fixtures/data/<config>/`` and travel to the GPU box, which never sees the
reference.  Every output is a pure function of the pinned parameters below.

Per config it writes
  scene.txt      mintri-scene v1   (reference ``Scene.save``, scene.py:62-65)
  cdt.tri        mintri-tri v1     (reference ``build_cdt`` + ``save_triangulation``,
                                    trimesh.py:811-848, :1284-1306)
  mwt.tri        mintri-tri v1     (reference ``full_pipeline`` with the pinned,
                                    deterministic ``PipelineConfig`` below, anneal.py:749-788)
  bvh_ct<c>.npz  flattened reference ``Bvh`` for every c_t in ``C_T_GRID`` (accel.py:373-426)
  kd_ct<c>.npz   flattened reference ``RopedKdTree`` (accel.py:561-710)
and ``manifest.json`` (sha256, parameters, achieved counts).

Scene recipes (BASELINE.json ``configs``) and the crossing policy
-----------------------------------------------------------------
The literal Grass-4096 / Hair-512 recipes produce crossing geometry that the
reference CDT rejects.  Policy (i) is used: each blade/strand
is grown segment by segment; the first segment that touches already-placed
geometry (reference predicate ``segments_cross``, geometry.py:169-198) is cut
back to 90% of the distance to its first contact and ends the polyline, and
a segment that leaves the unit square (then it is clipped with the
reference ``_clip_unit_square``, generators.py:24-45, and ends).  Lines
configs resample a crossing segment (as reference ``gen_lines`` does,
generators.py:71-89).  The achieved segment counts go to the manifest.

Usage:  python fixtures/gen_fixtures.py [config ...]
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from mintri.geometry import Point, Segment, SegmentKind, segments_cross  # noqa: E402
from mintri.scene import Scene, unit_square_boundary  # noqa: E402
from mintri.generators import _clip_unit_square  # noqa: E402
from mintri.trimesh import build_cdt, save_triangulation, load_triangulation  # noqa: E402
from mintri.anneal import PipelineConfig, Schedule, full_pipeline  # noqa: E402
from mintri.accel import C_T_GRID, build_bvh, build_kdtree  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(HERE, "data")


# ----------------------------------------------------------------------
# spatial hash over accepted segments (broad phase only; the narrow phase is
# the reference predicate)

class SegHash:
    def __init__(self, cell: float):
        self.cell = cell
        self.cells: dict[tuple[int, int], list[int]] = {}
        self.segs: list[Segment] = []

    def _range(self, s: Segment):
        tol = 1e-9
        c = self.cell
        x0, x1 = min(s.a.x, s.b.x) - tol, max(s.a.x, s.b.x) + tol
        y0, y1 = min(s.a.y, s.b.y) - tol, max(s.a.y, s.b.y) + tol
        for i in range(int(math.floor(x0 / c)), int(math.floor(x1 / c)) + 1):
            for j in range(int(math.floor(y0 / c)), int(math.floor(y1 / c)) + 1):
                yield (i, j)

    def crosses(self, s: Segment) -> bool:
        seen = set()
        for key in self._range(s):
            for k in self.cells.get(key, ()):
                if k in seen:
                    continue
                seen.add(k)
                if segments_cross(s, self.segs[k]):
                    return True
        return False

    def add(self, s: Segment) -> None:
        k = len(self.segs)
        self.segs.append(s)
        for key in self._range(s):
            self.cells.setdefault(key, []).append(k)


# ----------------------------------------------------------------------
# scene recipes (BASELINE.json configs[0..4])

def scene_lines(n: int, lmin: float, lmax: float, seed: int, name: str) -> Scene:
    rng = np.random.default_rng(seed)
    h = SegHash(0.05)
    budget = 400 * n + 100
    while len(h.segs) < n and budget > 0:
        budget -= 1
        cx, cy = rng.random(), rng.random()
        theta = rng.uniform(0.0, math.pi)
        length = rng.uniform(lmin, lmax)
        hx, hy = 0.5 * length * math.cos(theta), 0.5 * length * math.sin(theta)
        clipped = _clip_unit_square(Point(cx - hx, cy - hy), Point(cx + hx, cy + hy))
        if clipped is None:
            continue
        seg = Segment(*clipped)
        if seg.length < 1e-6 or h.crosses(seg):
            continue
        h.add(seg)
    if len(h.segs) < n:
        raise RuntimeError(f"{name}: placed only {len(h.segs)} of {n}")
    return Scene(h.segs + unit_square_boundary(), name=name,
                 provenance=f"fixtures/gen_fixtures.py scene_lines(n={n}, lengths=U[{lmin},{lmax}], seed={seed})")


def _first_contact(h: SegHash, s: Segment):
    """Smallest parameter along s of a proper crossing with accepted geometry
    (None when the only contacts are touching ones)."""
    best = None
    ax, ay = s.a
    ex, ey = s.b.x - ax, s.b.y - ay
    for key in h._range(s):
        for k in h.cells.get(key, ()):
            t = h.segs[k]
            fx, fy = t.b.x - t.a.x, t.b.y - t.a.y
            den = ex * fy - ey * fx
            if den == 0.0:
                continue
            wx, wy = t.a.x - ax, t.a.y - ay
            u = (wx * fy - wy * fx) / den
            v = (wx * ey - wy * ex) / den
            if -1e-9 <= v <= 1.0 + 1e-9 and 0.0 <= u <= 1.0 and (best is None or u < best):
                best = u
    return best


def _grow(h: SegHash, pts_iter) -> int:
    """Append consecutive polyline segments; the first segment that touches
    accepted geometry is cut back to 90% of the way to its first contact and
    ends the polyline (policy (i), truncate at first contact)."""
    added = 0
    prev = None
    for p in pts_iter:
        if prev is None:
            prev = p
            continue
        a, b = prev, p
        inside = 0.0 <= b.x <= 1.0 and 0.0 <= b.y <= 1.0
        if not inside:
            clipped = _clip_unit_square(a, b)
            if clipped is None or clipped[0] != a:
                break
            b = clipped[1]
        if a == b:
            break
        seg = Segment(a, b)
        truncated = False
        for _ in range(24):
            if seg.length < 1e-6 or not h.crosses(seg):
                break
            truncated = True
            u = _first_contact(h, seg)
            f = 0.5 if u is None else 0.9 * u
            nb = Point(a.x + f * (seg.b.x - a.x), a.y + f * (seg.b.y - a.y))
            if nb == a:
                break
            seg = Segment(a, nb)
        if seg.length < 1e-6 or (truncated and h.crosses(seg)):
            break
        h.add(seg)
        added += 1
        if truncated or not inside:
            break
        prev = seg.b
    return added


def scene_grass(n: int, seed: int, name: str) -> Scene:
    rng = np.random.default_rng(seed)
    h = SegHash(0.02)
    blades = 0
    for _ in range(n):
        x0 = float(rng.random())
        height = float(rng.uniform(0.1, 0.4))
        lean = float(rng.normal(0.0, math.radians(15.0)))
        bends = rng.normal(0.0, math.radians(5.0), size=3)
        step = height / 4.0

        def pts():
            p = Point(x0, 0.0)
            yield p
            phi = lean
            for k in range(4):
                if k > 0:
                    phi += float(bends[k - 1])
                p = Point(p.x + step * math.sin(phi), p.y + step * math.cos(phi))
                yield p
        if _grow(h, pts()):
            blades += 1
    return Scene(h.segs + unit_square_boundary(), name=name,
                 provenance=f"fixtures/gen_fixtures.py scene_grass(n={n}, seed={seed}, "
                            f"policy=cut-at-first-contact, blades_kept={blades})")


def scene_hair(n: int, seed: int, name: str) -> Scene:
    rng = np.random.default_rng(seed)
    h = SegHash(0.02)
    strands = 0
    for _ in range(n):
        alpha = float(rng.uniform(0.0, 2.0 * math.pi))
        turns = rng.normal(0.0, math.radians(10.0), size=31)

        def pts():
            p = Point(0.5 + 0.3 * math.cos(alpha), 0.5 + 0.3 * math.sin(alpha))
            yield p
            heading = alpha
            for k in range(32):
                if k > 0:
                    heading += float(turns[k - 1])
                p = Point(p.x + 0.01 * math.cos(heading), p.y + 0.01 * math.sin(heading))
                yield p
        if _grow(h, pts()):
            strands += 1
    return Scene(h.segs + unit_square_boundary(), name=name,
                 provenance=f"fixtures/gen_fixtures.py scene_hair(n={n}, seed={seed}, "
                            f"policy=cut-at-first-contact, strands_kept={strands})")


def scene_grass_lanes(n: int, seed: int, name: str) -> Scene:
    """Grass-4096 with the reference gen_grass's crossing policy (lane
    confinement, generators.py:113-131): blade k is rooted in lane
    [k/n, (k+1)/n] (x0 uniform in its inner 80%) and every vertex's x is
    clamped to the lane minus a 6% pad, so no two blades can touch and every
    blade keeps its 4 segments; height, base lean N(0, 15 deg) and per-segment
    bend N(0, 5 deg) as the recipe (equal segment lengths before the clamp)."""
    rng = np.random.default_rng(seed)
    h = SegHash(0.02)
    lane = 1.0 / n
    for k in range(n):
        lo, hi = k * lane, (k + 1) * lane
        pad = 0.06 * lane
        x0 = float(rng.uniform(lo + 0.1 * lane, hi - 0.1 * lane))
        height = float(rng.uniform(0.1, 0.4))
        lean = float(rng.normal(0.0, math.radians(15.0)))
        bends = rng.normal(0.0, math.radians(5.0), size=3)
        step = height / 4.0
        p = Point(x0, 0.0)
        phi = lean
        for q in range(4):
            if q > 0:
                phi += float(bends[q - 1])
            nx = min(max(p.x + step * math.sin(phi), lo + pad), hi - pad)
            b = Point(nx, p.y + step * abs(math.cos(phi)))
            seg = Segment(p, b)
            if h.crosses(seg):  # (cannot happen: lanes are disjoint and y grows)
                raise RuntimeError(f"{name}: blade {k} crosses")
            h.add(seg)
            p = b
    return Scene(h.segs + unit_square_boundary(), name=name,
                 provenance=f"fixtures/gen_fixtures.py scene_grass_lanes(n={n}, seed={seed}, "
                            f"policy=lane-confinement (reference gen_grass), blades_kept={n})")


def scene_hair_resample(n: int, seed: int, name: str, tries: int = 32) -> Scene:
    """Hair-512 with a resampling crossing policy: a strand step whose segment
    would touch placed geometry redraws its turning angle (N(0, 10 deg) added
    to the current heading) up to `tries` times, as the reference gen_lines
    redraws a crossing segment (generators.py:71-89); only when every draw
    touches is the step cut at its first contact and the strand ended (the
    policy of scene_hair).  A step leaving the unit square is clipped and ends
    the strand."""
    rng = np.random.default_rng(seed)
    h = SegHash(0.02)
    strands = 0
    for _ in range(n):
        alpha = float(rng.uniform(0.0, 2.0 * math.pi))
        p = Point(0.5 + 0.3 * math.cos(alpha), 0.5 + 0.3 * math.sin(alpha))
        heading = alpha
        added = 0
        for k in range(32):
            seg, end = None, False
            for t in range(tries):
                hd = heading + (float(rng.normal(0.0, math.radians(10.0))) if k > 0 else 0.0)
                b = Point(p.x + 0.01 * math.cos(hd), p.y + 0.01 * math.sin(hd))
                if not (0.0 <= b.x <= 1.0 and 0.0 <= b.y <= 1.0):
                    clipped = _clip_unit_square(p, b)
                    if clipped is None or clipped[0] != p:
                        break
                    b, end = clipped[1], True
                cand = Segment(p, b)
                if cand.length >= 1e-6 and not h.crosses(cand):
                    seg, heading = cand, hd
                    break
                end = False
            if seg is None:
                # every draw touches: cut the last draw at its first contact (scene_hair's rule)
                n_before = len(h.segs)
                _grow(h, iter([p, Point(p.x + 0.01 * math.cos(heading), p.y + 0.01 * math.sin(heading))]))
                added += len(h.segs) - n_before
                break
            h.add(seg)
            added += 1
            p = seg.b
            if end:
                break
        strands += added > 0
    return Scene(h.segs + unit_square_boundary(), name=name,
                 provenance=f"fixtures/gen_fixtures.py scene_hair_resample(n={n}, seed={seed}, "
                            f"policy=resample-turn x{tries} then cut-at-first-contact, strands_kept={strands})")


def scene_floorplan(n: int, seed: int, name: str) -> Scene:
    rng = np.random.default_rng(seed)
    ang = math.radians(30.0)
    ca, sa = math.cos(ang), math.sin(ang)
    # every grid node computed once so shared endpoints are bit-identical
    nodes = {}
    for i in range(n + 1):
        for j in range(n + 1):
            x, y = i / n - 0.5, j / n - 0.5
            nodes[(i, j)] = Point(0.5 + ca * x - sa * y, 0.5 + sa * x + ca * y)
    segs: list[Segment] = []

    def wall(pa: Point, pb: Point, interior: bool) -> None:
        door = interior and rng.random() < 0.5
        if not door:
            segs.append(Segment(pa, pb))
            return
        c = float(rng.uniform(0.15, 0.85))
        u0, u1 = c - 0.15, c + 0.15
        g0 = Point(pa.x + u0 * (pb.x - pa.x), pa.y + u0 * (pb.y - pa.y))
        g1 = Point(pa.x + u1 * (pb.x - pa.x), pa.y + u1 * (pb.y - pa.y))
        if u0 > 0.0:
            segs.append(Segment(pa, g0))
        if u1 < 1.0:
            segs.append(Segment(g1, pb))

    for j in range(n + 1):          # horizontal walls
        for i in range(n):
            wall(nodes[(i, j)], nodes[(i + 1, j)], 0 < j < n)
    for i in range(n + 1):          # vertical walls
        for j in range(n):
            wall(nodes[(i, j)], nodes[(i, j + 1)], 0 < i < n)
    return Scene.from_geometry(segs, name=name, normalize=True, validate=False,
                               provenance=f"fixtures/gen_fixtures.py scene_floorplan(n={n}, seed={seed}, "
                                          f"door_p=0.5, door_width=0.3, rotate=30deg)")


# ----------------------------------------------------------------------
# pinned configs

CONFIGS = {
    "lines64": dict(
        scene=lambda: scene_lines(64, 0.05, 0.2, 0, "lines64"),
        # small enough for the reference's full default refinement sweep and
        # a subdivision iteration (Steiner + on-segment vertices exercised)
        pipeline=dict(levels=20, steps_per_level=100, iterations=2,
                      angle_grid=None, area_grid=None),
        box=(0.0, 0.0, 1.0, 1.0), rays=1 << 20, structures=False),
    "lines1024": dict(
        scene=lambda: scene_lines(1024, 0.01, 0.05, 0, "lines1024"),
        # flip-only annealing: one 20-degree refinement cell of the reference's
        # refine_cdt ran > 60 CPU-minutes here (quadratic encroachment scan,
        # trimesh.py:1114, :1228-1236), so the refinement sweep is pinned off
        pipeline=dict(levels=10, steps_per_level=200, iterations=1,
                      angle_grid=[0.0], area_grid=[math.inf]),
        box=(0.0, 0.0, 1.0, 1.0), rays=1 << 24, structures=True),
    "grass4096": dict(
        scene=lambda: scene_grass(4096, 0, "grass4096"),
        pipeline=dict(levels=4, steps_per_level=200, iterations=1,
                      angle_grid=[0.0], area_grid=[math.inf]),
        box=(0.0, 0.0, 1.0, 0.5), rays=1 << 24, structures=True),
    "hair512": dict(
        scene=lambda: scene_hair(512, 0, "hair512"),
        pipeline=dict(levels=4, steps_per_level=200, iterations=1,
                      angle_grid=[0.0], area_grid=[math.inf]),
        box=(0.0, 0.0, 1.0, 1.0), rays=1 << 24, structures=True),
    # the two recipes above under the other crossing policies:
    # every blade keeps its 4 segments / strands steer around contacts
    "grass4096l": dict(
        scene=lambda: scene_grass_lanes(4096, 0, "grass4096l"),
        pipeline=dict(levels=4, steps_per_level=200, iterations=1,
                      angle_grid=[0.0], area_grid=[math.inf]),
        box=(0.0, 0.0, 1.0, 0.5), rays=1 << 24, structures=True),
    "hair512r": dict(
        scene=lambda: scene_hair_resample(512, 0, "hair512r"),
        pipeline=dict(levels=4, steps_per_level=200, iterations=1,
                      angle_grid=[0.0], area_grid=[math.inf]),
        box=(0.0, 0.0, 1.0, 1.0), rays=1 << 24, structures=True),
    "floorplan64": dict(
        scene=lambda: scene_floorplan(64, 0, "floorplan64"),
        pipeline=dict(levels=4, steps_per_level=200, iterations=1,
                      angle_grid=[0.0], area_grid=[math.inf]),
        box=(0.0, 0.0, 1.0, 1.0), rays=1 << 26, structures=True),
}


def sha256(path: str) -> str:
    hsh = hashlib.sha256()
    with open(path, "rb") as fh:
        hsh.update(fh.read())
    return hsh.hexdigest()


def flatten_bvh(bvh) -> dict:
    """DFS preorder; children stored as node indices, leaves as prim ranges."""
    boxes, left, right, poff, pcnt, prims = [], [], [], [], [], []

    def rec(node) -> int:
        k = len(boxes)
        boxes.append(node.box)
        left.append(-1); right.append(-1); poff.append(0); pcnt.append(0)
        if node.is_leaf:
            poff[k] = len(prims)
            pcnt[k] = len(node.prims)
            prims.extend(node.prims)
        else:
            left[k] = rec(node.left)
            right[k] = rec(node.right)
        return k

    sys.setrecursionlimit(100000)
    rec(bvh.root)
    return dict(format=np.array("mwt-bvh v1"), c_t=np.float64(bvh.c_t),
                box=np.array(boxes, dtype=np.float64).reshape(-1, 4),
                left=np.array(left, dtype=np.int32), right=np.array(right, dtype=np.int32),
                prim_off=np.array(poff, dtype=np.int32), prim_cnt=np.array(pcnt, dtype=np.int32),
                prims=np.array(prims, dtype=np.int32))


def flatten_kd(kd) -> dict:
    """DFS preorder node table; leaves carry box, prim range, ropes (node
    index or -1), rope counts and the reference rope cost
    max(1, ceil(log2(count))) evaluated with Python semantics (accel.py:818)."""
    nodes = []
    index = {}

    def rec(node) -> int:
        k = len(nodes)
        nodes.append(node)
        index[id(node)] = k
        if not node.is_leaf:
            rec(node.left)
            rec(node.right)
        return k

    sys.setrecursionlimit(100000)
    rec(kd.root)
    n = len(nodes)
    axis = np.full(n, -1, np.int32)
    pos = np.zeros(n, np.float64)
    left = np.full(n, -1, np.int32)
    right = np.full(n, -1, np.int32)
    box = np.zeros((n, 4), np.float64)
    ropes = np.full((n, 4), -1, np.int32)
    counts = np.zeros((n, 4), np.int32)
    cost = np.zeros((n, 4), np.int32)
    poff = np.zeros(n, np.int32)
    pcnt = np.zeros(n, np.int32)
    prims: list[int] = []
    for k, node in enumerate(nodes):
        box[k] = node.box
        if node.is_leaf:
            poff[k] = len(prims)
            pcnt[k] = len(node.prims)
            prims.extend(node.prims)
            for s in range(4):
                r = node.ropes[s]
                ropes[k, s] = -1 if r is None else index[id(r)]
                counts[k, s] = node.rope_counts[s]
                if r is not None:
                    cost[k, s] = max(1, math.ceil(math.log2(node.rope_counts[s])))
        else:
            axis[k] = node.axis
            pos[k] = node.pos
            left[k] = index[id(node.left)]
            right[k] = index[id(node.right)]
    return dict(format=np.array("mwt-kd v1"), c_t=np.float64(kd.c_t),
                num_leaves=np.int64(len(kd._leaves)),
                axis=axis, pos=pos, left=left, right=right, box=box, ropes=ropes,
                rope_counts=counts, rope_cost=cost, prim_off=poff, prim_cnt=pcnt,
                prims=np.array(prims, dtype=np.int32))


def build(name: str) -> None:
    cfg = CONFIGS[name]
    out = os.path.join(DATA, name)
    os.makedirs(out, exist_ok=True)
    entry: dict = {"box": cfg["box"], "rays": cfg["rays"]}
    t0 = time.time()
    scene = cfg["scene"]()
    scene.validate()
    scene.save(os.path.join(out, "scene.txt"))
    entry["segments_geometry"] = len(scene.geometry)
    entry["provenance"] = scene.provenance
    entry["t_scene_s"] = round(time.time() - t0, 2)
    print(f"[{name}] scene: {len(scene.geometry)} segments ({entry['t_scene_s']} s)", flush=True)

    t0 = time.time()
    cdt = build_cdt(scene)
    assert cdt.validate_topology() == []
    save_triangulation(cdt, os.path.join(out, "cdt.tri"))
    entry["cdt"] = {"triangles": cdt.num_tris, "vertices": cdt.num_verts,
                    "length": cdt.total_edge_length(), "t_s": round(time.time() - t0, 2)}
    print(f"[{name}] cdt: {cdt.num_tris} tris ({entry['cdt']['t_s']} s)", flush=True)

    p = cfg["pipeline"]
    pc = PipelineConfig(schedule=Schedule(levels=p["levels"], steps_per_level=p["steps_per_level"]),
                        iterations=p["iterations"], seed=0,
                        angle_grid=p["angle_grid"], area_grid=p["area_grid"])
    t0 = time.time()
    res = full_pipeline(scene, pc)
    mwt = res.triangulation
    assert mwt.validate_topology() == []
    path = os.path.join(out, "mwt.tri")
    save_triangulation(mwt, path)
    mwt2 = load_triangulation(path, scene)
    assert mwt2.validate_topology() == []
    entry["mwt"] = {"triangles": mwt.num_tris, "vertices": mwt.num_verts,
                    "length": mwt.total_edge_length(), "lengths": res.lengths,
                    "pipeline": {k: (v if not isinstance(v, list) else
                                     [x if math.isfinite(x) else "inf" for x in v])
                                 for k, v in p.items()},
                    "t_s": round(time.time() - t0, 2)}
    print(f"[{name}] mwt: {mwt.num_tris} tris, length {res.lengths} ({entry['mwt']['t_s']} s)",
          flush=True)

    if cfg["structures"]:
        t0 = time.time()
        for c_t in C_T_GRID:
            np.savez_compressed(os.path.join(out, f"bvh_ct{c_t:g}.npz"),
                                **flatten_bvh(build_bvh(scene, c_t)))
            np.savez_compressed(os.path.join(out, f"kd_ct{c_t:g}.npz"),
                                **flatten_kd(build_kdtree(scene, c_t)))
        entry["t_structures_s"] = round(time.time() - t0, 2)
        print(f"[{name}] structures ({entry['t_structures_s']} s)", flush=True)

    entry["files"] = {f: sha256(os.path.join(out, f)) for f in sorted(os.listdir(out))
                      if f != "manifest.json"}
    with open(os.path.join(out, "manifest.json"), "w") as fh:
        json.dump(entry, fh, indent=1, sort_keys=True)


def main(argv: list[str]) -> None:
    for name in argv or list(CONFIGS):
        build(name)


if __name__ == "__main__":
    main(sys.argv[1:])
