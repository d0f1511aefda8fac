"""Generate the golden vectors that pin the oracle (and the engine) to the
reference.  Runs ONLY in the build container: it imports the unmodified
reference package from /root/reference/pkg/src (and its test helpers from
/root/reference/pkg/tests/conftest.py) and records what the reference itself
returns.  Outputs (committed): tests/golden/*.npz.

  known.npz     hand-built and reference-test cases (test_accel.py, test_geometry.py)
  config_<c>.npz  per BASELINE config: rays, reference start/seg/t/u/steps on cdt & mwt
  struct_<c>.npz  per config: reference bvh/kd results + counters on a ray subset
  hypot.npz     math.hypot values (CPython's is correctly rounded)
  degenerate.npz  rays where the reference walk and brute force disagree
  kdstart.npz   kd_intersect from given start leaves (accel.py:761-771)
  branches.npz  hand-built inputs forcing the walk's fallback / TraversalError /
                parallel-exit branches and outside-the-mesh locates

Usage: python tests/golden/make_golden.py [group ...]
"""
from __future__ import annotations

import json
import math
import os
import random
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = ["/root/reference/pkg/src", "/root/reference/pkg/tests", ROOT]

from mintri.geometry import Point, Ray, Segment, ray_segment_intersect  # noqa: E402
from mintri.scene import Scene  # noqa: E402
from mintri.trimesh import build_cdt, load_triangulation, refine_cdt, save_triangulation  # noqa: E402
from mintri.accel import (SceneIndex, TraversalError, TriLocator, brute_force_closest,  # noqa: E402
                          build_bvh, build_kdtree, bvh_intersect, kd_intersect,
                          locate_triangle, traverse_triangulation)
from mintri.experiment import sample_rays  # noqa: E402
from conftest import random_segment_scene  # noqa: E402  (reference tests/conftest.py:10-42)

from oracle.raygen import raygen  # noqa: E402

CONFIGS = ["lines64", "lines1024", "grass4096", "hair512", "floorplan64", "grass4096l", "hair512r"]
BOXES = {"grass4096": (0.0, 0.0, 1.0, 0.5), "grass4096l": (0.0, 0.0, 1.0, 0.5)}
FIX = os.path.join(ROOT, "fixtures", "data")


def roundtrip(tri):
    """save + load: compact ids exactly as the engine and oracle see them."""
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.tri")
        save_triangulation(tri, p)
        return load_triangulation(p, tri.scene)


def scene_arrays(scene):
    xy = np.array([[s.a.x, s.a.y, s.b.x, s.b.y] for s in scene.segments], np.float64).reshape(-1, 4)
    kind = np.array([0 if s.kind.value == "G" else 1 for s in scene.segments], np.uint8)
    return xy, kind


def tri_arrays(tri):
    vxy = np.array([[v.x, v.y] for v in tri.verts], np.float64).reshape(-1, 2)
    v = np.array([t.v for t in tri.tris], np.int32).reshape(-1, 3)
    nbr = np.array([[-1 if n is None else n for n in t.nbr] for t in tri.tris], np.int32).reshape(-1, 3)
    flag = np.array([t.flag for t in tri.tris], np.int32).reshape(-1, 3)
    return vxy, v, nbr, flag


def ray_arr(rays):
    return np.array([[r.origin.x, r.origin.y, r.direction.x, r.direction.y] for r in rays],
                    np.float64).reshape(-1, 4)


def run_walk(tri, rays, starts=None, index=None):
    """Reference TriLocator.locate + traverse_triangulation per ray."""
    index = index or SceneIndex(tri.scene)
    loc = TriLocator(tri)
    n = len(rays)
    out = dict(start=np.empty(n, np.int32), seg=np.full(n, -1, np.int32), t=np.full(n, np.nan),
               u=np.full(n, np.nan), steps=np.zeros(n, np.int32), error=np.zeros(n, np.uint8))
    for i, r in enumerate(rays):
        s = loc.locate(r.origin) if starts is None else int(starts[i])
        out["start"][i] = s
        try:
            hit, st = traverse_triangulation(tri, r, s, index)
        except TraversalError:
            out["error"][i] = 1
            continue
        out["steps"][i] = st.tri_steps
        if hit is not None:
            out["seg"][i] = hit.seg
            out["t"][i] = hit.t
            seg = tri.scene.segments[hit.seg]
            # recover u from the hit point (point_at(u) is what the reference stores)
            ex, ey = seg.b.x - seg.a.x, seg.b.y - seg.a.y
            out["u"][i] = ((hit.point.x - seg.a.x) * ex + (hit.point.y - seg.a.y) * ey) / (ex * ex + ey * ey)
    return out


def prefixed(prefix, d):
    return {f"{prefix}{k}": v for k, v in d.items()}


def rays_from(arr):
    return [Ray(Point(float(a), float(b)), Point(float(c), float(d))) for a, b, c, d in arr]


# ----------------------------------------------------------------------

def make_known():
    out = {}
    cases = []

    # test_accel.py:40-44 empty square
    sc = Scene.from_geometry([], name="empty")
    cases.append(("empty", sc, [Ray(Point(0.5, 0.5), Point(1, 0)), Ray(Point(0.25, 0.75), Point(0.6, -0.8))]))
    # test_accel.py:62-71 ray through a shared vertex
    sc = Scene.from_geometry([Segment(Point(0.5, 0.5), Point(0.75, 0.85)),
                              Segment(Point(0.5, 0.5), Point(0.75, 0.15))], normalize=False)
    cases.append(("shared_vertex", sc, [Ray(Point(0.2, 0.5), Point(1, 0)),
                                        Ray(Point(0.2, 0.5), Point(0.6, 0.8)),
                                        Ray(Point(0.9, 0.5), Point(-1, 0))]))
    # test_accel.py:31-37 tie at a joint (lowest id)
    sc = Scene.from_geometry([Segment(Point(0.5, 0.5), Point(0.7, 0.8)),
                              Segment(Point(0.5, 0.5), Point(0.7, 0.2))], normalize=False)
    cases.append(("tie_lowest_id", sc, [Ray(Point(0.1, 0.5), Point(1, 0))]))
    # polyline joint hit from the higher-id side + ray along an edge + collinear segment
    sc = Scene.from_geometry([Segment(Point(0.3, 0.6), Point(0.5, 0.4)),
                              Segment(Point(0.5, 0.4), Point(0.7, 0.6)),
                              Segment(Point(0.2, 0.2), Point(0.8, 0.2)),
                              Segment(Point(0.1, 0.85), Point(0.4, 0.85))], normalize=False)
    cases.append(("joint_and_collinear", sc, [
        Ray(Point(0.5, 0.05), Point(0, 1)),              # through the joint (0.5, 0.4)
        Ray(Point(0.9, 0.4), Point(-1, 0)),              # horizontal through the joint
        Ray(Point(0.05, 0.2), Point(1, 0)),              # collinear with segment 2
        Ray(Point(0.95, 0.2), Point(-1, 0)),             # collinear, from the other side
        Ray(Point(0.05, 0.85), Point(1, 0)),             # collinear with segment 3
        Ray(Point(0.5, 0.5), Point(0, -1)),              # straight down onto the joint
        Ray(Point(0.0, 0.0), Point(1, 1)),               # from the corner (box vertex)
        Ray(Point(1.0, 0.5), Point(-1, 0)),              # from the boundary
    ]))
    # reference test scene (test_accel.py:47-59)
    sc = random_segment_scene(25, seed=70)
    cases.append(("random25", sc, sample_rays(sc, 1500, seed=1)))
    # a refined mesh (Steiner + on-segment vertices, test_accel.py:74-81)
    sc = random_segment_scene(15, seed=71)
    cases.append(("refined15", sc, sample_rays(sc, 1500, seed=2)))

    names = []
    for name, sc, rays in cases:
        tri = build_cdt(sc) if name != "refined15" else refine_cdt(build_cdt(sc), 20.0, 0.05)
        tri = roundtrip(tri)
        xy, kind = scene_arrays(sc)
        vxy, v, nbr, flag = tri_arrays(tri)
        r = ray_arr(rays)
        walk = run_walk(tri, rays)
        idx = SceneIndex(sc)
        bf = [brute_force_closest(sc, ray, idx) for ray in rays]
        d = dict(seg_xy=xy, seg_kind=kind, vxy=vxy, v=v, nbr=nbr, flag=flag, rays=r,
                 bf_seg=np.array([-1 if h is None else h.seg for h in bf], np.int32),
                 bf_t=np.array([np.nan if h is None else h.t for h in bf]))
        d.update(prefixed("w_", walk))
        # point location: brute vs anchor on origins, centroids and shared-edge midpoints
        pts = [r_.origin for r_ in rays]
        for tid in range(len(tri.tris)):
            vv = tri.tris[tid].v
            pts.append(Point(sum(tri.pos(k).x for k in vv) / 3, sum(tri.pos(k).y for k in vv) / 3))
        for tid, i, a, b in tri.iter_edges():
            pa, pb = tri.pos(a), tri.pos(b)
            pts.append(Point((pa.x + pb.x) / 2, (pa.y + pb.y) / 2))
        pts.extend(tri.pos(k) for k in range(len(tri.verts)))  # exact vertices (fan ties)
        loc = TriLocator(tri)
        d["loc_pts"] = np.array(pts, np.float64).reshape(-1, 2)
        d["loc_anchor"] = np.array([loc.locate(p) for p in pts], np.int32)
        d["loc_brute"] = np.array([locate_triangle(tri, p, "brute") for p in pts], np.int32)
        out.update(prefixed(f"{name}__", d))
        names.append(name)
        print(f"known/{name}: {len(rays)} rays, {len(pts)} points", flush=True)
    out["cases"] = np.array(names)

    # geometry.py:136-166 against random cases (test_geometry.py:92-119 style)
    rng = random.Random(42)
    rs, ss, res = [], [], []
    for _ in range(20000):
        o = Point(rng.uniform(-1, 1), rng.uniform(-1, 1))
        th = rng.uniform(0, 2 * math.pi)
        ray = Ray(o, Point(math.cos(th), math.sin(th)))
        a = Point(rng.uniform(-1, 1), rng.uniform(-1, 1))
        b = Point(rng.uniform(-1, 1), rng.uniform(-1, 1))
        if a == b:
            continue
        h = ray_segment_intersect(ray, Segment(a, b))
        rs.append([ray.origin.x, ray.origin.y, ray.direction.x, ray.direction.y])
        ss.append([a.x, a.y, b.x, b.y])
        res.append([np.nan, np.nan] if h is None else [h[0], h[1]])
    # degenerate: parallel / collinear (test_geometry.py:78-89)
    for (ox, oy, dx, dy), (ax, ay, bx, by) in [((0, 0, 1, 0), (2, 0, 5, 0)), ((0, 0, 1, 0), (5, 0, 2, 0)),
                                               ((0, 0, 1, 0), (-5, 0, -2, 0)), ((0, 0, 1, 0), (-1, 0, 3, 0)),
                                               ((0, 0, 1, 0), (0.5, -1, 0.5, 1)), ((0, 0, 1, 0), (0.5, 1, 1.5, 1)),
                                               ((0, 0, 0.6, 0.8), (0, 1, 1, 0))]:
        ray = Ray(Point(ox, oy), Point(dx, dy))
        h = ray_segment_intersect(ray, Segment(Point(ax, ay), Point(bx, by)))
        rs.append([ray.origin.x, ray.origin.y, ray.direction.x, ray.direction.y])
        ss.append([ax, ay, bx, by])
        res.append([np.nan, np.nan] if h is None else [h[0], h[1]])
    out["rsi_rays"] = np.array(rs, np.float64)
    out["rsi_segs"] = np.array(ss, np.float64)
    out["rsi_tu"] = np.array(res, np.float64)
    np.savez_compressed(os.path.join(HERE, "known.npz"), **out)


def make_hypot():
    rng = np.random.default_rng(5)
    n = 200000
    x = rng.uniform(-1, 1, n) * 10.0 ** rng.uniform(-12, 2, n)
    y = rng.uniform(-1, 1, n) * 10.0 ** rng.uniform(-12, 2, n)
    y[:1000] = 0.0
    x[1000:2000] = y[1000:2000]
    h = np.array([math.hypot(a, b) for a, b in zip(x.tolist(), y.tolist())])
    np.savez_compressed(os.path.join(HERE, "hypot.npz"), x=x, y=y, h=h)


def make_config(cfg, nrays=4096):
    d = os.path.join(FIX, cfg)
    scene = Scene.load(os.path.join(d, "scene.txt"))
    index = SceneIndex(scene)
    box = BOXES.get(cfg, (0.0, 0.0, 1.0, 1.0))
    out = {}
    modes = [0, 1] if cfg in ("lines1024", "lines64") else [0]
    for mode in modes:
        arr = raygen(mode, box, 0, 0, nrays)
        out[f"rays{mode}"] = arr
        rays = rays_from(arr)
        for which in ("cdt", "mwt"):
            p = os.path.join(d, f"{which}.tri")
            if not os.path.exists(p):
                continue
            tri = load_triangulation(p, scene)
            w = run_walk(tri, rays, index=index)
            out.update(prefixed(f"{which}{mode}_", w))
            print(f"{cfg}/{which}/mode{mode}: steps {w['steps'].mean():.3f} hit {(w['seg'] >= 0).mean():.3f}",
                  flush=True)
        bf = [brute_force_closest(scene, r, index) for r in rays[:1024]]
        out[f"bf{mode}_seg"] = np.array([-1 if h is None else h.seg for h in bf], np.int32)
        out[f"bf{mode}_t"] = np.array([np.nan if h is None else h.t for h in bf])
    np.savez_compressed(os.path.join(HERE, f"config_{cfg}.npz"), **out)


def make_struct(cfg, nrays=1024):
    from mintri.accel import C_T_GRID
    d = os.path.join(FIX, cfg)
    scene = Scene.load(os.path.join(d, "scene.txt"))
    box = BOXES.get(cfg, (0.0, 0.0, 1.0, 1.0))
    out = {}
    for mode in (0, 1):
        arr = raygen(mode, box, 0, 0, nrays)
        out[f"rays{mode}"] = arr
        rays = rays_from(arr)
        grid = C_T_GRID if cfg == "lines1024" else (1.0,)
        for c_t in grid:
            bvh = build_bvh(scene, c_t)
            kd = build_kdtree(scene, c_t)
            rb = [bvh_intersect(bvh, r) for r in rays]
            rk = []
            for r in rays:
                try:
                    rk.append(kd_intersect(kd, r))
                except TraversalError:
                    rk.append((None, None))
            tag = f"{mode}_ct{c_t:g}"
            out[f"bvh{tag}_seg"] = np.array([-1 if h is None else h.seg for h, _ in rb], np.int32)
            out[f"bvh{tag}_t"] = np.array([np.nan if h is None else h.t for h, _ in rb])
            out[f"bvh{tag}_nodes"] = np.array([s.bvh_node_tests for _, s in rb], np.int32)
            out[f"bvh{tag}_prims"] = np.array([s.bvh_prim_tests for _, s in rb], np.int32)
            out[f"kd{tag}_seg"] = np.array([-1 if h is None else h.seg for h, _ in rk], np.int32)
            out[f"kd{tag}_t"] = np.array([np.nan if h is None else h.t for h, _ in rk])
            out[f"kd{tag}_nodes"] = np.array([-1 if s is None else s.kd_nodes_visited for _, s in rk], np.int32)
            out[f"kd{tag}_ropes"] = np.array([-1 if s is None else s.kd_rope_steps for _, s in rk], np.int32)
            out[f"kd{tag}_prims"] = np.array([-1 if s is None else s.kd_prim_tests for _, s in rk], np.int32)
            print(f"struct {cfg} mode{mode} c_t={c_t}: bvh ops {np.mean(out[f'bvh{tag}_nodes'] + out[f'bvh{tag}_prims']):.2f}"
                  f" kd ops {np.mean(out[f'kd{tag}_nodes'] + out[f'kd{tag}_ropes'] + out[f'kd{tag}_prims']):.2f}",
                  flush=True)
    np.savez_compressed(os.path.join(HERE, f"struct_{cfg}.npz"), **out)


def make_experiment():
    """Reference sample_rays + run_experiment on Lines-1024 (both meshes, all
    7 c_t), for the device run_experiment (report JSON without timings)."""
    from mintri.experiment import run_experiment
    d = os.path.join(FIX, "lines1024")
    scene = Scene.load(os.path.join(d, "scene.txt"))
    tris = [load_triangulation(os.path.join(d, f"{w}.tri"), scene) for w in ("cdt", "mwt")]
    rays = sample_rays(scene, 3000, seed=11)
    rep = run_experiment(scene, tris, rays, labels=["cdt", "mwt"])
    payload = json.loads(rep.to_json())
    payload.pop("timing")
    small = sample_rays(scene, 5000, seed=5)
    np.savez_compressed(os.path.join(HERE, "experiment.npz"),
                        rays=ray_arr(rays), report=np.array(json.dumps(payload, sort_keys=True)),
                        csv=np.array(rep.to_csv()), sample5000_seed5=ray_arr(small))


# Rays where the reference's walk and its brute-force oracle disagree (so its
# own run_experiment stops with HitMismatchError): found by tools/paper_table.py
# over the full BASELINE ray sets on the device; (config, box, raygen index).
DEGENERATE = [("grass4096", (0.0, 0.0, 1.0, 0.5), 7031414)]


def make_degenerate():
    """The reference walk (both meshes), brute_force_closest and _check on the
    near-degenerate rays: pins that the engine reproduces the reference's
    walk result, not the brute-force one, exactly where the two differ."""
    from mintri.experiment import HitMismatchError, run_experiment
    out = {}
    for k, (cfg, box, index) in enumerate(DEGENERATE):
        d = os.path.join(FIX, cfg)
        scene = Scene.load(os.path.join(d, "scene.txt"))
        idx = SceneIndex(scene)
        arr = raygen(0, box, 0, index, 1)
        ray = rays_from(arr)[0]
        bf = brute_force_closest(scene, ray, idx)
        out[f"{k}_cfg"] = np.array(cfg)
        out[f"{k}_index"] = np.array(index)
        out[f"{k}_ray"] = arr
        out[f"{k}_brute"] = np.array([bf.seg if bf else -1, bf.t if bf else np.nan])
        tris = []
        for w in ("cdt", "mwt"):
            tri = load_triangulation(os.path.join(d, f"{w}.tri"), scene)
            tris.append(tri)
            st = TriLocator(tri).locate(ray.origin)
            hit, stats = traverse_triangulation(tri, ray, st, idx)
            out[f"{k}_{w}"] = np.array([st, hit.seg if hit else -1, stats.tri_steps])
            out[f"{k}_{w}_t"] = np.array(hit.t if hit else np.nan)
        try:
            run_experiment(scene, tris, [ray], labels=["cdt", "mwt"], ct_grid=[1.0])
            raised = False
        except HitMismatchError:
            raised = True
        out[f"{k}_harness_raises"] = np.array(raised)
        print(cfg, index, {kk: v for kk, v in out.items() if kk.startswith(f"{k}_")}, flush=True)
    np.savez_compressed(os.path.join(HERE, "degenerate.npz"), **out)


# ----------------------------------------------------------------------
# Branches random rays never reach (accel.py:164-168, :182-191, :198 into
# geometry.py:149-161, accel.py:241-246, :287-288), each forced by a
# hand-built input and recorded from the reference itself.

def run_walk_given(tri, rays, starts, index=None):
    """traverse_triangulation from GIVEN start triangles; error = 1 for a
    revisit ('traversal loop', accel.py:164-168), 2 for no exit edge
    (accel.py:190-191)."""
    from mintri.accel import TraversalError
    index = index or SceneIndex(tri.scene)
    n = len(rays)
    out = dict(start=np.asarray(starts, np.int32).copy(), seg=np.full(n, -1, np.int32), t=np.full(n, np.nan),
               u=np.full(n, np.nan), steps=np.zeros(n, np.int32), error=np.zeros(n, np.uint8))
    for i, r in enumerate(rays):
        try:
            hit, st = traverse_triangulation(tri, r, int(starts[i]), index)
        except TraversalError as e:
            out["error"][i] = 1 if "loop" in str(e) else 2
            continue
        out["steps"][i] = st.tri_steps
        if hit is not None:
            out["seg"][i] = hit.seg
            out["t"][i] = hit.t
            seg = tri.scene.segments[hit.seg]
            ex, ey = seg.b.x - seg.a.x, seg.b.y - seg.a.y
            out["u"][i] = ((hit.point.x - seg.a.x) * ex + (hit.point.y - seg.a.y) * ey) / (ex * ex + ey * ey)
    return out


def fan_mesh(cx, cy, constrained=True):
    """The unit square as a 4-triangle fan around a centre vertex (cx, cy), the
    edge corner0 -> centre constrained as geometry segment 0 (or nothing
    constrained but the square).  Moving the centre onto a side makes a
    triangle degenerate (three collinear corners: no exit edge for a ray
    parallel to it, accel.py:190-191); moving it outside the square inverts
    triangles: fallback exits, and a ray whose line separates the centre from
    the four corners circles the centre forever (revisit, accel.py:164-168)."""
    from mintri.scene import Scene, unit_square_boundary
    from mintri.trimesh import Triangulation
    geo = [Segment(Point(0.0, 0.0), Point(cx, cy))] if constrained else []
    g = len(geo)
    sc = Scene(geo + unit_square_boundary(), name="fan")
    tri = Triangulation(sc)
    for x, y in ((0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0), (cx, cy)):
        tri.add_vertex(x, y, 0)
    c = 0 if constrained else -1
    # T0=(0,1,4) T1=(1,2,4) T2=(2,3,4) T3=(3,0,4); edge i opposite v[i]
    tri._new_tri(0, 1, 4, nbr=[1, 3, None], flag=[-1, c, g + 0])
    tri._new_tri(1, 2, 4, nbr=[2, 0, None], flag=[-1, -1, g + 1])
    tri._new_tri(2, 3, 4, nbr=[3, 1, None], flag=[-1, -1, g + 2])
    tri._new_tri(3, 0, 4, nbr=[0, 2, None], flag=[c, -1, g + 3])
    return sc, tri


def diagonal_chain_mesh():
    """A diagonal segment (0.25, 0.25) -> (0.75, 0.75) whose constrained chain
    runs through a vertex 2^-40 off its line: rays exactly parallel to the
    segment (direction (s, s)) cross the chain edge, so ray_segment_intersect
    takes its parallel branch at a walk exit (accel.py:198, geometry.py:149-161):
    collinear rays hit an endpoint, offset ones fall to the grazing fallback."""
    from mintri.scene import Scene, unit_square_boundary
    a, b = Point(0.25, 0.25), Point(0.75, 0.75)
    m = Point(0.5, 0.5 + 2.0 ** -40)
    sc1 = Scene([Segment(a, m), Segment(m, b)] + unit_square_boundary(), name="chain")
    tri = build_cdt(sc1)
    sc2 = Scene([Segment(a, b)] + unit_square_boundary(), name="diagonal")
    remap = {0: 0, 1: 0, 2: 1, 3: 2, 4: 3, 5: 4}
    for tid in tri.alive_tris():
        t = tri.tris[tid]
        t.flag = [f if f == -1 else remap[f] for f in t.flag]
    tri.scene = sc2
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.tri")
        save_triangulation(tri, p)
        return sc2, load_triangulation(p, sc2)


def make_branches():
    import warnings
    out = {}
    names = []
    rng = np.random.default_rng(7)

    def record(name, sc, tri, rays, starts=None, loc_pts=None):
        xy, kind = scene_arrays(sc)
        vxy, v, nbr, flag = tri_arrays(tri)
        d = dict(seg_xy=xy, seg_kind=kind, vxy=vxy, v=v, nbr=nbr, flag=flag, rays=ray_arr(rays))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")  # locate_brute_force's "outside all triangles"
            if starts is None:
                loc = TriLocator(tri)
                starts = [loc.locate(r.origin) for r in rays]
            d.update(prefixed("w_", run_walk_given(tri, rays, starts)))
            if loc_pts is not None:
                loc = TriLocator(tri)
                d["loc_pts"] = np.array(loc_pts, np.float64).reshape(-1, 2)
                d["loc_anchor"] = np.array([loc.locate(Point(*p)) for p in loc_pts], np.int32)
                d["loc_brute"] = np.array([locate_triangle(tri, Point(*p), "brute") for p in loc_pts], np.int32)
        out.update(prefixed(f"{name}__", d))
        names.append(name)
        e = d["w_error"]
        print(f"branches/{name}: {len(rays)} rays, loop errors {int((e == 1).sum())}, "
              f"no-exit errors {int((e == 2).sum())}, hits {int((d['w_seg'] >= 0).sum())}", flush=True)

    # (1) wrong start triangles on real meshes: the first triangle does not hold
    # the origin, so exits come from the fallback rule (accel.py:182-184, :188-189)
    for cfg, which in (("lines64", "mwt"), ("lines1024", "cdt")):
        d = os.path.join(FIX, cfg)
        scene = Scene.load(os.path.join(d, "scene.txt"))
        tri = load_triangulation(os.path.join(d, f"{which}.tri"), scene)
        arr = raygen(1, (0.0, 0.0, 1.0, 1.0), 101, 0, 3000)
        starts = rng.integers(0, tri.num_tris, len(arr))
        record(f"wrongstart_{cfg}_{which}", scene, tri, rays_from(arr), starts=starts)

    # (2) fans: degenerate and inverted triangles -> no-exit and loop errors
    fans = [(0.3, 0.6, True), (0.5, 0.0, True), (0.5, -0.3, True), (1.4, 0.5, True), (0.5, 1.0, True),
            (0.5, -0.3, False), (1.4, 0.5, False), (-0.25, 0.7, False)]
    for k, (cx, cy, con) in enumerate(fans):
        sc, tri = fan_mesh(cx, cy, con)
        arr = raygen(1, (-0.5, -0.5, 1.5, 1.5), 200 + k, 0, 300)
        rays = rays_from(arr)
        extra = [Ray(Point(x, y), Point(dx, 0.0)) for y in (0.0, cy, 1.0) for x in (-0.2, 0.1, 0.5, 0.7, 1.2)
                 for dx in (1.0, -1.0)]
        extra += [Ray(Point(cx, y), Point(0.0, dy)) for y in (-0.3, 0.2, 0.8) for dy in (1.0, -1.0)]
        # lines between the centre and the square (a displaced centre: circling rays)
        for f in (0.3, 0.5, 0.7):
            if cy < 0.0 or cy > 1.0:
                yy = (0.0 if cy < 0.0 else 1.0) * (1 - f) + cy * f
                extra += [Ray(Point(x, yy), Point(dx, 0.0)) for x in (0.2, 0.5, 0.9) for dx in (1.0, -1.0)]
            if cx < 0.0 or cx > 1.0:
                xx = (0.0 if cx < 0.0 else 1.0) * (1 - f) + cx * f
                extra += [Ray(Point(xx, y), Point(0.0, dy)) for y in (0.2, 0.5, 0.9) for dy in (1.0, -1.0)]
        rays = rays + extra
        starts = np.arange(len(rays) * 4, dtype=np.int32) % 4
        rays4 = [r for r in rays for _ in range(4)]
        record(f"fan{k}", sc, tri, rays4, starts=starts)

    # (3) parallel branch at a constrained exit
    sc, tri = diagonal_chain_mesh()
    s = math.sqrt(0.5)
    rays = []
    for delta in (0.0, 2.0 ** -50, 2.0 ** -45, 2.0 ** -42, 2.0 ** -41, 3 * 2.0 ** -42, -2.0 ** -45, -2.0 ** -42):
        for t0 in (0.05, 0.3, 0.45, 0.55, 0.6):
            rays.append(Ray(Point(t0, t0 + delta), Point(s, s)))
            rays.append(Ray(Point(1.0 - t0, 1.0 - t0 + delta), Point(-s, -s)))
    record("parallel_exit", sc, tri, rays)

    # (4) locate outside every triangle: anchor walk fails, brute force finds
    # nothing, nearest centroid by math.hypot (accel.py:241-246, :287-288)
    pts = [(x, y) for x in (-6.0, -0.7, -1e-9, 0.4, 1.0 + 1e-9, 1.3, 5.0) for y in (-3.0, -0.2, 0.6, 1.5, 7.0)
           if not (0.0 <= x <= 1.0 and 0.0 <= y <= 1.0)]
    for cfg in ("lines64", "floorplan64"):
        d = os.path.join(FIX, cfg)
        scene = Scene.load(os.path.join(d, "scene.txt"))
        tri = load_triangulation(os.path.join(d, "mwt.tri"), scene)
        arr = raygen(1, (-0.5, -0.5, 1.5, 1.5), 300, 0, 120 if cfg == "floorplan64" else 400)
        record(f"outside_{cfg}", scene, tri, rays_from(arr), loc_pts=pts)
    out["cases"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "branches.npz"), **out)


def make_kdstart(nrays=2000):
    """kd_intersect(kd, ray, start_leaf=leaf) (accel.py:761-771) from random
    leaves of the reference-built Lines-1024 kd-tree (c_t = 1): results,
    counters and errors, with each leaf's preorder index in the flattened tree."""
    from paper_2112_05570_b200.accel import flatten_kd
    d = os.path.join(FIX, "lines1024")
    scene = Scene.load(os.path.join(d, "scene.txt"))
    kd = build_kdtree(scene, 1.0)
    flat = flatten_kd(kd)
    index = flat.pop("_node_index")
    rng = np.random.default_rng(17)
    arr = raygen(1, (0.0, 0.0, 1.0, 1.0), 55, 0, nrays)
    leaves = rng.integers(0, len(kd._leaves), nrays)
    out = {k: v for k, v in flat.items()}
    out["rays"] = arr
    out["start"] = np.array([index[id(kd._leaves[k])] for k in leaves], np.int32)
    seg, t, nodes, ropes, prims, err = [], [], [], [], [], []
    for r, k in zip(rays_from(arr), leaves):
        try:
            h, st = kd_intersect(kd, r, start_leaf=kd._leaves[k])
        except TraversalError:
            seg.append(-1); t.append(np.nan); nodes.append(-1); ropes.append(-1); prims.append(-1); err.append(1)
            continue
        seg.append(-1 if h is None else h.seg); t.append(np.nan if h is None else h.t)
        nodes.append(st.kd_nodes_visited); ropes.append(st.kd_rope_steps); prims.append(st.kd_prim_tests)
        err.append(0)
    # results under out_*: the flattened tree already owns `ropes` and `prims`
    out.update(out_seg=np.array(seg, np.int32), out_t=np.array(t), out_nodes=np.array(nodes, np.int32),
               out_ropes=np.array(ropes, np.int32), out_prims=np.array(prims, np.int32),
               out_error=np.array(err, np.uint8))
    print(f"kdstart: {nrays} rays, {int(np.sum(err))} errors, hits {int((out['out_seg'] >= 0).sum())}", flush=True)
    np.savez_compressed(os.path.join(HERE, "kdstart.npz"), **out)


if __name__ == "__main__":
    groups = sys.argv[1:] or ["known", "hypot"] + [f"config:{c}" for c in CONFIGS] + \
        [f"struct:{c}" for c in CONFIGS[1:]]
    for g in groups:
        if g == "known":
            make_known()
        elif g == "hypot":
            make_hypot()
        elif g == "experiment":
            make_experiment()
        elif g == "degenerate":
            make_degenerate()
        elif g == "branches":
            make_branches()
        elif g == "kdstart":
            make_kdstart()
        elif g.startswith("config:"):
            make_config(g.split(":", 1)[1])
        elif g.startswith("struct:"):
            make_struct(g.split(":", 1)[1])
        else:
            raise SystemExit(f"unknown group {g}")
