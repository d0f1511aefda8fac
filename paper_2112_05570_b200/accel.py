"""Drop-in for the reference's ray-query API (mintri/accel.py), backed by the
CUDA engine.  Same names, argument meaning, return types and errors:

  traverse_triangulation(tri, ray, start_tri, index=None)   accel.py:138-213
  TriLocator(tri).locate(p)                                  accel.py:256-289
  locate_triangle(tri, p, method="anchor", locator=None)     accel.py:333-353
  bvh_intersect(bvh, ray)                                    accel.py:482-518
  kd_intersect(kd, ray, start_leaf=None)                     accel.py:761-832
  brute_force_closest(scene, ray, index=None)                accel.py:101-132
  sweep_structure_params(builder, scene, rays, grid)         accel.py:845-862
  Hit, TraversalStats, TraversalError, C_T_GRID              accel.py:28-61

``tri`` / ``scene`` / ``bvh`` / ``kd`` may be the reference's own objects
(duck-typed: Triangulation.verts/.tris/.scene, Scene.segments, Bvh.root,
RopedKdTree.root/._leaves) or this package's arrays.  The first call on an
object packs it onto the GPU (cached per object); every query then runs on
the device.  The batched entry points (``trace_batch`` etc.) are the fast
path; the per-ray functions exist so the reference's tests and callers run
unchanged.
"""
from __future__ import annotations

import math
import operator
import weakref
from dataclasses import dataclass
from typing import Callable, Iterable, Optional

import numpy as np

from . import _lib
from .engine import DeviceBvh, DeviceKd, DeviceMesh
from .formats import SceneArrays, TriArrays
from .geometry import Point, Ray

C_T_GRID = (0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0)


class TraversalError(RuntimeError):
    pass


@dataclass
class Hit:
    seg: int
    t: float
    point: Point


@dataclass
class TraversalStats:
    tri_steps: int = 0
    bvh_node_tests: int = 0
    bvh_prim_tests: int = 0
    kd_nodes_visited: int = 0
    kd_rope_steps: int = 0
    kd_prim_tests: int = 0

    def total(self) -> int:
        return (self.tri_steps + self.bvh_node_tests + self.bvh_prim_tests
                + self.kd_nodes_visited + self.kd_rope_steps + self.kd_prim_tests)

    def add(self, other: "TraversalStats") -> None:
        self.tri_steps += other.tri_steps
        self.bvh_node_tests += other.bvh_node_tests
        self.bvh_prim_tests += other.bvh_prim_tests
        self.kd_nodes_visited += other.kd_nodes_visited
        self.kd_rope_steps += other.kd_rope_steps
        self.kd_prim_tests += other.kd_prim_tests


# ----------------------------------------------------------------------
# conversion of reference objects to the packer's arrays

def scene_arrays(scene) -> SceneArrays:
    if isinstance(scene, SceneArrays):
        return scene
    segs = scene.segments
    xy = np.array([[s.a.x, s.a.y, s.b.x, s.b.y] for s in segs], dtype=np.float64).reshape(-1, 4)
    kind = np.array([0 if _kind(s) == "G" else 1 for s in segs], dtype=np.uint8)
    return SceneArrays(xy, kind, getattr(scene, "name", "scene"), getattr(scene, "provenance", ""))


def _kind(seg) -> str:
    k = seg.kind
    return getattr(k, "value", k)


class _TriMap:
    """Reference Triangulation -> compact arrays (dead slots dropped; the
    order-preserving map keeps 'lowest id' semantics)."""

    def __init__(self, tri):
        alive = [t for t, tr in enumerate(tri.tris) if tr is not None]
        self.to_ref = np.array(alive, dtype=np.int64)
        to_compact = {t: k for k, t in enumerate(alive)}
        self.to_compact = to_compact
        nv = len(tri.verts)
        vxy = np.array([[v.x, v.y] for v in tri.verts], dtype=np.float64).reshape(nv, 2)
        v = np.array([tri.tris[t].v for t in alive], dtype=np.int32).reshape(-1, 3)
        nbr = np.array([[-1 if n is None else to_compact[n] for n in tri.tris[t].nbr] for t in alive],
                       dtype=np.int32).reshape(-1, 3)
        flag = np.array([tri.tris[t].flag for t in alive], dtype=np.int32).reshape(-1, 3)
        self.arrays = TriArrays(vxy, v, nbr, flag)


class _IdCache:
    """Per-object cache keyed by identity (the reference's Scene and
    Triangulation are unhashable dataclasses); entries die with the object."""

    def __init__(self):
        self._d: dict = {}

    def get(self, obj):
        got = self._d.get(id(obj))
        return got[1] if got is not None and got[0]() is obj else None

    def pop(self, obj):
        got = self._d.get(id(obj))
        if got is not None and got[0]() is obj:
            del self._d[id(obj)]

    def __setitem__(self, obj, value):
        key = id(obj)
        self._d[key] = (weakref.ref(obj), value)
        weakref.finalize(obj, self._d.pop, key, None)


_mesh_cache = _IdCache()


class _Packed:
    def __init__(self, mesh: DeviceMesh, tmap: Optional[_TriMap], scene):
        self.mesh = mesh
        self.tmap = tmap
        self.scene = scene


def _segment_of(scene, sid: int):
    """Scene segment ``sid`` (a reference Scene or this package's SceneArrays)."""
    if isinstance(scene, SceneArrays):
        from .geometry import Segment, SegmentKind
        r = scene.xy[sid].tolist()
        return Segment(Point(*r[:2]), Point(*r[2:]),
                       SegmentKind.GEOMETRY if int(scene.kind[sid]) == 0 else SegmentKind.BOUNDARY)
    return scene.segments[sid]


# The reference edits triangulations in place (trimesh.flip_edge, the
# annealer's vertex moves) and its walk reads the live mesh, so a cached pack
# is reused only while the mesh's content is unchanged: every call compares a
# value snapshot of the vertex coordinates, triangle corners, neighbours and
# flags, and the scene's (immutable) segments, with the one taken at packing
# time (O(triangles) host work, ~50 us for a 200-triangle mesh).  Set
# CHECK_MUTATION = False for meshes known to be immutable, or call
# invalidate(tri) after an edit.
CHECK_MUTATION = True
_XY = operator.attrgetter("x", "y")


def _fingerprint(tri) -> tuple:
    """Value snapshot of everything the walk reads (copies, not references:
    the reference mutates Tri.v / nbr / flag lists in place)."""
    return (list(map(_XY, tri.verts)),
            [None if t is None else (*t.v, *t.nbr, *t.flag) for t in tri.tris],
            list(tri.scene.segments))


def invalidate(obj) -> None:
    """Drop the cached device copy of a triangulation (or structure / scene)."""
    for c in (_mesh_cache, _struct_cache, _scene_mesh_cache):
        c.pop(obj)


def pack(tri, device: int = 0) -> _Packed:
    """Packed device mesh for a reference Triangulation (cached while its
    content is unchanged) or for a (SceneArrays, TriArrays) pair."""
    if isinstance(tri, tuple):
        scene, arrays = tri
        return _Packed(DeviceMesh(scene_arrays(scene), arrays, device), None, scene)
    got = _mesh_cache.get(tri)
    fp = _fingerprint(tri) if CHECK_MUTATION else None
    if got is not None and (got.device != device or (fp is not None and got.fp != fp)):
        got = None  # edited since it was packed (or another device): repack
    if got is None:
        tmap = _TriMap(tri)
        mesh = DeviceMesh(scene_arrays(tri.scene), tmap.arrays, device)
        got = _Packed(mesh, tmap, tri.scene)
        got.fp, got.device = fp, device
        _mesh_cache[tri] = got
    return got


def _ray_array(rays) -> np.ndarray:
    if isinstance(rays, np.ndarray):
        return np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 4)
    return np.array([[r.origin[0], r.origin[1], r.direction[0], r.direction[1]] for r in rays],
                    dtype=np.float64).reshape(-1, 4)


def _hit(scene, seg: int, t: float, u: float) -> Optional[Hit]:
    if seg < 0:
        return None
    return Hit(int(seg), float(t), _segment_of(scene, int(seg)).point_at(float(u)))


# ----------------------------------------------------------------------
# batched API

def trace_batch(tri, rays, start=None, device: int = 0) -> dict:
    """Every ray through ``tri``: start triangles located on the device unless
    given.  Returns numpy arrays start/seg/t/u/steps/status (reference ids)."""
    P = tri if isinstance(tri, _Packed) else pack(tri, device)
    r = _ray_array(rays)
    s = None
    if start is not None:
        s = np.asarray(start, dtype=np.int64)
        if P.tmap is not None:
            s = np.array([P.tmap.to_compact.get(int(x), -1) for x in s], dtype=np.int32)
        s = s.astype(np.int32)
    out = P.mesh.trace(r, s)
    if P.tmap is not None:
        out["start"] = P.tmap.to_ref[out["start"]].astype(np.int64) if len(r) else out["start"]
    return out


def locate_batch(tri, pts, device: int = 0):
    P = pack(tri, device)
    tid, st = P.mesh.locate(np.asarray(pts, dtype=np.float64).reshape(-1, 2))
    if P.tmap is not None and len(tid):
        tid = P.tmap.to_ref[tid]
    return tid, st


# ----------------------------------------------------------------------
# per-ray drop-ins

def traverse_triangulation(tri, ray: Ray, start_tri: int, index=None
                           ) -> tuple[Optional[Hit], TraversalStats]:
    """accel.py:138-213 on the device.  Raises TraversalError exactly where the
    reference does (revisited state or no exit edge)."""
    P = pack(tri)
    out = trace_batch(P, _ray_array([ray]), [start_tri])
    st = int(out["status"][0])
    if st & (_lib.ST_ERROR | _lib.ST_OVERFLOW):
        raise TraversalError(f"traversal failed from triangle {start_tri} (status {st:#x})")
    stats = TraversalStats(tri_steps=int(out["steps"][0]))
    return _hit(P.scene, int(out["seg"][0]), out["t"][0], out["u"][0]), stats


class TriLocator:
    """accel.py:256-289: anchor grid, walk, brute-force fallback, lowest-id tie
    flood -- all on the device.

    ``resolution`` (accel.py:263-268) sets the reference's anchor grid, which
    only chooses where its walk starts: the answer is the lowest id over the
    neighbour-connected triangles containing p, the same from any containing
    seed.  The device seeds its search from its own finer grid (the packer's
    cell-centre triangles), so every resolution gives the reference's result;
    ``res`` keeps the value asked for."""

    def __init__(self, tri, resolution: Optional[int] = None):
        self.tri = tri
        pack(tri)
        if resolution is None:
            resolution = max(2, int(math.sqrt(max(_num_tris(tri), 4) / 2.0)))
        if int(resolution) < 1:
            raise ValueError("resolution must be positive")
        self.res = int(resolution)

    def locate(self, p: Point) -> int:
        tid, _ = locate_batch(self.tri, [[p[0], p[1]]])
        return int(tid[0])

    def locate_many(self, pts) -> np.ndarray:
        return locate_batch(self.tri, pts)[0]


def _num_tris(tri) -> int:
    n = getattr(tri, "num_tris", None)
    return int(n) if n is not None else sum(1 for t in tri.tris if t is not None)


def locate_triangle(tri, p: Point, method: str = "anchor",
                    locator: Optional[TriLocator] = None) -> int:
    """accel.py:333-353.  "anchor": TriLocator.locate on the device; "brute":
    the lowest triangle id containing p (a device scan in id order), else the
    nearest centroid (mwt_locate_brute_dev)."""
    if method == "brute":
        P = pack(tri)
        tid, _ = P.mesh.locate(np.array([[p[0], p[1]]], dtype=np.float64), method="brute")
        t = int(tid[0])
        return int(P.tmap.to_ref[t]) if P.tmap is not None else t
    if method == "anchor":
        if locator is None:
            locator = TriLocator(tri)
        return locator.locate(p)
    raise ValueError(f"unknown location method {method!r}")


# -- BVH / kd-tree -------------------------------------------------------

def flatten_bvh(bvh) -> dict:
    """Reference Bvh object -> mwt-bvh v1 arrays (DFS preorder)."""
    boxes, left, right, poff, pcnt, prims = [], [], [], [], [], []

    def visit(node):
        k = len(boxes)
        boxes.append(node.box)
        left.append(-1); right.append(-1); poff.append(0); pcnt.append(0)
        return k
    work = [(bvh.root, None, None)]
    while work:
        node, parent, side = work.pop()
        k = visit(node)
        if parent is not None:
            (left if side == 0 else right)[parent] = k
        if node.prims is not None:
            poff[k] = len(prims)
            pcnt[k] = len(node.prims)
            prims.extend(node.prims)
        else:
            work.append((node.right, k, 1))
            work.append((node.left, k, 0))
    return dict(c_t=np.float64(getattr(bvh, "c_t", np.nan)),
                box=np.array(boxes, dtype=np.float64).reshape(-1, 4),
                left=np.array(left, np.int32), right=np.array(right, np.int32),
                prim_off=np.array(poff, np.int32), prim_cnt=np.array(pcnt, np.int32),
                prims=np.array(prims, np.int32))


def flatten_kd(kd) -> dict:
    """Reference RopedKdTree object -> mwt-kd v1 arrays (DFS preorder), rope
    cost max(1, ceil(log2(count))) evaluated as the reference does (accel.py:818)."""
    nodes, index = [], {}
    work = [kd.root]
    while work:
        node = work.pop()
        index[id(node)] = len(nodes)
        nodes.append(node)
        if node.prims is None:
            work.append(node.right)
            work.append(node.left)
    n = len(nodes)
    axis = np.full(n, -1, np.int32); pos = np.zeros(n); left = np.full(n, -1, np.int32)
    right = np.full(n, -1, np.int32); box = np.zeros((n, 4)); ropes = np.full((n, 4), -1, np.int32)
    counts = np.zeros((n, 4), np.int32); cost = np.zeros((n, 4), np.int32)
    poff = np.zeros(n, np.int32); pcnt = np.zeros(n, np.int32); prims: list = []
    for k, node in enumerate(nodes):
        box[k] = node.box
        if node.prims is not None:
            poff[k] = len(prims); pcnt[k] = len(node.prims); prims.extend(node.prims)
            for s in range(4):
                r = node.ropes[s]
                if r is not None:
                    ropes[k, s] = index[id(r)]
                    counts[k, s] = node.rope_counts[s]
                    cost[k, s] = max(1, math.ceil(math.log2(node.rope_counts[s])))
        else:
            axis[k] = node.axis; pos[k] = node.pos
            left[k] = index[id(node.left)]; right[k] = index[id(node.right)]
    return dict(c_t=np.float64(getattr(kd, "c_t", np.nan)), num_leaves=np.int64(len(kd._leaves)),
                axis=axis, pos=pos, left=left, right=right, box=box, ropes=ropes,
                rope_counts=counts, rope_cost=cost, prim_off=poff, prim_cnt=pcnt,
                prims=np.array(prims, np.int32), _node_index=index)


_struct_cache = _IdCache()
_scene_mesh_cache = _IdCache()


def _scene_mesh(scene) -> DeviceMesh:
    got = _scene_mesh_cache.get(scene)
    if got is None:
        got = DeviceMesh(scene_arrays(scene), None)
        _scene_mesh_cache[scene] = got
    return got


def _device_struct(obj):
    got = _struct_cache.get(obj)
    if got is None:
        mesh = _scene_mesh(obj.scene)
        if hasattr(obj, "_leaves"):
            flat = flatten_kd(obj)
            got = DeviceKd(mesh, flat)
            got.node_index = flat["_node_index"]
            got.is_internal = flat["axis"] >= 0
        else:
            got = DeviceBvh(mesh, flatten_bvh(obj))
        _struct_cache[obj] = got
    return got


def bvh_intersect(bvh, ray: Ray) -> tuple[Optional[Hit], TraversalStats]:
    """accel.py:482-518 on the device."""
    d = _device_struct(bvh)
    o = d.trace(_ray_array([ray]))
    if int(o["status"][0]) & _lib.ST_OVERFLOW:
        raise TraversalError("bvh stack overflow")
    stats = TraversalStats(bvh_node_tests=int(o["node_tests"][0]), bvh_prim_tests=int(o["prim_tests"][0]))
    return _hit(bvh.scene, int(o["seg"][0]), o["t"][0], o["u"][0]), stats


def kd_intersect(kd, ray: Ray, start_leaf=None) -> tuple[Optional[Hit], TraversalStats]:
    """accel.py:761-832 on the device.  ``start_leaf``: a leaf node of ``kd``
    (as the reference takes it) or its preorder index in the flattened tree;
    None locates the origin's leaf (locate_leaf, accel.py:712-724)."""
    d = _device_struct(kd)
    start = None
    if start_leaf is not None:
        k = start_leaf if isinstance(start_leaf, (int, np.integer)) else d.node_index.get(id(start_leaf))
        if k is None or not (0 <= int(k) < d.num_nodes) or d.is_internal[int(k)]:
            raise ValueError("start_leaf is not a leaf of this kd-tree")
        start = np.array([int(k)], np.int32)
    o = d.trace(_ray_array([ray]), start)
    if int(o["status"][0]) & (_lib.ST_ERROR | _lib.ST_OVERFLOW):
        raise TraversalError("kd walk did not terminate")
    stats = TraversalStats(kd_nodes_visited=int(o["nodes"][0]), kd_rope_steps=int(o["ropes"][0]),
                           kd_prim_tests=int(o["prims"][0]))
    return _hit(kd.scene, int(o["seg"][0]), o["t"][0], o["u"][0]), stats


def brute_force_closest(scene, ray: Ray, index=None) -> Optional[Hit]:
    """accel.py:101-132 on the device."""
    m = _scene_mesh(scene)
    o = m.brute_force(_ray_array([ray]))
    return _hit(scene, int(o["seg"][0]), o["t"][0], o["u"][0])


@dataclass
class SweepResult:
    structure: object
    totals: dict
    best_c_t: float


def sweep_structure_params(builder: Callable, scene, rays: Iterable[Ray],
                           grid: Iterable[float] = C_T_GRID) -> SweepResult:
    """accel.py:845-862: one structure per c_t (built by ``builder`` -- the
    reference's builders), total unweighted ops over the SAME rays on the
    device, strict '<' keeps the earliest minimum."""
    r = _ray_array(list(rays))
    totals: dict = {}
    best = None
    for c_t in grid:
        structure = builder(scene, c_t)
        d = _device_struct(structure)
        o = d.trace(r)
        if isinstance(d, DeviceKd):
            total = int(o["nodes"].astype(np.int64).sum() + o["ropes"].astype(np.int64).sum()
                        + o["prims"].astype(np.int64).sum())
        else:
            total = int(o["node_tests"].astype(np.int64).sum() + o["prim_tests"].astype(np.int64).sum())
        totals[c_t] = total
        if best is None or total < best[0]:
            best = (total, c_t, structure)
    return SweepResult(best[2], totals, best[1])
