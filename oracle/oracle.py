"""ctypes front end of the C oracle (oracle/mwt_oracle.c) + independent file
loaders for the reference's text formats.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never
imports this module.

Loaders restate the reference readers:
  mintri-scene v1  scene.py:125-165 (parse_scene)
  mintri-tri v1    trimesh.py:1309-1337 (load_triangulation)
so that the oracle does not share a parser with the engine's packer.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libmwt_oracle.so")

ST_ERROR = 1
ST_FALLBACK = 2
ST_GRAZING = 4
ST_CANON = 8
ST_PARALLEL = 16
ST_ZERO_SIDE = 32
ST_MULTI = 64
ST_LOC_TIE = 128
ST_LOC_BRUTE = 256
ST_LOC_OUTSIDE = 512
ST_OVERFLOW = 1024


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, u64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.orc_hypot.restype = dbl
        L.orc_hypot.argtypes = [dbl, dbl]
        L.orc_raygen.restype = ctypes.c_int
        L.orc_raygen.argtypes = [ctypes.c_int, P, u64, u64, i64, P]
        L.orc_mesh_create.restype = P
        L.orc_mesh_create.argtypes = [ctypes.c_int, P, P, ctypes.c_int, P, P, P,
                                      ctypes.c_int, P, P, P, P, P]
        L.orc_mesh_destroy.argtypes = [P]
        L.orc_anchor_res.restype = ctypes.c_int
        L.orc_anchor_res.argtypes = [P]
        L.orc_anchors.argtypes = [P, P]
        L.orc_locate.argtypes = [P, P, i64, P, P]
        L.orc_trace.argtypes = [P, P, P, i64, P, P, P, P, P, P]
        L.orc_trace_ex.argtypes = [P, P, P, i64, P, P, P, P, P, P, P]
        L.orc_brute_force.argtypes = [P, P, i64, P, P, P]
        L.orc_ray_segment_intersect.restype = ctypes.c_int
        L.orc_ray_segment_intersect.argtypes = [P, P, P, P]
        L.orc_bvh_create.restype = P
        L.orc_bvh_create.argtypes = [ctypes.c_int, P, P, P, P, P, P]
        L.orc_bvh_destroy.argtypes = [P]
        L.orc_bvh_trace.argtypes = [P, P, P, i64, P, P, P, P, P]
        L.orc_kd_create.restype = P
        L.orc_kd_create.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, P, P, P, P]
        L.orc_kd_destroy.argtypes = [P]
        L.orc_kd_trace.argtypes = [P, P, P, i64, P, P, P, P, P, P, P]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------
# reference text formats

@dataclass
class RawScene:
    ax: np.ndarray
    ay: np.ndarray
    bx: np.ndarray
    by: np.ndarray
    kind: np.ndarray  # uint8: 0 geometry 'G', 1 boundary 'B'
    name: str = "scene"


@dataclass
class RawTri:
    vx: np.ndarray
    vy: np.ndarray
    v: np.ndarray     # (T, 3) int32
    nbr: np.ndarray   # (T, 3) int32, -1 = None
    flag: np.ndarray  # (T, 3) int32, -1 = INTERNAL


def load_scene(path: str) -> RawScene:
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines or lines[0].strip() != "mintri-scene v1":
        raise ValueError("not a scene file")
    name, idx, count = "scene", 1, None
    while idx < len(lines):
        line = lines[idx].strip()
        idx += 1
        if line.startswith("name "):
            name = line[5:]
        elif line.startswith("segments "):
            count = int(line.split()[1])
            break
    rows = [lines[idx + k].split() for k in range(count)]
    xy = np.array([[float(v) for v in r[:4]] for r in rows], dtype=np.float64).reshape(-1, 4)
    kind = np.array([0 if r[4] == "G" else 1 for r in rows], dtype=np.uint8)
    return RawScene(xy[:, 0].copy(), xy[:, 1].copy(), xy[:, 2].copy(), xy[:, 3].copy(), kind, name)


def load_tri(path: str) -> RawTri:
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines or lines[0].strip() != "mintri-tri v1":
        raise ValueError("not a triangulation file")
    k = 1
    if lines[k].startswith("scene "):
        k += 1
    nv = int(lines[k].split()[1])
    k += 1
    vv = np.array([[float(s) for s in lines[k + i].split()[:2]] for i in range(nv)],
                  dtype=np.float64).reshape(-1, 2)
    k += nv
    nt = int(lines[k].split()[1])
    k += 1
    tt = np.array([[int(s) for s in lines[k + i].split()] for i in range(nt)],
                  dtype=np.int32).reshape(-1, 9)
    return RawTri(vv[:, 0].copy(), vv[:, 1].copy(), np.ascontiguousarray(tt[:, 0:3]),
                  np.ascontiguousarray(tt[:, 3:6]), np.ascontiguousarray(tt[:, 6:9]))


# ----------------------------------------------------------------------

def hypot(x: float, y: float) -> float:
    return lib().orc_hypot(x, y)


def raygen(mode: int, box, seed: int, first: int, n: int) -> np.ndarray:
    out = np.empty((n, 4), dtype=np.float64)
    b = np.ascontiguousarray(box, dtype=np.float64)
    if lib().orc_raygen(mode, _p(b), seed, first, n, _p(out)) != 0:
        raise ValueError(f"malformed ray generator mode word {mode:#x}")
    return out


class Mesh:
    """Oracle view of (scene, triangulation); keeps its arrays alive."""

    def __init__(self, scene: RawScene, tri: RawTri | None):
        self.scene = scene
        self.tri = tri
        L = lib()
        if tri is None:
            tri = RawTri(np.zeros(0), np.zeros(0), np.zeros((0, 3), np.int32),
                         np.zeros((0, 3), np.int32), np.zeros((0, 3), np.int32))
        self._keep = (tri.vx, tri.vy, tri.v, tri.nbr, tri.flag,
                      scene.ax, scene.ay, scene.bx, scene.by, scene.kind)
        self.h = L.orc_mesh_create(len(tri.vx), _p(tri.vx), _p(tri.vy), len(tri.v), _p(tri.v),
                                   _p(tri.nbr), _p(tri.flag), len(scene.ax), _p(scene.ax),
                                   _p(scene.ay), _p(scene.bx), _p(scene.by), _p(scene.kind))

    def __del__(self):
        try:
            lib().orc_mesh_destroy(self.h)
        except Exception:
            pass

    @classmethod
    def from_files(cls, scene_path: str, tri_path: str | None) -> "Mesh":
        return cls(load_scene(scene_path), load_tri(tri_path) if tri_path else None)

    def anchors(self) -> np.ndarray:
        L = lib()
        res = L.orc_anchor_res(self.h)
        out = np.empty(res * res, dtype=np.int32)
        L.orc_anchors(self.h, _p(out))
        return out.reshape(res, res)

    def locate(self, pts: np.ndarray):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        n = len(pts)
        tid = np.empty(n, np.int32)
        st = np.empty(n, np.uint32)
        lib().orc_locate(self.h, _p(pts), n, _p(tid), _p(st))
        return tid, st

    def trace(self, rays: np.ndarray, start: np.ndarray | None = None) -> dict:
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 4)
        n = len(rays)
        out = dict(start=np.empty(n, np.int32), seg=np.empty(n, np.int32), t=np.empty(n),
                   u=np.empty(n), steps=np.empty(n, np.int32), status=np.empty(n, np.uint32),
                   end=np.empty(n, np.int32))
        sp = None
        if start is not None:
            start = np.ascontiguousarray(start, dtype=np.int32)
            sp = _p(start)
        lib().orc_trace_ex(self.h, _p(rays), sp, n, _p(out["start"]), _p(out["seg"]), _p(out["t"]),
                           _p(out["u"]), _p(out["steps"]), _p(out["status"]), _p(out["end"]))
        return out

    def brute_force(self, rays: np.ndarray) -> dict:
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 4)
        n = len(rays)
        out = dict(seg=np.empty(n, np.int32), t=np.empty(n), u=np.empty(n))
        lib().orc_brute_force(self.h, _p(rays), n, _p(out["seg"]), _p(out["t"]), _p(out["u"]))
        return out


def load_npz(path: str) -> dict:
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


class Bvh:
    def __init__(self, mesh: Mesh, arrays: dict):
        self.mesh = mesh
        a = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
        self._a = a
        self.h = lib().orc_bvh_create(len(a["left"]), _p(a["box"]), _p(a["left"]), _p(a["right"]),
                                      _p(a["prim_off"]), _p(a["prim_cnt"]), _p(a["prims"]))

    def __del__(self):
        try:
            lib().orc_bvh_destroy(self.h)
        except Exception:
            pass

    def trace(self, rays: np.ndarray) -> dict:
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 4)
        n = len(rays)
        out = dict(seg=np.empty(n, np.int32), t=np.empty(n), u=np.empty(n),
                   node_tests=np.empty(n, np.int32), prim_tests=np.empty(n, np.int32))
        lib().orc_bvh_trace(self.mesh.h, self.h, _p(rays), n, _p(out["seg"]), _p(out["t"]),
                            _p(out["u"]), _p(out["node_tests"]), _p(out["prim_tests"]))
        return out


class Kd:
    def __init__(self, mesh: Mesh, arrays: dict):
        self.mesh = mesh
        a = {k: np.ascontiguousarray(v) for k, v in arrays.items()}
        self._a = a
        self.h = lib().orc_kd_create(len(a["axis"]), int(np.asarray(a["num_leaves"]).reshape(-1)[0]), _p(a["axis"]), _p(a["pos"]),
                                     _p(a["left"]), _p(a["right"]), _p(a["box"]), _p(a["ropes"]),
                                     _p(a["rope_cost"]), _p(a["prim_off"]), _p(a["prim_cnt"]),
                                     _p(a["prims"]))

    def __del__(self):
        try:
            lib().orc_kd_destroy(self.h)
        except Exception:
            pass

    def trace(self, rays: np.ndarray) -> dict:
        rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 4)
        n = len(rays)
        out = dict(seg=np.empty(n, np.int32), t=np.empty(n), u=np.empty(n),
                   nodes=np.empty(n, np.int32), ropes=np.empty(n, np.int32),
                   prims=np.empty(n, np.int32), status=np.empty(n, np.uint32))
        lib().orc_kd_trace(self.mesh.h, self.h, _p(rays), n, _p(out["seg"]), _p(out["t"]),
                           _p(out["u"]), _p(out["nodes"]), _p(out["ropes"]), _p(out["prims"]),
                           _p(out["status"]))
        return out


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))
