"""Batched device API over libmwt.so.

``DeviceMesh`` owns one packed triangulation on one GPU (K1) and exposes the
engine's batched operations; ``DeviceBvh`` / ``DeviceKd`` own flattened
reference structures.  Device buffers are torch tensors (torch is plumbing:
allocation, streams, torch.distributed); all computation is in libmwt.so.

Methods taking numpy arrays copy in/out and synchronise; methods named
``*_device`` take/return CUDA tensors and run asynchronously on the current
torch stream (or ``stream``).
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr
from .formats import SceneArrays, TriArrays, load_scene, load_structure, load_tri


def _stream(stream=None, device: int | None = None):
    """The stream a call launches on: ``stream``, else the current stream of
    the handle's own ``device`` (the C side switches to that device)."""
    s = torch.cuda.current_stream(device) if stream is None else stream
    return ctypes_void(s.cuda_stream)


def _held(t: torch.Tensor | None, stream=None) -> torch.Tensor | None:
    """``t`` made contiguous.  When the kernel runs on a side ``stream`` and a
    temporary copy was needed, that stream first waits for the copy (made on
    the current stream of t's device) and the copy is kept alive for its work
    (record_stream) so the caching allocator does not hand it out early."""
    if t is None:
        return None
    c = t.contiguous()
    if stream is not None and c.data_ptr() != t.data_ptr():
        stream.wait_stream(torch.cuda.current_stream(t.device))
        c.record_stream(stream)
    return c


def ctypes_void(v: int):
    import ctypes
    return ctypes.c_void_p(v)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class DeviceMesh:
    """Packed (scene, triangulation) on ``device`` -- the K1 packer's output."""

    def __init__(self, scene: SceneArrays, tri: TriArrays | None, device: int = 0):
        """``tri=None`` packs the scene only (for the BVH / kd / brute-force engines)."""
        import ctypes
        self.scene = scene
        self.tri = tri
        if tri is None:
            tri = TriArrays(np.zeros((0, 2)), np.zeros((0, 3), np.int32), np.zeros((0, 3), np.int32),
                            np.zeros((0, 3), np.int32))
        self.device = int(device)
        vxy = _f64(tri.vxy).reshape(-1, 2)
        vx, vy = _f64(vxy[:, 0]), _f64(vxy[:, 1])
        h = ctypes.c_void_p()
        check(lib.mwt_mesh_create(ptr(vx), ptr(vy), len(vx), ptr(_i32(tri.v)), ptr(_i32(tri.nbr)),
                                  ptr(_i32(tri.flag)), len(tri.v), ptr(_f64(scene.xy)),
                                  ptr(np.ascontiguousarray(scene.kind, dtype=np.uint8)),
                                  len(scene.kind), self.device, ctypes.byref(h)), "mesh_create")
        self._h = h
        info = _lib.MeshInfo()
        check(lib.mwt_mesh_info_get(h, ctypes.byref(info)), "mesh_info")
        self.info = info

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.mwt_mesh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def from_files(cls, scene_path: str, tri_path: str, device: int = 0) -> "DeviceMesh":
        return cls(load_scene(scene_path), load_tri(tri_path), device)

    @classmethod
    def from_binary(cls, path: str, device: int = 0) -> "DeviceMesh":
        """A ``mwt-mesh v1`` directory (formats.save_mesh_binary)."""
        from .formats import load_mesh_binary
        scene, tri = load_mesh_binary(path)
        return cls(scene, tri, device)

    @property
    def num_triangles(self) -> int:
        return self.info.num_triangles

    def anchors(self) -> np.ndarray:
        res = self.info.anchor_res
        out = np.empty(res * res, dtype=np.int32)
        check(lib.mwt_mesh_anchors(self._h, ptr(out)), "mesh_anchors")
        return out.reshape(res, res)

    # -- device-resident operations -------------------------------------
    def _dev(self):
        return torch.device("cuda", self.device)

    def raygen_device(self, mode: int, box, seed: int, first: int, n: int, stream=None) -> torch.Tensor:
        out = torch.empty((n, 4), dtype=torch.float64, device=self._dev())
        b = _f64(box)
        check(lib.mwt_raygen_dev(int(mode), ptr(b), int(seed), int(first), int(n), ptr(out),
                                 _stream(stream, self.device)), "raygen")
        return out

    def locate_device(self, pts: torch.Tensor, stream=None):
        pts = _held(pts, stream)
        n = pts.shape[0]
        tid = torch.empty(n, dtype=torch.int32, device=pts.device)
        st = torch.empty(n, dtype=torch.int32, device=pts.device)
        check(lib.mwt_locate_dev(self._h, ptr(pts), n, ptr(tid), ptr(st), _stream(stream, self.device)), "locate")
        return tid, st

    def trace_device(self, rays: torch.Tensor, start: torch.Tensor | None = None, stream=None,
                     want=("start", "seg", "t", "u", "steps", "status")) -> dict:
        rays, start = _held(rays, stream), _held(start, stream)
        n = rays.shape[0]
        d = rays.device
        out = {}
        spec = dict(start=torch.int32, seg=torch.int32, t=torch.float64, u=torch.float64,
                    steps=torch.int32, status=torch.int32)
        for k in want:
            out[k] = torch.empty(n, dtype=spec[k], device=d)
        g = out.get
        check(lib.mwt_trace_dev(self._h, ptr(rays), ptr(start) if start is not None else None,
                                n, ptr(g("start")), ptr(g("seg")), ptr(g("t")), ptr(g("u")),
                                ptr(g("steps")), ptr(g("status")), _stream(stream, self.device)), "trace")
        return out

    def trace_chain_device(self, rays: torch.Tensor, start: torch.Tensor | None = None,
                           stream=None) -> dict:
        """Walk and also return each walk's final triangle (``end``), to start
        secondary rays there without a locate (mwt_trace_chain_dev)."""
        rays, start = _held(rays, stream), _held(start, stream)
        n = rays.shape[0]
        d = rays.device
        out = dict(end=torch.empty(n, dtype=torch.int32, device=d),
                   seg=torch.empty(n, dtype=torch.int32, device=d),
                   t=torch.empty(n, dtype=torch.float64, device=d),
                   u=torch.empty(n, dtype=torch.float64, device=d),
                   steps=torch.empty(n, dtype=torch.int32, device=d),
                   status=torch.empty(n, dtype=torch.int32, device=d))
        check(lib.mwt_trace_chain_dev(self._h, ptr(rays),
                                      ptr(start) if start is not None else None, n,
                                      ptr(out["end"]), ptr(out["seg"]), ptr(out["t"]), ptr(out["u"]),
                                      ptr(out["steps"]), ptr(out["status"]), _stream(stream, self.device)),
              "trace_chain")
        return out

    def trace_generated_device(self, mode: int, box, seed: int, first: int, n: int,
                               outputs: bool = True, hist: torch.Tensor | None = None,
                               stream=None) -> dict:
        d = self._dev()
        out = {}
        if outputs:
            out = dict(seg=torch.empty(n, dtype=torch.int32, device=d),
                       t=torch.empty(n, dtype=torch.float64, device=d),
                       steps=torch.empty(n, dtype=torch.int32, device=d))
        g = out.get
        b = _f64(box)
        check(lib.mwt_trace_generated_dev(self._h, int(mode), ptr(b), int(seed), int(first), int(n),
                                          ptr(g("seg")), ptr(g("t")), ptr(g("steps")), ptr(hist),
                                          _stream(stream, self.device)), "trace_generated")
        return out

    def brute_force_device(self, rays: torch.Tensor, stream=None) -> dict:
        rays = _held(rays, stream)
        n = rays.shape[0]
        out = dict(seg=torch.empty(n, dtype=torch.int32, device=rays.device),
                   t=torch.empty(n, dtype=torch.float64, device=rays.device),
                   u=torch.empty(n, dtype=torch.float64, device=rays.device))
        check(lib.mwt_brute_force_dev(self._h, ptr(rays), n, ptr(out["seg"]), ptr(out["t"]),
                                      ptr(out["u"]), _stream(stream, self.device)), "brute_force")
        return out

    # -- host-buffer operations -------------------------------------------
    def trace(self, rays: np.ndarray, start: np.ndarray | None = None) -> dict:
        """Host arrays in and out through mwt_trace_host (copies + sync)."""
        rays = _f64(rays).reshape(-1, 4)
        n = len(rays)
        out = dict(start=np.empty(n, np.int32), seg=np.empty(n, np.int32), t=np.empty(n),
                   u=np.empty(n), steps=np.empty(n, np.int32), status=np.empty(n, np.uint32))
        s = _i32(start) if start is not None else None
        check(lib.mwt_trace_host(self._h, ptr(rays), ptr(s), n, ptr(out["start"]), ptr(out["seg"]),
                                 ptr(out["t"]), ptr(out["u"]), ptr(out["steps"]),
                                 ptr(out["status"])), "trace_host")
        return out

    def _to_dev(self, a: np.ndarray) -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(a)).to(self._dev())

    def locate_brute_device(self, pts: torch.Tensor, stream=None):
        """locate_triangle(tri, p, "brute"): lowest containing id, else nearest centroid."""
        pts = _held(pts, stream)
        n = pts.shape[0]
        tid = torch.empty(n, dtype=torch.int32, device=pts.device)
        st = torch.empty(n, dtype=torch.int32, device=pts.device)
        check(lib.mwt_locate_brute_dev(self._h, ptr(pts), n, ptr(tid), ptr(st), _stream(stream, self.device)),
              "locate_brute")
        return tid, st

    def locate(self, pts: np.ndarray, method: str = "anchor"):
        pts = _f64(pts).reshape(-1, 2)
        if len(pts) == 0:
            return np.zeros(0, np.int32), np.zeros(0, np.uint32)
        fn = self.locate_brute_device if method == "brute" else self.locate_device
        tid, st = fn(self._to_dev(pts))
        torch.cuda.synchronize(self.device)
        return tid.cpu().numpy(), st.cpu().numpy().view(np.uint32)

    def raygen(self, mode: int, box, seed: int, first: int, n: int) -> np.ndarray:
        r = self.raygen_device(mode, box, seed, first, n)
        torch.cuda.synchronize(self.device)
        return r.cpu().numpy()

    def brute_force(self, rays: np.ndarray) -> dict:
        rays = _f64(rays).reshape(-1, 4)
        if len(rays) == 0:
            return dict(seg=np.zeros(0, np.int32), t=np.zeros(0), u=np.zeros(0))
        out = self.brute_force_device(self._to_dev(rays))
        torch.cuda.synchronize(self.device)
        return {k: v.cpu().numpy() for k, v in out.items()}


class DeviceBvh:
    """Flattened reference Bvh (accel.py:373-426) on the mesh's device."""

    def __init__(self, mesh: DeviceMesh, arrays: dict):
        import ctypes
        self.mesh = mesh
        self.c_t = float(arrays.get("c_t", np.nan))
        box = _f64(arrays["box"]).reshape(-1, 4)
        left, right = _i32(arrays["left"]), _i32(arrays["right"])
        poff, pcnt, prims = _i32(arrays["prim_off"]), _i32(arrays["prim_cnt"]), _i32(arrays["prims"])
        h = ctypes.c_void_p()
        check(lib.mwt_bvh_create(mesh.handle, len(left), ptr(box), ptr(left), ptr(right), ptr(poff),
                                 ptr(pcnt), len(prims), ptr(prims), ctypes.byref(h)), "bvh_create")
        self._h = h
        self.num_nodes = len(left)

    @classmethod
    def from_file(cls, mesh: DeviceMesh, path: str) -> "DeviceBvh":
        return cls(mesh, load_structure(path))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.mwt_bvh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def trace_device(self, rays: torch.Tensor, stream=None) -> dict:
        rays = _held(rays, stream)
        n = rays.shape[0]
        d = rays.device
        out = dict(seg=torch.empty(n, dtype=torch.int32, device=d),
                   t=torch.empty(n, dtype=torch.float64, device=d),
                   u=torch.empty(n, dtype=torch.float64, device=d),
                   node_tests=torch.empty(n, dtype=torch.int32, device=d),
                   prim_tests=torch.empty(n, dtype=torch.int32, device=d),
                   status=torch.empty(n, dtype=torch.int32, device=d))
        check(lib.mwt_bvh_trace_dev(self._h, ptr(rays), n, ptr(out["seg"]), ptr(out["t"]),
                                    ptr(out["u"]), ptr(out["node_tests"]), ptr(out["prim_tests"]),
                                    ptr(out["status"]), _stream(stream, self.mesh.device)), "bvh_trace")
        return out

    def trace(self, rays: np.ndarray) -> dict:
        rays = _f64(rays).reshape(-1, 4)
        out = self.trace_device(torch.from_numpy(rays).to(self.mesh._dev()))
        torch.cuda.synchronize(self.mesh.device)
        return {k: v.cpu().numpy() for k, v in out.items()}


class DeviceKd:
    """Flattened reference RopedKdTree (accel.py:561-710) on the mesh's device."""

    def __init__(self, mesh: DeviceMesh, arrays: dict):
        import ctypes
        self.mesh = mesh
        self.c_t = float(arrays.get("c_t", np.nan))
        a = {k: arrays[k] for k in ("axis", "left", "right", "ropes", "rope_cost", "prim_off",
                                    "prim_cnt", "prims")}
        a = {k: _i32(v) for k, v in a.items()}
        pos = _f64(arrays["pos"])
        box = _f64(arrays["box"]).reshape(-1, 4)
        h = ctypes.c_void_p()
        check(lib.mwt_kd_create(mesh.handle, len(a["axis"]), int(arrays["num_leaves"]), ptr(a["axis"]),
                                ptr(pos), ptr(a["left"]), ptr(a["right"]), ptr(box), ptr(a["ropes"]),
                                ptr(a["rope_cost"]), ptr(a["prim_off"]), ptr(a["prim_cnt"]),
                                len(a["prims"]), ptr(a["prims"]), ctypes.byref(h)), "kd_create")
        self._h = h
        self._keep = (a, pos, box)
        self.num_nodes = len(a["axis"])
        self.num_leaves = int(arrays["num_leaves"])

    @classmethod
    def from_file(cls, mesh: DeviceMesh, path: str) -> "DeviceKd":
        return cls(mesh, load_structure(path))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.mwt_kd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def trace_device(self, rays: torch.Tensor, start_leaf: torch.Tensor | None = None, stream=None) -> dict:
        """``start_leaf``: per-ray node indices of the leaves to start from
        (kd_intersect's start_leaf), else each ray's origin leaf."""
        rays, start_leaf = _held(rays, stream), _held(start_leaf, stream)
        n = rays.shape[0]
        d = rays.device
        out = dict(seg=torch.empty(n, dtype=torch.int32, device=d),
                   t=torch.empty(n, dtype=torch.float64, device=d),
                   u=torch.empty(n, dtype=torch.float64, device=d),
                   nodes=torch.empty(n, dtype=torch.int32, device=d),
                   ropes=torch.empty(n, dtype=torch.int32, device=d),
                   prims=torch.empty(n, dtype=torch.int32, device=d),
                   status=torch.empty(n, dtype=torch.int32, device=d))
        check(lib.mwt_kd_trace_dev(self._h, ptr(rays), ptr(start_leaf), n, ptr(out["seg"]), ptr(out["t"]),
                                   ptr(out["u"]), ptr(out["nodes"]), ptr(out["ropes"]),
                                   ptr(out["prims"]), ptr(out["status"]), _stream(stream, self.mesh.device)), "kd_trace")
        return out

    def trace(self, rays: np.ndarray, start_leaf: np.ndarray | None = None) -> dict:
        rays = _f64(rays).reshape(-1, 4)
        dev = self.mesh._dev()
        s = None if start_leaf is None else torch.from_numpy(_i32(start_leaf)).to(dev)
        out = self.trace_device(torch.from_numpy(rays).to(dev), s)
        torch.cuda.synchronize(self.mesh.device)
        return {k: v.cpu().numpy() for k, v in out.items()}


def _handles(meshes):
    import ctypes
    arr = (ctypes.c_void_p * len(meshes))(*[m.handle.value for m in meshes])
    return arr


def trace_generated_sharded(meshes, mode: int, box, seed: int, first: int, n: int) -> np.ndarray:
    """Rays [first, first+n) split over ``meshes`` (the same mesh on each
    device), one host thread per device; returns the summed histogram
    (mwt_trace_generated_sharded)."""
    import ctypes
    h = np.zeros(_lib.HIST_LEN, np.int64)
    arr = _handles(meshes)
    check(lib.mwt_trace_generated_sharded(ctypes.cast(arr, ctypes.c_void_p), len(meshes), int(mode),
                                          ptr(_f64(box)), int(seed), int(first), int(n), ptr(h)),
          "trace_generated_sharded")
    return h


def trace_sharded(meshes, rays: np.ndarray, start: np.ndarray | None = None) -> dict:
    """Host rays split over ``meshes`` (mwt_trace_host_sharded)."""
    import ctypes
    rays = _f64(rays).reshape(-1, 4)
    n = len(rays)
    out = dict(start=np.empty(n, np.int32), seg=np.empty(n, np.int32), t=np.empty(n),
               u=np.empty(n), steps=np.empty(n, np.int32), status=np.empty(n, np.uint32))
    s = _i32(start) if start is not None else None
    arr = _handles(meshes)
    check(lib.mwt_trace_host_sharded(ctypes.cast(arr, ctypes.c_void_p), len(meshes), ptr(rays), ptr(s), n,
                                     ptr(out["start"]), ptr(out["seg"]), ptr(out["t"]), ptr(out["u"]),
                                     ptr(out["steps"]), ptr(out["status"])), "trace_host_sharded")
    return out


def probe_l2_read_gbs(device: int = 0, nbytes: int = 64 << 20, passes: int = 200) -> float:
    """L2 read bandwidth of ``device`` (mwt_probe_l2_read): 128-bit streaming
    loads over an L2-resident buffer -- the walk's on-chip memory roof."""
    import ctypes
    g = ctypes.c_double(0.0)
    check(lib.mwt_probe_l2_read(int(device), int(nbytes), int(passes), ctypes.byref(g)), "probe_l2_read")
    return float(g.value)


def new_histogram(device: int = 0) -> torch.Tensor:
    return torch.zeros(_lib.HIST_LEN, dtype=torch.int64, device=torch.device("cuda", device))


def summarize_histogram(h) -> dict:
    h = np.asarray(h.cpu() if hasattr(h, "cpu") else h, dtype=np.int64)
    steps = h[:_lib.HIST_STEP_BINS]
    n = int(steps.sum())
    return {
        "rays": n,
        "hits": int(h[_lib.HIST_HIT]),
        "misses": int(h[_lib.HIST_MISS]),
        "steps_sum": int(h[_lib.HIST_STEPS_SUM]),
        "steps_per_ray": float(h[_lib.HIST_STEPS_SUM]) / n if n else 0.0,
        "max_steps_bin": int(np.nonzero(steps)[0].max()) if n else 0,
        "status": {name: int(h[_lib.HIST_STATUS0 + b]) for b, name in enumerate(_lib.STATUS_NAMES)},
    }


def pack_dry_run(scene: SceneArrays, tri: TriArrays) -> dict:
    """Run the K1 packer on the host only (no device): returns the packed walk
    words, locate words and seed grid exactly as mwt_mesh_create builds them."""
    import ctypes
    vxy = _f64(tri.vxy).reshape(-1, 2)
    vx, vy = _f64(vxy[:, 0]), _f64(vxy[:, 1])
    nt = len(tri.v)
    link = np.empty((nt, 4), np.int32)
    lnbr = np.empty((nt, 4), np.int32)
    res = ctypes.c_int32(0)
    args = (ptr(vx), ptr(vy), len(vx), ptr(_i32(tri.v)), ptr(_i32(tri.nbr)), ptr(_i32(tri.flag)), nt,
            ptr(_f64(scene.xy)), ptr(np.ascontiguousarray(scene.kind, dtype=np.uint8)), len(scene.kind))
    check(lib.mwt_pack_dry_run(*args, ptr(link), ptr(lnbr), ctypes.byref(res), None), "pack_dry_run")
    anchor = np.empty(max(res.value, 0) ** 2, np.int32)
    check(lib.mwt_pack_dry_run(*args, None, None, ctypes.byref(res), ptr(anchor)), "pack_dry_run")
    return dict(link=link, lnbr=lnbr, res=res.value, anchor=anchor.reshape(res.value, res.value))
