"""Readers/writers of the reference's text formats, producing the packer's SoA
input directly (numpy), plus the flattened kd-tree / BVH archives.

  mintri-scene v1   scene.py:118-165  (serialize_scene / parse_scene)
  mintri-tri v1     trimesh.py:1277-1337 (save_triangulation / load_triangulation)
  mwt-bvh v1 (.npz) flattened reference Bvh   (fixtures/gen_fixtures.py flatten_bvh)
  mwt-kd v1 (.npz)  flattened RopedKdTree     (fixtures/gen_fixtures.py flatten_kd)
  mwt-mesh v1       binary SoA of a scene + triangulation: a
                    directory of raw .npy arrays, memory-mapped on load -- the
                    packer's input without text parsing

Ids follow the files exactly: scene segments in file order (geometry first,
then the four boundary sides, scene.py:5-6), triangles and vertices in the
compacted file order (trimesh.py:1289-1305).  '%.17g' text round-trips fp64
bit-exactly, so the packed mesh equals the reference's in-memory one.
"""
from __future__ import annotations

import gzip
from dataclasses import dataclass, field

import numpy as np

SCENE_HEADER = "mintri-scene v1"
TRI_HEADER = "mintri-tri v1"


class FormatError(ValueError):
    pass


def _open_text(path: str) -> str:
    if path.endswith(".gz"):
        with gzip.open(path, "rt") as fh:
            return fh.read()
    with open(path) as fh:
        return fh.read()


@dataclass
class SceneArrays:
    """Scene segments as SoA: xy (S, 4) float64 = (ax, ay, bx, by); kind (S,)
    uint8 = 0 GEOMETRY / 1 BOUNDARY."""
    xy: np.ndarray
    kind: np.ndarray
    name: str = "scene"
    provenance: str = ""

    @property
    def num_segments(self) -> int:
        return len(self.kind)

    def geometry_ids(self) -> np.ndarray:
        return np.nonzero(self.kind == 0)[0]


@dataclass
class TriArrays:
    """Triangulation in the reference data model (trimesh.py:39-60):
    vxy (V, 2) float64; v, nbr, flag (T, 3) int32 (nbr -1 = None,
    flag -1 = INTERNAL or a scene segment id); dof/vseg per vertex."""
    vxy: np.ndarray
    v: np.ndarray
    nbr: np.ndarray
    flag: np.ndarray
    dof: np.ndarray = field(default=None)
    vseg: np.ndarray = field(default=None)
    scene_name: str = ""

    @property
    def num_triangles(self) -> int:
        return len(self.v)

    @property
    def num_vertices(self) -> int:
        return len(self.vxy)


def parse_scene_text(text: str) -> SceneArrays:
    """scene.py:135-165."""
    lines = text.splitlines()
    if not lines or lines[0].strip() != SCENE_HEADER:
        raise FormatError(f"not a scene file (expected header {SCENE_HEADER!r})")
    name, provenance, count, idx = "scene", "", None, 1
    while idx < len(lines):
        line = lines[idx].strip()
        idx += 1
        if line.startswith("name "):
            name = line[5:]
        elif line.startswith("provenance"):
            provenance = line[10:].strip()
        elif line.startswith("segments "):
            count = int(line.split()[1])
            break
        elif line:
            raise FormatError(f"line {idx}: unexpected {line!r}")
    if count is None:
        raise FormatError("missing 'segments' section")
    body = lines[idx:idx + count]
    if len(body) < count:
        raise FormatError(f"expected {count} segments, file ends early")
    xy = np.empty((count, 4), dtype=np.float64)
    kind = np.empty(count, dtype=np.uint8)
    for k, line in enumerate(body):
        parts = line.split()
        if len(parts) != 5:
            raise FormatError(f"line {idx + k + 1}: expected 'x1 y1 x2 y2 kind'")
        xy[k] = [float(p) for p in parts[:4]]
        if parts[4] not in ("G", "B"):
            raise FormatError(f"line {idx + k + 1}: bad segment kind {parts[4]!r}")
        kind[k] = 0 if parts[4] == "G" else 1
    return SceneArrays(xy, kind, name, provenance)


def load_scene(path: str) -> SceneArrays:
    return parse_scene_text(_open_text(path))


def _fmt(x: float) -> str:
    return format(float(x), ".17g")


def serialize_scene(sc: SceneArrays) -> str:
    lines = [SCENE_HEADER, f"name {sc.name}", f"provenance {sc.provenance}",
             f"segments {sc.num_segments}"]
    for (ax, ay, bx, by), k in zip(sc.xy, sc.kind):
        lines.append(f"{_fmt(ax)} {_fmt(ay)} {_fmt(bx)} {_fmt(by)} {'G' if k == 0 else 'B'}")
    return "\n".join(lines) + "\n"


def parse_tri_text(text: str) -> TriArrays:
    """trimesh.py:1309-1337."""
    lines = text.splitlines()
    if not lines or lines[0].strip() != TRI_HEADER:
        raise FormatError(f"not a triangulation file (expected {TRI_HEADER!r})")
    k = 1
    scene_name = ""
    if k < len(lines) and lines[k].startswith("scene "):
        scene_name = lines[k][6:]
        k += 1
    if k >= len(lines) or not lines[k].startswith("vertices "):
        raise FormatError(f"line {k + 1}: expected vertex section")
    nv = int(lines[k].split()[1])
    k += 1
    vrows = [ln.split() for ln in lines[k:k + nv]]
    if len(vrows) != nv or any(len(r) != 4 for r in vrows):
        raise FormatError("vertex section ends early")
    vxy = np.array([[float(r[0]), float(r[1])] for r in vrows], dtype=np.float64).reshape(-1, 2)
    dof = np.array([int(r[2]) for r in vrows], dtype=np.int32)
    vseg = np.array([int(r[3]) for r in vrows], dtype=np.int32)
    k += nv
    if k >= len(lines) or not lines[k].startswith("triangles "):
        raise FormatError(f"line {k + 1}: expected triangle section")
    nt = int(lines[k].split()[1])
    k += 1
    body = lines[k:k + nt]
    if len(body) != nt:
        raise FormatError("triangle section ends early")
    tt = np.array([[int(s) for s in ln.split()] for ln in body], dtype=np.int64).reshape(-1, 9)
    if tt.size and (tt.min() < -1 or tt.max() >= 2 ** 31):
        raise FormatError("triangle index out of range")
    tt = tt.astype(np.int32)
    return TriArrays(vxy, np.ascontiguousarray(tt[:, 0:3]), np.ascontiguousarray(tt[:, 3:6]),
                     np.ascontiguousarray(tt[:, 6:9]), dof, vseg, scene_name)


def load_tri(path: str) -> TriArrays:
    return parse_tri_text(_open_text(path))


def load_structure(path: str) -> dict:
    """A flattened reference Bvh or RopedKdTree (.npz)."""
    with np.load(path) as z:
        out = {k: z[k] for k in z.files}
    fmt = str(out.get("format", ""))
    if fmt not in ("mwt-bvh v1", "mwt-kd v1"):
        raise FormatError(f"{path}: unknown structure format {fmt!r}")
    return out


# ---------------------------------------------------------------------------
# mwt-mesh v1: binary SoA (one .npy per array, memory-mappable)

MESH_FORMAT = "mwt-mesh v1"
_MESH_ARRAYS = {  # name: (dtype, columns)
    "seg_xy": (np.float64, 4), "seg_kind": (np.uint8, 0),
    "vxy": (np.float64, 2), "tri_v": (np.int32, 3), "tri_nbr": (np.int32, 3),
    "tri_flag": (np.int32, 3),
}


def save_mesh_binary(path: str, scene: SceneArrays, tri: TriArrays) -> None:
    """Write ``path/`` with format.txt and one .npy per SoA array."""
    import json
    import os
    os.makedirs(path, exist_ok=True)
    arrays = {"seg_xy": scene.xy, "seg_kind": scene.kind, "vxy": tri.vxy, "tri_v": tri.v,
              "tri_nbr": tri.nbr, "tri_flag": tri.flag}
    for name, (dt, cols) in _MESH_ARRAYS.items():
        a = np.ascontiguousarray(arrays[name], dtype=dt)
        if cols:
            a = a.reshape(-1, cols)
        np.save(os.path.join(path, name + ".npy"), a)
    meta = {"format": MESH_FORMAT, "scene_name": scene.name, "num_segments": int(scene.num_segments),
            "num_vertices": int(tri.num_vertices), "num_triangles": int(tri.num_triangles)}
    with open(os.path.join(path, "format.txt"), "w") as fh:
        fh.write(json.dumps(meta) + "\n")


def load_mesh_binary(path: str, mmap: bool = True):
    """Read a ``mwt-mesh v1`` directory: (SceneArrays, TriArrays), arrays
    memory-mapped read-only when ``mmap``."""
    import json
    import os
    try:
        with open(os.path.join(path, "format.txt")) as fh:
            meta = json.loads(fh.read())
    except (OSError, ValueError) as e:
        raise FormatError(f"{path}: not a {MESH_FORMAT} directory ({e})") from None
    if meta.get("format") != MESH_FORMAT:
        raise FormatError(f"{path}: unknown mesh format {meta.get('format')!r}")
    a = {}
    for name, (dt, cols) in _MESH_ARRAYS.items():
        x = np.load(os.path.join(path, name + ".npy"), mmap_mode="r" if mmap else None)
        if x.dtype != dt or (cols and (x.ndim != 2 or x.shape[1] != cols)):
            raise FormatError(f"{path}/{name}.npy: expected {np.dtype(dt).name} with {cols} columns")
        a[name] = x
    if len(a["seg_xy"]) != meta["num_segments"] or len(a["tri_v"]) != meta["num_triangles"] or \
            len(a["vxy"]) != meta["num_vertices"] or len(a["seg_kind"]) != meta["num_segments"]:
        raise FormatError(f"{path}: array sizes disagree with format.txt")
    scene = SceneArrays(a["seg_xy"], a["seg_kind"], meta.get("scene_name", "scene"))
    tri = TriArrays(a["vxy"], a["tri_v"], a["tri_nbr"], a["tri_flag"], scene_name=scene.name)
    return scene, tri
