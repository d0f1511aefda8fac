"""Minimal host data model mirroring the reference's, for callers that do not
have `mintri` at hand (e.g. on a GPU box):

  Scene, Scene.load / save           scene.py:29-71, :118-165
  Triangulation (verts / tris / scene, pos, alive_tris, num_tris)
                                     trimesh.py:39-60, :93-150
  load_triangulation(path, scene)    trimesh.py:1309-1337

Objects from this module and the reference's own objects are interchangeable
as arguments of paper_2112_05570_b200.accel.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, Optional

from .formats import SceneArrays, TriArrays, load_scene, load_tri, serialize_scene
from .geometry import Point, Segment, SegmentKind

INTERNAL = -1


@dataclass
class Scene:
    segments: list
    name: str = "scene"
    provenance: str = ""

    @property
    def geometry(self) -> list:
        return [s for s in self.segments if s.kind is SegmentKind.GEOMETRY]

    def geometry_ids(self) -> list:
        return [i for i, s in enumerate(self.segments) if s.kind is SegmentKind.GEOMETRY]

    @classmethod
    def from_arrays(cls, a: SceneArrays) -> "Scene":
        segs = [Segment(Point(r[0], r[1]), Point(r[2], r[3]),
                        SegmentKind.GEOMETRY if k == 0 else SegmentKind.BOUNDARY)
                for r, k in zip(a.xy.tolist(), a.kind.tolist())]
        return cls(segs, a.name, a.provenance)

    def to_arrays(self) -> SceneArrays:
        import numpy as np
        xy = np.array([[s.a.x, s.a.y, s.b.x, s.b.y] for s in self.segments], np.float64).reshape(-1, 4)
        kind = np.array([0 if s.kind is SegmentKind.GEOMETRY else 1 for s in self.segments], np.uint8)
        return SceneArrays(xy, kind, self.name, self.provenance)

    @classmethod
    def load(cls, path: str) -> "Scene":
        return cls.from_arrays(load_scene(path))

    def save(self, path: str) -> None:
        with open(path, "w") as fh:
            fh.write(serialize_scene(self.to_arrays()))


class Vertex:
    __slots__ = ("x", "y", "dof", "seg", "alive")

    def __init__(self, x: float, y: float, dof: int = 0, seg: Optional[int] = None):
        self.x, self.y, self.dof, self.seg, self.alive = x, y, dof, seg, True


class Tri:
    __slots__ = ("v", "nbr", "flag")

    def __init__(self, v, nbr, flag):
        self.v, self.nbr, self.flag = v, nbr, flag


class Triangulation:
    def __init__(self, scene):
        self.scene = scene
        self.verts: list = []
        self.tris: list = []

    @classmethod
    def from_arrays(cls, scene, t: TriArrays) -> "Triangulation":
        tri = cls(scene)
        dof = t.dof if t.dof is not None else [0] * len(t.vxy)
        vseg = t.vseg if t.vseg is not None else [-1] * len(t.vxy)
        tri.verts = [Vertex(float(x), float(y), int(d), None if s == -1 else int(s))
                     for (x, y), d, s in zip(t.vxy.tolist(), list(dof), list(vseg))]
        tri.tris = [Tri(list(v), [None if n == -1 else n for n in nb], list(f))
                    for v, nb, f in zip(t.v.tolist(), t.nbr.tolist(), t.flag.tolist())]
        return tri

    def pos(self, vid: int) -> Point:
        v = self.verts[vid]
        return Point(v.x, v.y)

    def alive_tris(self) -> Iterator[int]:
        for tid, t in enumerate(self.tris):
            if t is not None:
                yield tid

    @property
    def num_tris(self) -> int:
        return sum(1 for t in self.tris if t is not None)

    def edge_verts(self, t: int, i: int):
        v = self.tris[t].v
        return v[(i + 1) % 3], v[(i + 2) % 3]


def load_triangulation(path: str, scene) -> Triangulation:
    return Triangulation.from_arrays(scene, load_tri(path))
