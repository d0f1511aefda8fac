"""Host-side value types of the ray-query API, mirroring the reference's
geometry.py so existing callers keep working:

  Point            geometry.py:28-30
  SegmentKind      geometry.py:33-35
  Segment          geometry.py:38-59  (point_at / param_of used to build Hit)
  Ray              geometry.py:62-78  (renormalises only if |hypot-1| > 1e-12)

These are plain data holders; no geometry predicate runs on the host -- the
predicates live in the CUDA kernels.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple, Optional


class Point(NamedTuple):
    x: float
    y: float


class SegmentKind(Enum):
    GEOMETRY = "G"
    BOUNDARY = "B"


@dataclass(frozen=True)
class Segment:
    a: Point
    b: Point
    kind: SegmentKind = SegmentKind.GEOMETRY

    def __post_init__(self) -> None:
        if self.a == self.b:
            raise ValueError(f"degenerate segment at {self.a}")

    @property
    def length(self) -> float:
        return math.hypot(self.b.x - self.a.x, self.b.y - self.a.y)

    def point_at(self, u: float) -> Point:
        return Point(self.a.x + u * (self.b.x - self.a.x),
                     self.a.y + u * (self.b.y - self.a.y))

    def param_of(self, p: Point) -> float:
        ex, ey = self.b.x - self.a.x, self.b.y - self.a.y
        return ((p.x - self.a.x) * ex + (p.y - self.a.y) * ey) / (ex * ex + ey * ey)


@dataclass
class Ray:
    origin: Point
    direction: Point
    start_tri: Optional[int] = None

    def __post_init__(self) -> None:
        dx, dy = self.direction
        n = math.hypot(dx, dy)
        if not math.isfinite(n) or n == 0.0:
            raise ValueError("ray direction must be a nonzero finite vector")
        if abs(n - 1.0) > 1e-12:
            self.direction = Point(dx / n, dy / n)
        self.origin = Point(*self.origin)
        self.direction = Point(*self.direction)

    @classmethod
    def from_angle(cls, origin: Point, theta: float) -> "Ray":
        return cls(origin, Point(math.cos(theta), math.sin(theta)))
