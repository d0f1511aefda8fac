"""Host-side value types of the ray-query API.

When the reference package is importable its own types are used, so a
caller's `Point` / `Segment` / `Ray` objects and the drop-in's results are the
same classes.  Otherwise this module supplies stand-ins with the same fields,
values and arithmetic (reference geometry.py:28-78):

  Point          (x, y) named tuple
  SegmentKind    GEOMETRY = "G", BOUNDARY = "B"
  Segment        a, b, kind; length, point_at(u), param_of(p)  (builds `Hit.point`)
  Ray            origin, direction, start_tri; a direction whose length differs
                 from 1 by more than 1e-12 is rescaled by its hypot

No geometric predicate runs on the host: those live in the CUDA kernels.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple, Optional

try:  # the reference's own types (the drop-in's results then compare equal by type)
    from mintri.geometry import Point, Ray, Segment, SegmentKind  # type: ignore  # noqa: F401
    REFERENCE_TYPES = True
except ImportError:
    REFERENCE_TYPES = False

    class Point(NamedTuple):  # type: ignore[no-redef]
        x: float
        y: float

    class SegmentKind(Enum):  # type: ignore[no-redef]
        GEOMETRY = "G"
        BOUNDARY = "B"

    def _delta(a: Point, b: Point) -> tuple[float, float]:
        return b.x - a.x, b.y - a.y

    @dataclass(frozen=True)
    class Segment:  # type: ignore[no-redef]
        a: Point
        b: Point
        kind: SegmentKind = SegmentKind.GEOMETRY

        def __post_init__(self) -> None:
            if self.a == self.b:
                raise ValueError(f"degenerate segment at {self.a}")

        @property
        def length(self) -> float:
            return math.hypot(*_delta(self.a, self.b))

        def point_at(self, u: float) -> Point:
            # a + u (b - a) per component, in this operation order (bit-exact Hit.point)
            ex, ey = _delta(self.a, self.b)
            return Point(self.a.x + u * ex, self.a.y + u * ey)

        def param_of(self, p: Point) -> float:
            ex, ey = _delta(self.a, self.b)
            return ((p.x - self.a.x) * ex + (p.y - self.a.y) * ey) / (ex * ex + ey * ey)

    def _direction(d) -> Point:
        dx, dy = d
        n = math.hypot(dx, dy)
        if n == 0.0 or not math.isfinite(n):
            raise ValueError("ray direction must be a nonzero finite vector")
        return Point(dx / n, dy / n) if abs(n - 1.0) > 1e-12 else Point(dx, dy)

    @dataclass
    class Ray:  # type: ignore[no-redef]
        origin: Point
        direction: Point
        start_tri: Optional[int] = None

        def __post_init__(self) -> None:
            self.origin = Point(*self.origin)
            self.direction = _direction(self.direction)

        @classmethod
        def from_angle(cls, origin: Point, theta: float) -> "Ray":
            return cls(origin, Point(math.cos(theta), math.sin(theta)))
