"""numpy host twin of the engine's seeded ray generator.

TEST INFRASTRUCTURE ONLY (see oracle/mwt_oracle.c header).  Bit-identical to
``orc_raygen`` (oracle/mwt_oracle.c) and to the device generator in
``paper_2112_05570_b200/csrc/mwt_kernels.cu``: counter-based SplitMix64 draws
keyed by (seed, stream, ray index) -- optionally with the top bits of every
draw shared by a group of consecutive rays (coherent order, include/mwt.h
MWT_RAYS_COHERENT); isotropic directions by unit-disk rejection
on 32-bit coordinates and angle doubling (one IEEE division, no cos/sin/sqrt);
the side / offset draws are the two 32-bit halves of one draw; and
only + - * / sqrt afterwards (numpy never fuses a*b+c).

The reference has no box-entry generator; its ``sample_rays``
(experiment.py:29-63) draws interior origins with PCG64 and cos/sin.  This
generator realises BASELINE.json's ray recipe: theta ~ U[0, 2pi), offset
uniform over the box's projected width, origin at the box entry point.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)

MODE_BOX_ENTRY = 0
MODE_INTERIOR = 1


def _mix(z):
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * C1
        z = (z ^ (z >> np.uint64(27))) * C2
        return z ^ (z >> np.uint64(31))


def ray_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        a = _mix(np.uint64(seed) + GOLDEN)
        return _mix(a ^ (np.uint64(stream) * STREAM_MUL))


GROUP_SALT = np.uint64(0x6A09E667F3BCC909)


def coherent(base: int, group_log2: int = 9, cell_bits: int = 12) -> int:
    """include/mwt.h MWT_RAYS_COHERENT(base, group_log2, cell_bits)."""
    return base | (group_log2 << 8) | (cell_bits << 16)


def decode(mode: int):
    """(base, group_log2, cell_bits) of a mode word; ValueError if malformed."""
    w = int(mode)
    base, gs, c = w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF
    if w < 0 or w >> 24 or base > 1 or gs > 40 or c > 16:
        raise ValueError(f"malformed ray generator mode word {mode:#x}")
    return base, gs, c


def raygen(mode: int, box, seed: int, first: int, n: int) -> np.ndarray:
    """(n, 4) float64 array of rays (ox, oy, dx, dy)."""
    base, gshift, c = decode(mode)
    key = ray_key(seed, base)
    idx = np.arange(first, first + n, dtype=np.uint64)
    s0 = key ^ idx  # per-ray SplitMix64 stream: draws mix64(s0 + (k + 1) * golden)
    h = ((1 << c) - 1) << (32 - c) if c else 0
    cmask = np.uint64((h << 32) | h)
    gs = _mix(key ^ GROUP_SALT) ^ (idx >> np.uint64(gshift))  # the group's stream

    def draw(k, sel=slice(None)):
        # draw k: mix64(s0 + (k + 1) * golden), top c bits of each half from the group's draw k
        with np.errstate(over="ignore"):
            z = _mix(s0[sel] + np.uint64(k + 1) * GOLDEN)
            if c:
                z = (z & ~cmask) | (_mix(gs[sel] + np.uint64(k + 1) * GOLDEN) & cmask)
        return z

    x = np.ones(n)
    y = np.zeros(n)
    r2 = np.ones(n)
    ok = np.zeros(n, dtype=bool)
    for a in range(64):
        todo = ~ok
        if not todo.any():
            break
        sel = np.nonzero(todo)[0]
        z = draw(a, sel)
        # one 64-bit draw per attempt -> two 32-bit coordinates in [-1, 1)
        xa = 2.0 * ((z >> np.uint64(32)).astype(np.float64) * 2.0 ** -32) - 1.0
        ya = 2.0 * ((z & np.uint64(0xFFFFFFFF)).astype(np.float64) * 2.0 ** -32) - 1.0
        ra = xa * xa + ya * ya
        acc = (ra <= 1.0) & (ra > 2.0 ** -60)
        x[sel] = xa
        y[sel] = ya
        r2[sel] = ra
        ok[sel[acc]] = True
    # angle doubling: (x^2 - y^2, 2xy) / r2 is isotropic and unit up to rounding
    inv = 1.0 / r2
    dx = np.where(ok, (x * x - y * y) * inv, 1.0)
    dy = np.where(ok, (2.0 * x * y) * inv, 0.0)
    x0, y0, x1, y1 = (float(v) for v in box)
    W, H = x1 - x0, y1 - y0
    zuv = draw(128)  # draw 128: u, v = its 32-bit halves * 2^-32
    u = (zuv >> np.uint64(32)).astype(np.float64) * 2.0 ** -32
    v = (zuv & np.uint64(0xFFFFFFFF)).astype(np.float64) * 2.0 ** -32
    if base == MODE_INTERIOR:
        ox = x0 + W * u
        oy = y0 + H * v
    else:
        # entry side with probability proportional to its projected length,
        # uniform position along it (isotropic lines through the box)
        wx = H * np.abs(dx)
        wy = W * np.abs(dy)
        xside = u * (wx + wy) < wx
        ox = np.where(xside, np.where(dx > 0.0, x0, x1), x0 + W * v)
        oy = np.where(xside, y0 + H * v, np.where(dy > 0.0, y0, y1))
    return np.ascontiguousarray(np.stack([ox, oy, dx, dy], axis=1))
