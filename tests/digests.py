"""Per-chunk digests of per-ray walk results (tests/golden/make_digests.py
records the reference's; the tests recompute them from the oracle and the
engine).  d_walk hashes seg (int32; -1 miss, -2 TraversalError) | t (float64,
every NaN as one pattern) | steps (int32; 0 on TraversalError); d_start
hashes the start triangles (int32)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_NAN = np.frombuffer(np.uint64(0x7FF8000000000000).tobytes(), np.float64)[0]


def normalize(seg, t, steps, error=None):
    seg = np.asarray(seg, np.int32).copy()
    t = np.asarray(t, np.float64).copy()
    steps = np.asarray(steps, np.int32).copy()
    if error is not None:
        e = np.asarray(error).astype(bool)
        seg[e] = -2
        t[e] = np.nan
        steps[e] = 0
    t[np.isnan(t)] = _NAN
    return seg, t, steps


def digest_walk(seg, t, steps) -> str:
    seg, t, steps = normalize(seg, t, steps)
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(seg).tobytes())
    h.update(np.ascontiguousarray(t).tobytes())
    h.update(np.ascontiguousarray(steps).tobytes())
    return h.hexdigest()


def digest_start(start) -> str:
    return hashlib.sha256(np.ascontiguousarray(start, np.int32).tobytes()).hexdigest()


def load(mesh: str):
    p = os.path.join(GOLDEN, f"digests_{mesh}.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh)


def chunk_digests(seg, t, steps, start, error, chunk):
    """[(d_walk, d_start)] per chunk of a part's per-ray arrays."""
    seg, t, steps = normalize(seg, t, steps, error)
    out = []
    for lo in range(0, len(seg), chunk):
        hi = lo + chunk
        out.append((digest_walk(seg[lo:hi], t[lo:hi], steps[lo:hi]),
                    None if start is None else digest_start(start[lo:hi])))
    return out
