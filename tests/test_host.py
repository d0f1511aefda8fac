"""Host-side tests (no GPU): the C ABI library, the reference-format readers,
the K1 packer's host dry run, and the product/oracle separation."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import CONFIGS, ROOT, fixture_paths


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mwt.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mwt_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2112_05570_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_lib.lib, s), f"libmwt.so does not export {s}"
        assert s in _lib.SIGNATURES, f"ctypes binding missing for {s}"
    assert set(_lib.SIGNATURES) == set(syms)
    assert _lib.lib.mwt_abi_version() == _lib.ABI_VERSION


def test_invalid_arguments_fail_loudly():
    from paper_2112_05570_b200 import _lib
    h = ctypes.c_void_p()
    rc = _lib.lib.mwt_mesh_create(None, None, -1, None, None, None, 1, None, None, 0, 0, ctypes.byref(h))
    assert rc == -1 and b"mesh_create" in _lib.lib.mwt_last_error()
    with pytest.raises(_lib.MwtError):
        _lib.check(rc, "mesh_create")
    assert _lib.lib.mwt_trace_host(None, None, None, 1, None, None, None, None, None, None) == -1
    # the single-process sharded entry points validate before touching a device
    h = np.zeros(_lib.HIST_LEN, np.int64)
    box = np.array([0.0, 0.0, 1.0, 1.0])
    assert _lib.lib.mwt_trace_generated_sharded(None, 1, 0, _lib.ptr(box), 0, 0, 10, _lib.ptr(h)) == -1
    assert b"trace_generated_sharded" in _lib.lib.mwt_last_error()
    none2 = (ctypes.c_void_p * 2)(None, None)
    assert _lib.lib.mwt_trace_generated_sharded(ctypes.cast(none2, ctypes.c_void_p), 2, 0, _lib.ptr(box),
                                                0, 0, 10, _lib.ptr(h)) == -1
    assert _lib.lib.mwt_trace_generated_sharded(ctypes.cast(none2, ctypes.c_void_p), 0, 0, _lib.ptr(box),
                                                0, 0, 10, _lib.ptr(h)) == -1
    assert _lib.lib.mwt_trace_host_sharded(None, 1, None, None, 5, None, None, None, None, None,
                                           None) == -1
    assert b"trace_host_sharded" in _lib.lib.mwt_last_error()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2112_05570_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "libmwt_oracle" not in src and "orc_" not in src, f
                assert not re.search(r'#include\s+"[^"]*oracle', src), f


@pytest.mark.parametrize("cfg", CONFIGS)
def test_formats_match_oracle_reader(cfg):
    from oracle import oracle as orc
    from paper_2112_05570_b200.formats import load_scene, load_tri, parse_scene_text, serialize_scene
    paths = fixture_paths(cfg, "mwt") or fixture_paths(cfg, "cdt")
    sc, tri = load_scene(paths[0]), load_tri(paths[1])
    osc, otri = orc.load_scene(paths[0]), orc.load_tri(paths[1])
    assert np.array_equal(sc.xy[:, 0].view(np.uint64), osc.ax.view(np.uint64))
    assert np.array_equal(sc.xy[:, 3].view(np.uint64), osc.by.view(np.uint64))
    assert np.array_equal(sc.kind, osc.kind)
    assert np.array_equal(tri.vxy[:, 0], otri.vx) and np.array_equal(tri.v, otri.v)
    assert np.array_equal(tri.nbr, otri.nbr) and np.array_equal(tri.flag, otri.flag)
    # '%.17g' round trip is bit exact (scene.py:118-133)
    sc2 = parse_scene_text(serialize_scene(sc))
    assert np.array_equal(sc2.xy.view(np.uint64), sc.xy.view(np.uint64))
    # geometry first, then the 4 boundary sides (scene.py:5-6, :20-22)
    assert sc.kind[-4:].tolist() == [1, 1, 1, 1] and (sc.kind[:-4] == 0).all()


def test_format_errors():
    from paper_2112_05570_b200.formats import FormatError, parse_scene_text, parse_tri_text
    with pytest.raises(FormatError):
        parse_scene_text("not a scene\n")
    with pytest.raises(FormatError):
        parse_scene_text("mintri-scene v1\nsegments 2\n0 0 1 1 G\n")
    with pytest.raises(FormatError):
        parse_tri_text("mintri-tri v1\nvertices 1\n0 0 0 -1\n")


@pytest.mark.parametrize("cfg", CONFIGS)
def test_packer_dry_run(cfg):
    """K1 on the host: walk words decode back to the reference's nbr/flag
    tables with mirror indices, and every seed-grid cell centre lies in its
    triangle."""
    from paper_2112_05570_b200.engine import pack_dry_run
    from paper_2112_05570_b200.formats import load_scene, load_tri
    paths = fixture_paths(cfg, "mwt") or fixture_paths(cfg, "cdt")
    sc, tri = load_scene(paths[0]), load_tri(paths[1])
    p = pack_dry_run(sc, tri)
    link = p["link"][:, :3].view(np.uint32)
    lnbr = p["lnbr"][:, :3]
    stop = (link & 0x80000000) != 0
    assert np.array_equal(stop, (tri.flag != -1) | (tri.nbr == -1))
    internal = ~stop
    # internal word = step-record index 3 * nbr + mirror
    assert np.array_equal((link[internal] // 3).astype(np.int32), tri.nbr[internal])
    assert np.array_equal((link[internal] % 3).astype(np.int32), p["lnbr"][:, :3][internal] & 3)
    assert np.array_equal(lnbr >= 0, tri.nbr >= 0)
    has = lnbr >= 0
    assert np.array_equal(lnbr[has] >> 2, tri.nbr[has])
    # mirror j: neighbour's edge j has the same two vertices reversed
    t, i = np.nonzero(has)
    nb, j = lnbr[t, i] >> 2, lnbr[t, i] & 3
    a, b = tri.v[t, (i + 1) % 3], tri.v[t, (i + 2) % 3]
    assert np.array_equal(tri.v[nb, (j + 1) % 3], b) and np.array_equal(tri.v[nb, (j + 2) % 3], a)
    # constrained words carry the scene segment id and its kind
    c = (tri.flag != -1)
    assert np.array_equal((link[c] & 0x3FFFFFFF).astype(np.int32), tri.flag[c])
    assert np.array_equal(((link[c] >> 30) & 1).astype(np.uint8), sc.kind[tri.flag[c]])
    # seed grid: each cell centre inside (tolerance 1e-15) its triangle
    res = p["res"]
    cy, cx = np.mgrid[0:res, 0:res]
    px, py = (cx + 0.5) * (1.0 / res), (cy + 0.5) * (1.0 / res)
    tv = tri.v[p["anchor"]]
    P = tri.vxy[tv]  # (res, res, 3, 2)
    for k in range(3):
        A, B = P[:, :, (k + 1) % 3], P[:, :, (k + 2) % 3]
        s = (B[..., 0] - A[..., 0]) * (py - A[..., 1]) - (B[..., 1] - A[..., 1]) * (px - A[..., 0])
        assert (s >= -1e-15).all()


def test_packer_rejects_broken_topology():
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import pack_dry_run
    from paper_2112_05570_b200.formats import load_scene, load_tri
    paths = fixture_paths("lines64", "cdt")
    sc, tri = load_scene(paths[0]), load_tri(paths[1])
    bad = tri.nbr.copy()
    t = int(np.nonzero(bad[:, 0] >= 0)[0][0])
    bad[t, 0] = (bad[t, 0] + 1) % len(bad)
    tri.nbr = bad
    with pytest.raises(_lib.MwtError, match="symmetry"):
        pack_dry_run(sc, tri)


def test_shard_ranges():
    from paper_2112_05570_b200.sharding import strong_shard, weak_shard
    for world in (1, 2, 3, 8):
        parts = [strong_shard(r, world, 1000003) for r in range(world)]
        assert parts[0].first == 0 and sum(p.count for p in parts) == 1000003
        assert all(parts[k].first + parts[k].count == parts[k + 1].first for k in range(world - 1))
        assert [weak_shard(r, world, 10).first for r in range(world)] == [10 * r for r in range(world)]


def test_binary_mesh_roundtrip(tmp_path):
    """mwt-mesh v1: text -> binary -> identical SoA, and
    the packer produces the same walk words from either."""
    import ctypes
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.formats import (FormatError, load_mesh_binary, load_scene, load_tri,
                                               save_mesh_binary)
    sp, tp = fixture_paths("lines1024", "mwt")
    scene, tri = load_scene(sp), load_tri(tp)
    save_mesh_binary(str(tmp_path / "m"), scene, tri)
    s2, t2 = load_mesh_binary(str(tmp_path / "m"))
    assert np.array_equal(s2.xy.view(np.uint64), scene.xy.view(np.uint64))
    assert np.array_equal(s2.kind, scene.kind)
    assert np.array_equal(t2.vxy.view(np.uint64), tri.vxy.view(np.uint64))
    for k in ("v", "nbr", "flag"):
        assert np.array_equal(getattr(t2, k), getattr(tri, k))

    def words(sc, tr):
        vxy = np.ascontiguousarray(tr.vxy, np.float64).reshape(-1, 2)
        vx, vy = np.ascontiguousarray(vxy[:, 0]), np.ascontiguousarray(vxy[:, 1])
        link = np.empty(4 * len(tr.v), np.int32)
        P = _lib.ptr
        i32 = lambda a: np.ascontiguousarray(a, np.int32)  # noqa: E731
        _lib.check(_lib.lib.mwt_pack_dry_run(
            P(vx), P(vy), len(vx), P(i32(tr.v)), P(i32(tr.nbr)), P(i32(tr.flag)), len(tr.v),
            P(np.ascontiguousarray(sc.xy, np.float64)), P(np.ascontiguousarray(sc.kind, np.uint8)),
            len(sc.kind), P(link), None, None, None), "dry run")
        return link
    assert np.array_equal(words(scene, tri), words(s2, t2))
    (tmp_path / "bad").mkdir()
    (tmp_path / "bad" / "format.txt").write_text('{"format": "other"}\n')
    with pytest.raises(FormatError):
        load_mesh_binary(str(tmp_path / "bad"))
