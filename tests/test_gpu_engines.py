"""Device engines against the oracle at scale, the drop-in API, histograms,
edge cases and full-size properties."""
import os
import struct

import numpy as np
import pytest

from conftest import CONFIGS, box_of, fixture_paths

pytestmark = pytest.mark.gpu

C_T_GRID = (0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0)


@pytest.mark.parametrize("cfg", CONFIGS[1:])
@pytest.mark.parametrize("mode", [0, 1])
def test_bvh_kd_match_oracle_all_ct(cfg, mode):
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceBvh, DeviceKd, DeviceMesh
    from paper_2112_05570_b200.formats import load_scene
    paths = fixture_paths(cfg, "cdt")
    d = os.path.dirname(paths[0])
    m = DeviceMesh(load_scene(paths[0]), None)
    om = orc.Mesh.from_files(paths[0], None)
    rays = orc.raygen(mode, box_of(cfg), 5, 0, 1 << 14)
    for ct in C_T_GRID:
        arr = orc.load_npz(os.path.join(d, f"bvh_ct{ct:g}.npz"))
        got, ref = DeviceBvh(m, arr).trace(rays), orc.Bvh(om, arr).trace(rays)
        for k in ("seg", "node_tests", "prim_tests"):
            assert np.array_equal(got[k], ref[k]), (ct, k)
        h = ref["seg"] >= 0
        assert np.array_equal(got["t"][h], ref["t"][h])
        arr = orc.load_npz(os.path.join(d, f"kd_ct{ct:g}.npz"))
        got, ref = DeviceKd(m, arr).trace(rays), orc.Kd(om, arr).trace(rays)
        for k in ("seg", "nodes", "ropes", "prims"):
            assert np.array_equal(got[k], ref[k]), (ct, k)
        assert np.array_equal(got["status"].view(np.uint32) & 1, ref["status"] & 1)


@pytest.mark.parametrize("cfg", CONFIGS)
def test_brute_force_matches_oracle(cfg):
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    paths = fixture_paths(cfg, "cdt")
    m = DeviceMesh.from_files(*paths)
    om = orc.Mesh.from_files(*paths)
    rays = orc.raygen(1, box_of(cfg), 9, 0, 4096)
    got, ref = m.brute_force(rays), om.brute_force(rays)
    assert np.array_equal(got["seg"], ref["seg"])
    h = ref["seg"] >= 0
    assert np.array_equal(got["t"][h], ref["t"][h])
    # the walk finds the same closest hits as the brute-force oracle (test_accel.py:47-59)
    w = m.trace(rays)
    assert np.array_equal(w["seg"], ref["seg"])
    assert np.allclose(w["t"][h], ref["t"][h], rtol=1e-9, atol=0)


def test_locate_matches_oracle_everywhere():
    """start triangles for origins on vertices, edge midpoints, centroids and
    random points (test_accel.py:74-101)."""
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    from paper_2112_05570_b200.formats import load_tri
    for cfg in ("lines64", "floorplan64"):
        paths = fixture_paths(cfg, "mwt")
        m, om, tri = DeviceMesh.from_files(*paths), orc.Mesh.from_files(*paths), load_tri(paths[1])
        P = tri.vxy[tri.v]
        pts = [tri.vxy, P.mean(axis=1), 0.5 * (P[:, 0] + P[:, 1]), 0.5 * (P[:, 1] + P[:, 2]),
               np.random.default_rng(1).random((20000, 2))]
        pts = np.ascontiguousarray(np.concatenate(pts))
        got, gst = m.locate(pts)
        ref, rst = om.locate(pts)
        assert np.array_equal(got, ref)
        assert np.array_equal(gst & 128, rst & 128)  # tie flag


@pytest.mark.parametrize("cfg", ["lines1024", "hair512"])  # record table / per-triangle table
def test_generated_kernel_equals_explicit_rays_and_histogram(cfg):
    import torch
    from paper_2112_05570_b200.engine import DeviceMesh, new_histogram
    from paper_2112_05570_b200.sharding import histogram_host
    paths = fixture_paths(cfg, "mwt") or fixture_paths(cfg, "cdt")
    m = DeviceMesh.from_files(*paths)
    n = (1 << 18) + 77  # (first = 777, n: neither a multiple of the 512-ray grabs nor of 128)
    from oracle import raygen as rg
    for mode in (0, 1, rg.coherent(0), rg.coherent(1)):
        h = new_histogram()
        gen = m.trace_generated_device(mode, (0, 0, 1, 1), 3, 777, n, outputs=True, hist=h)
        rays = m.raygen_device(mode, (0, 0, 1, 1), 3, 777, n)
        ex = m.trace_device(rays)
        torch.cuda.synchronize()
        for k in ("seg", "steps"):
            assert torch.equal(gen[k], ex[k])
        hit = ex["seg"] >= 0
        assert torch.equal(gen["t"][hit], ex["t"][hit])
        ref = histogram_host(ex["seg"].cpu().numpy(), ex["steps"].cpu().numpy(),
                             ex["status"].cpu().numpy().view(np.uint32))
        assert np.array_equal(h.cpu().numpy(), ref)
        h2 = new_histogram()
        m_hist = __import__("paper_2112_05570_b200._lib", fromlist=["x"])
        m_hist.check(m_hist.lib.mwt_histogram_dev(m_hist.ptr(ex["seg"]), m_hist.ptr(ex["steps"]),
                                                  m_hist.ptr(ex["status"]), n, m_hist.ptr(h2), None))
        torch.cuda.synchronize()
        assert np.array_equal(h2.cpu().numpy(), ref)


@pytest.mark.parametrize("cfg,refill,minb,variant,mode", [
    ("hair512", 0, 4, 1, 0), ("hair512", 4, 3, 1, 0), ("hair512", 16, 2, 1, 0), ("hair512", 31, 4, 1, 0),
    # record table too large for shared memory: the per-triangle table is staged
    ("hair512", 4, 4, 2, 0), ("hair512", 6, 4, 2, 1), ("hair512", 0, 4, 3, 0),
    # variant 3: the per-triangle table where the record table also fits
    ("lines1024", 6, 4, 3, 0), ("lines1024", 6, 4, 3, 1), ("lines64", 31, 4, 3, 0),
    ("lines1024", 0, 4, 2, 0), ("lines1024", 4, 4, 2, 0), ("lines1024", 31, 4, 2, 0), ("lines1024", 4, 4, 1, 0),
    ("lines1024", 6, 3, 2, 0), ("lines1024", 6, 2, 2, 0), ("floorplan64", 6, 4, 2, 0),
    ("grass4096", 6, 4, 2, 0), ("grass4096", 6, 4, 3, 1),
    # variant 1: 256-thread CTAs from global memory, min_blocks 2 / 3 / 4
    ("grass4096", 6, 2, 1, 0), ("grass4096", 6, 3, 1, 0), ("floorplan64", 6, 3, 1, 0)])  # nothing fits: 896-thread CTAs, all from L1/L2
def test_tuning_knobs_do_not_change_results(cfg, refill, minb, variant, mode):
    from oracle import oracle as orc
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import DeviceMesh
    paths = fixture_paths(cfg, "mwt")
    m, om = DeviceMesh.from_files(*paths), orc.Mesh.from_files(*paths)
    rays = orc.raygen(mode, (0, 0, 1, 1), 2, 0, 50000)
    ref = om.trace(rays)
    _lib.check(_lib.lib.mwt_set_tuning(refill, minb, variant))
    try:
        got = m.trace(rays)
    finally:
        _lib.lib.mwt_set_tuning(6, 4, 2)  # the defaults
    for k in ("start", "seg", "steps"):
        assert np.array_equal(got[k], ref[k])


def test_edge_cases():
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    paths = fixture_paths("lines64", "mwt")
    m, om = DeviceMesh.from_files(*paths), orc.Mesh.from_files(*paths)
    # empty batch
    out = m.trace(np.zeros((0, 4)))
    assert len(out["seg"]) == 0
    # invalid start triangles -> error status, no crash
    rays = orc.raygen(0, (0, 0, 1, 1), 0, 0, 8)
    bad = m.trace(rays, np.array([-1, 10 ** 6, 0, 1, 2, 3, 4, 5], np.int32))
    assert (bad["status"][:2] & 1).all() and (bad["seg"][:2] == -1).all()
    # axis-aligned rays from every box side, rays through mesh vertices
    tri = om.tri
    v = np.stack([tri.vx, tri.vy], 1)
    dirs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
    rr = []
    for (dx, dy) in dirs:
        for p in v:
            rr.append([p[0], p[1], dx, dy])
    c = v.mean(0)
    for p in v:  # from the centre through each vertex
        d = p - c
        n = np.hypot(*d)
        if n > 0:
            rr.append([c[0], c[1], d[0] / n, d[1] / n])
    rr = np.array(rr)
    got, ref = m.trace(rr), om.trace(rr)
    assert np.array_equal(got["start"], ref["start"])
    assert np.array_equal(got["seg"], ref["seg"])
    ok = (ref["status"] & 1) == 0
    assert np.array_equal(got["steps"][ok], ref["steps"][ok])
    mask = ~np.uint32(256 | 2048)  # engine-only bits (own seed walk, boundary-table start)
    assert np.array_equal(got["status"].view(np.uint32) & mask, ref["status"] & mask)
    hit = ok & (ref["seg"] >= 0)
    assert np.array_equal(got["t"][hit], ref["t"][hit])
    # non-finite rays and origins far outside the mesh: terminate, no hang
    odd = np.array([[np.nan, 0.5, 1.0, 0.0], [0.5, 0.5, np.nan, 1.0], [np.inf, 0.5, -1.0, 0.0],
                    [0.5, 0.5, np.inf, 0.0], [1e6, -1e6, 0.6, 0.8], [-3.0, 0.5, 1.0, 0.0],
                    [0.5, 0.5, 0.0, 0.0]], np.float64)
    o2 = m.trace(odd)
    assert len(o2["seg"]) == len(odd)
    assert (o2["steps"] >= 0).all() and (o2["steps"] <= 4 * tri.v.shape[0] + 16).all()


def test_full_size_floorplan_properties():
    """2^26 box-entry rays (the FloorPlan config size): no error / overflow,
    histogram totals consistent with the per-ray outputs, four 2^24-ray shards
    (the weak-scaling split) sum to the whole, and 4,096 rays spread over the
    whole index range bit-exact vs the oracle."""
    import torch
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh, new_histogram, summarize_histogram
    paths = fixture_paths("floorplan64", "mwt")
    m = DeviceMesh.from_files(*paths)
    n = 1 << 26
    box = (0, 0, 1, 1)
    h = new_histogram()
    out = m.trace_generated_device(0, box, 0, 0, n, outputs=True, hist=h)
    torch.cuda.synchronize()
    s = summarize_histogram(h)
    assert s["rays"] == n and s["hits"] + s["misses"] == n
    assert s["status"]["error"] == 0 and s["status"]["overflow"] == 0
    assert s["steps_sum"] == int(out["steps"].to(torch.int64).sum())
    assert s["hits"] == int((out["seg"] >= 0).sum())
    shards = new_histogram()
    for k in range(4):
        m.trace_generated_device(0, box, 0, k << 24, 1 << 24, outputs=False, hist=shards)
    torch.cuda.synchronize()
    assert torch.equal(shards, h)
    idx = np.sort(np.random.default_rng(0).choice(n, 4096, replace=False))
    om = orc.Mesh.from_files(*paths)
    rays = np.concatenate([orc.raygen(0, box, 0, int(i), 1) for i in idx])
    ref = om.trace(rays)
    sel = torch.from_numpy(idx).cuda()
    assert np.array_equal(out["seg"][sel].cpu().numpy(), ref["seg"])
    assert np.array_equal(out["steps"][sel].cpu().numpy(), ref["steps"])
    t = out["t"][sel].cpu().numpy()
    hit = ref["seg"] >= 0
    assert np.array_equal(t[hit], ref["t"][hit])


def test_drop_in_api_on_model_objects():
    """The reference's call shapes (test_accel.py) through the drop-in API."""
    from oracle import oracle as orc
    from paper_2112_05570_b200 import accel
    from paper_2112_05570_b200.geometry import Point, Ray
    from paper_2112_05570_b200.model import Scene, load_triangulation
    paths = fixture_paths("lines64", "mwt")
    scene = Scene.load(paths[0])
    tri = load_triangulation(paths[1], scene)
    om = orc.Mesh.from_files(*paths)
    rays_np = orc.raygen(1, (0, 0, 1, 1), 4, 0, 200)
    ref = om.trace(rays_np)
    loc = accel.TriLocator(tri)
    for k, r in enumerate(rays_np):
        ray = Ray(Point(r[0], r[1]), Point(r[2], r[3]))
        start = loc.locate(ray.origin)
        assert start == ref["start"][k]
        hit, stats = accel.traverse_triangulation(tri, ray, start)
        assert stats.tri_steps == ref["steps"][k]
        assert (hit is None) == (ref["seg"][k] < 0)
        if hit is not None:
            assert hit.seg == ref["seg"][k] and hit.t == ref["t"][k]
            assert isinstance(hit.point, Point)
        bf = accel.brute_force_closest(scene, ray)
        assert (bf is None) == (hit is None) and (bf is None or bf.seg == hit.seg)
    assert accel.locate_triangle(tri, Point(0.5, 0.5), "brute") == loc.locate(Point(0.5, 0.5))
    with pytest.raises(ValueError):
        accel.locate_triangle(tri, Point(0.5, 0.5), "nope")
    batch = accel.trace_batch(tri, rays_np)
    assert np.array_equal(batch["seg"], ref["seg"])


def test_chained_secondary_rays():
    """mwt_trace_chain_dev: the final triangle of every
    walk equals the oracle's, and secondary rays started there (no locate)
    trace identically to the oracle given the same start triangles."""
    import torch
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    for cfg in ("lines1024", "hair512"):
        paths = fixture_paths(cfg, "mwt")
        m, om = DeviceMesh.from_files(*paths), orc.Mesh.from_files(*paths)
        rays = orc.raygen(0, box_of(cfg), 7, 0, 1 << 16)
        ref = om.trace(rays)
        got = m.trace_chain_device(torch.from_numpy(rays).cuda())
        got = {k: v.cpu().numpy() for k, v in got.items()}
        for k in ("end", "seg", "steps"):
            assert np.array_equal(got[k], ref[k]), (cfg, k)
        # secondary rays from the hit points, mirrored about the hit segment
        hit = ref["seg"] >= 0
        o = rays[hit, :2] + ref["t"][hit, None] * rays[hit, 2:]
        sc, sid = om.scene, ref["seg"][hit]
        e = np.stack([sc.bx[sid] - sc.ax[sid], sc.by[sid] - sc.ay[sid]], 1)
        e /= np.hypot(e[:, 0], e[:, 1])[:, None]
        d = rays[hit, 2:]
        d = 2.0 * (d * e).sum(1)[:, None] * e - d  # mirror about the segment
        d /= np.hypot(d[:, 0], d[:, 1])[:, None]
        r2 = np.ascontiguousarray(np.concatenate([o, d], 1))
        start2 = np.ascontiguousarray(ref["end"][hit])
        ref2 = om.trace(r2, start2)
        got2 = m.trace_chain_device(torch.from_numpy(r2).cuda(), torch.from_numpy(start2).cuda())
        got2 = {k: v.cpu().numpy() for k, v in got2.items()}
        for k in ("end", "seg", "steps"):
            assert np.array_equal(got2[k], ref2[k]), (cfg, "secondary", k)
        h2 = ref2["seg"] >= 0
        assert np.array_equal(got2["t"][h2], ref2["t"][h2])


def _dkey(x):
    b = struct.unpack("<q", struct.pack("<d", x))[0]
    return b if b >= 0 else -(1 << 63) - b


def _dval(k):
    b = k if k >= 0 else -(1 << 63) - k
    return struct.unpack("<d", struct.pack("<q", b))[0]


def _sa2(a, b, p):  # geometry.py:81-83, CPython floats (binary64, no FMA)
    return (b[0] - a[0]) * (p[1] - a[1]) - (b[1] - a[1]) * (p[0] - a[0])


def _switch(f, lo, hi):
    """Key of the first double in [lo, hi] where the monotone predicate f flips."""
    a, b = lo, hi
    fa = f(a)
    while a + 1 < b:
        m = (a + b) // 2
        if f(m) == fa:
            a = m
        else:
            b = m
    return b


@pytest.mark.parametrize("cfg", ["lines64", "lines1024"])
def test_box_entry_start_at_interval_bounds(cfg):
    """Origins on the bottom side at the exact switch points of the start test
    (accel.py:219-238: _contains and the flood bound of the edge's other two
    values), +-1 ulp: the packer's precomputed intervals must agree with the
    reference rule on both sides of every bound (start, steps, hit bit-exact)."""
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    paths = fixture_paths(cfg, "mwt")
    m, om = DeviceMesh.from_files(*paths), orc.Mesh.from_files(*paths)
    tri = om.tri
    xy = np.stack([tri.vx, tri.vy], 1)
    us = []
    for t in range(len(tri.v)):
        for i in range(3):
            P, Q, A = (xy[tri.v[t][(i + 1) % 3]], xy[tri.v[t][(i + 2) % 3]], xy[tri.v[t][i]])
            if not (P[1] == 0.0 and Q[1] == 0.0 and A[1] > 0.0):
                continue
            lo, hi = _dkey(float(min(P[0], Q[0]))) + 1, _dkey(float(max(P[0], Q[0]))) - 1
            for g in (lambda k: _sa2(Q, A, (_dval(k), 0.0)) > 1e-12,
                      lambda k: _sa2(A, P, (_dval(k), 0.0)) > 1e-12):
                if g(lo) == g(hi):
                    continue
                k = _switch(g, lo, hi)
                us += [_dval(k + d) for d in (-2, -1, 0, 1)]
    assert len(us) >= 16
    rng = np.random.default_rng(5)
    th = rng.uniform(0.05, np.pi - 0.05, len(us))
    rays = np.stack([np.array(us), np.zeros(len(us)), np.cos(th), np.sin(th)], 1)
    got, ref = m.trace(rays), om.trace(rays)
    for k in ("start", "seg", "steps"):
        assert np.array_equal(got[k], ref[k]), k
    hit = ref["seg"] >= 0
    assert np.array_equal(got["t"][hit], ref["t"][hit])
    fast = (got["status"].view(np.uint32) & np.uint32(2048)) != 0
    assert fast.any() and (~fast).any()  # both sides of the bounds were exercised


@pytest.mark.parametrize("ndev", [1, 2, 3])
def test_single_process_sharded_entry_points(ndev):
    """mwt_trace_generated_sharded / mwt_trace_host_sharded (one host thread
    and stream per device handle; here ndev handles of the same mesh, all on
    cuda:0 of this one-GPU box): the summed histogram and the per-ray outputs
    equal one unsharded call."""
    import torch
    from paper_2112_05570_b200.engine import (DeviceMesh, new_histogram, trace_generated_sharded,
                                              trace_sharded)
    from paper_2112_05570_b200.sharding import histogram_host
    paths = fixture_paths("lines1024", "mwt")
    meshes = [DeviceMesh.from_files(*paths) for _ in range(ndev)]
    n = 300001
    h1 = new_histogram()
    meshes[0].trace_generated_device(0, (0, 0, 1, 1), 9, 123, n, False, h1)
    torch.cuda.synchronize()
    hs = trace_generated_sharded(meshes, 0, (0, 0, 1, 1), 9, 123, n)
    assert np.array_equal(hs, h1.cpu().numpy())
    rays = meshes[0].raygen(1, (0, 0, 1, 1), 9, 5, 100003)
    a, b = meshes[0].trace(rays), trace_sharded(meshes, rays)
    for k in ("start", "seg", "steps", "status"):
        assert np.array_equal(a[k], b[k]), k
    hit = a["seg"] >= 0
    assert np.array_equal(a["t"][hit], b["t"][hit]) and np.array_equal(a["u"][hit], b["u"][hit])
    assert np.array_equal(histogram_host(b["seg"], b["steps"], b["status"])[:1027],
                          histogram_host(a["seg"], a["steps"], a["status"])[:1027])


def test_binary_mesh_traces_like_the_text_mesh(tmp_path):
    """mwt-mesh v1 (formats.save_mesh_binary) loaded by DeviceMesh.from_binary
    walks exactly like the text fixture and the oracle."""
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    from paper_2112_05570_b200.formats import load_scene, load_tri, save_mesh_binary
    paths = fixture_paths("hair512", "mwt")
    save_mesh_binary(str(tmp_path / "m"), load_scene(paths[0]), load_tri(paths[1]))
    mb = DeviceMesh.from_binary(str(tmp_path / "m"))
    om = orc.Mesh.from_files(*paths)
    for mode in (0, 1):
        rays = orc.raygen(mode, (0, 0, 1, 1), 5, 0, 1 << 16)
        got, ref = mb.trace(rays), om.trace(rays)
        for k in ("start", "seg", "steps"):
            assert np.array_equal(got[k], ref[k]), k
        hit = ref["seg"] >= 0
        assert np.array_equal(got["t"][hit], ref["t"][hit])
