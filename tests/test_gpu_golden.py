"""The CUDA engine against the golden vectors recorded from the reference
itself (tests/golden/make_golden.py): hand-built degenerate scenes, the
reference tests' scenes, all five configs, and the BVH / kd-tree counters."""
import os

import numpy as np
import pytest

from conftest import CONFIGS, GOLDEN, fixture_paths

pytestmark = pytest.mark.gpu


def _golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"golden file {name} not generated")
    return np.load(p)


def _known_cases():
    p = os.path.join(GOLDEN, "known.npz")
    return [str(c) for c in np.load(p)["cases"]] if os.path.exists(p) else []


def _mesh(g, name):
    from paper_2112_05570_b200.engine import DeviceMesh
    from paper_2112_05570_b200.formats import SceneArrays, TriArrays
    sc = SceneArrays(np.ascontiguousarray(g[f"{name}__seg_xy"]), np.ascontiguousarray(g[f"{name}__seg_kind"]))
    tri = TriArrays(g[f"{name}__vxy"], g[f"{name}__v"], g[f"{name}__nbr"], g[f"{name}__flag"])
    return DeviceMesh(sc, tri)


def _check(out, g, prefix):
    err = g[prefix + "error"].astype(bool)
    assert np.array_equal((out["status"].view(np.uint32) & 1).astype(bool), err)
    ok = ~err
    for k in ("start", "seg", "steps"):
        bad = np.nonzero(out[k][ok] != g[prefix + k][ok])[0]
        assert len(bad) == 0, f"{k}: {len(bad)} mismatches, first {bad[:5]}"
    hit = ok & (g[prefix + "seg"] >= 0)
    # north_star tolerance: t within 1e-12 relative (the engine is bit-exact)
    rel = np.abs(out["t"][hit] - g[prefix + "t"][hit]) / np.maximum(1.0, np.abs(g[prefix + "t"][hit]))
    assert rel.max(initial=0.0) <= 1e-12
    assert np.array_equal(out["t"][hit], g[prefix + "t"][hit])


@pytest.mark.parametrize("name", _known_cases())
def test_known_cases_on_device(name):
    g = _golden("known.npz")
    m = _mesh(g, name)
    rays = g[f"{name}__rays"]
    _check(m.trace(rays), g, f"{name}__w_")
    tid, _ = m.locate(g[f"{name}__loc_pts"])
    assert np.array_equal(tid, g[f"{name}__loc_anchor"])
    bf = m.brute_force(rays)
    assert np.array_equal(bf["seg"], g[f"{name}__bf_seg"])


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("which", ["cdt", "mwt"])
def test_configs_on_device(cfg, which):
    from paper_2112_05570_b200.engine import DeviceMesh
    g = _golden(f"config_{cfg}.npz")
    paths = fixture_paths(cfg, which)
    if paths is None or f"{which}0_seg" not in g.files:
        pytest.skip("fixture/golden not generated")
    m = DeviceMesh.from_files(*paths)
    box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
    for mode in (0, 1):
        if f"{which}{mode}_seg" not in g.files:
            continue
        rays = g[f"rays{mode}"]
        dev_rays = m.raygen(mode, box, 0, 0, len(rays))
        assert np.array_equal(dev_rays.view(np.uint64), rays.view(np.uint64)), "device raygen != golden rays"
        _check(m.trace(rays), g, f"{which}{mode}_")
        n = len(g[f"bf{mode}_seg"])
        bf = m.brute_force(rays[:n])
        assert np.array_equal(bf["seg"], g[f"bf{mode}_seg"])


@pytest.mark.parametrize("cfg", CONFIGS[1:])
def test_structures_on_device(cfg):
    from paper_2112_05570_b200.engine import DeviceBvh, DeviceKd, DeviceMesh
    from paper_2112_05570_b200.formats import load_scene
    g = _golden(f"struct_{cfg}.npz")
    paths = fixture_paths(cfg, "cdt")
    d = os.path.dirname(paths[0])
    m = DeviceMesh(load_scene(paths[0]), None)
    for key in [k for k in g.files if k.startswith("bvh") and k.endswith("_seg")]:
        tag = key[3:-4]
        mode, ct = tag.split("_ct")
        rays = g[f"rays{mode}"]
        o = DeviceBvh.from_file(m, os.path.join(d, f"bvh_ct{ct}.npz")).trace(rays)
        assert np.array_equal(o["seg"], g[f"bvh{tag}_seg"])
        h = o["seg"] >= 0
        assert np.array_equal(o["t"][h], g[f"bvh{tag}_t"][h])
        assert np.array_equal(o["node_tests"], g[f"bvh{tag}_nodes"])
        assert np.array_equal(o["prim_tests"], g[f"bvh{tag}_prims"])
        o = DeviceKd.from_file(m, os.path.join(d, f"kd_ct{ct}.npz")).trace(rays)
        ok = g[f"kd{tag}_nodes"] >= 0
        assert np.array_equal(o["seg"][ok], g[f"kd{tag}_seg"][ok])
        assert np.array_equal(o["nodes"][ok], g[f"kd{tag}_nodes"][ok])
        assert np.array_equal(o["ropes"][ok], g[f"kd{tag}_ropes"][ok])
        assert np.array_equal(o["prims"][ok], g[f"kd{tag}_prims"][ok])


def test_degenerate_rays_on_device():
    """The rays where the reference walk and brute force disagree
    (tests/golden/degenerate.npz): the device walk returns the reference walk's
    answer -- through the host API, from the explicit rays, and fused with the
    on-device ray generator at the ray's own index -- and the device brute
    force the reference brute force's."""
    import torch
    from paper_2112_05570_b200.engine import DeviceMesh, new_histogram
    g = _golden("degenerate.npz")
    k = 0
    while f"{k}_cfg" in g:
        cfg, index = str(g[f"{k}_cfg"]), int(g[f"{k}_index"])
        box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
        ray = g[f"{k}_ray"]
        for w in ("cdt", "mwt"):
            m = DeviceMesh.from_files(*fixture_paths(cfg, w))
            assert np.array_equal(m.raygen(0, box, 0, index, 1).view(np.uint64), ray.view(np.uint64))
            o = m.trace(ray)
            start, seg, steps = (int(x) for x in g[f"{k}_{w}"])
            assert (int(o["start"][0]), int(o["seg"][0]), int(o["steps"][0])) == (start, seg, steps)
            assert o["t"][0] == float(g[f"{k}_{w}_t"])
            gen = m.trace_generated_device(0, box, 0, index, 1, True, new_histogram())
            torch.cuda.synchronize()
            assert (int(gen["seg"][0]), int(gen["steps"][0])) == (seg, steps)
            bf = m.brute_force(ray)
            assert int(bf["seg"][0]) == int(g[f"{k}_brute"][0]) and bf["t"][0] == g[f"{k}_brute"][1]
        k += 1
    assert k > 0


def _branch_cases():
    p = os.path.join(GOLDEN, "branches.npz")
    return [str(c) for c in np.load(p)["cases"]] if os.path.exists(p) else []


LOCATED = ("parallel_exit", "outside_")  # starts located by the reference's TriLocator


@pytest.mark.parametrize("name", _branch_cases())
def test_branch_fixtures_on_device(name):
    """The walk's fallback exit, both TraversalError kinds, the parallel branch
    at a constrained exit and outside-the-mesh locates (tests/golden/branches.npz,
    recorded from the reference): the device reproduces the reference's
    outcomes and sets exactly the oracle's status bits."""
    from oracle import oracle as orc
    from paper_2112_05570_b200 import _lib
    g = _golden("branches.npz")
    m = _mesh(g, name)
    rays = g[f"{name}__rays"]
    given = None if name.startswith(LOCATED) else g[f"{name}__w_start"]
    out = m.trace(rays, given)
    _check(out, g, f"{name}__w_")
    # status bits: the oracle's, bit for bit (minus the engine's own seed-search notes)
    sc = orc.RawScene(*(np.ascontiguousarray(g[f"{name}__seg_xy"][:, k]) for k in range(4)),
                      np.ascontiguousarray(g[f"{name}__seg_kind"]))
    vxy = g[f"{name}__vxy"]
    om = orc.Mesh(sc, orc.RawTri(np.ascontiguousarray(vxy[:, 0]), np.ascontiguousarray(vxy[:, 1]),
                                 np.ascontiguousarray(g[f"{name}__v"]), np.ascontiguousarray(g[f"{name}__nbr"]),
                                 np.ascontiguousarray(g[f"{name}__flag"])))
    ref = om.trace(rays, given)
    mask = np.uint32(~_lib.ST_ENGINE_ONLY & 0xFFFFFFFF)
    assert np.array_equal(out["status"].view(np.uint32) & mask, ref["status"] & mask)
    if f"{name}__loc_pts" in g.files:
        pts = g[f"{name}__loc_pts"]
        tid, st = m.locate(pts)
        assert np.array_equal(tid, g[f"{name}__loc_anchor"])
        assert (st & _lib.ST_LOC_OUTSIDE).all()
        tb, _ = m.locate(pts, method="brute")
        assert np.array_equal(tb, g[f"{name}__loc_brute"])


def test_branch_fixtures_through_the_drop_in():
    """The drop-in raises TraversalError on exactly the rays where the reference
    raised it (revisit and no-exit kinds), and returns its hits elsewhere."""
    from paper_2112_05570_b200 import accel
    from paper_2112_05570_b200.formats import SceneArrays, TriArrays
    from paper_2112_05570_b200.geometry import Point, Ray
    from paper_2112_05570_b200.model import Scene, Triangulation
    g = _golden("branches.npz")
    raised = {1: 0, 2: 0}
    for name in _branch_cases():
        if not name.startswith("fan"):
            continue
        scene = Scene.from_arrays(SceneArrays(g[f"{name}__seg_xy"], g[f"{name}__seg_kind"]))
        tri = Triangulation.from_arrays(scene, TriArrays(g[f"{name}__vxy"], g[f"{name}__v"], g[f"{name}__nbr"],
                                                          g[f"{name}__flag"]))
        rays, err = g[f"{name}__rays"], g[f"{name}__w_error"]
        sel = np.concatenate([np.nonzero(err)[0], np.nonzero(err == 0)[0][:40]])
        for i in sel:
            r = rays[i]
            ray = Ray(Point(r[0], r[1]), Point(r[2], r[3]))
            start = int(g[f"{name}__w_start"][i])
            if err[i]:
                with pytest.raises(accel.TraversalError):
                    accel.traverse_triangulation(tri, ray, start)
                raised[int(err[i])] += 1
            else:
                hit, stats = accel.traverse_triangulation(tri, ray, start)
                assert stats.tri_steps == g[f"{name}__w_steps"][i]
                assert (hit is None) == (g[f"{name}__w_seg"][i] < 0)
                if hit is not None:
                    assert hit.seg == g[f"{name}__w_seg"][i] and hit.t == g[f"{name}__w_t"][i]
    assert raised[1] > 0 and raised[2] > 0


def test_drop_in_repacks_an_edited_triangulation():
    """the reference edits triangulations in place; the drop-in's
    cached device copy must follow (content fingerprint), not walk a stale mesh."""
    from oracle import oracle as orc
    from paper_2112_05570_b200 import accel
    from paper_2112_05570_b200.accel import _TriMap
    from paper_2112_05570_b200.model import Scene, load_triangulation
    paths = fixture_paths("lines64", "mwt")
    scene = Scene.load(paths[0])
    tri = load_triangulation(paths[1], scene)
    rays = orc.raygen(1, (0, 0, 1, 1), 3, 0, 4000)
    p0 = accel.pack(tri)
    before = accel.trace_batch(tri, rays)
    # an in-place edit: shear every interior vertex (same topology, new geometry)
    for v in tri.verts:
        if 0.0 < v.x < 1.0 and 0.0 < v.y < 1.0:
            v.x, v.y = v.x, v.y + 2e-3 * (v.x - 0.5)
    p1 = accel.pack(tri)
    assert p1 is not p0
    after = accel.trace_batch(tri, rays)
    sa = scene.to_arrays()
    arr = _TriMap(tri).arrays
    om = orc.Mesh(orc.RawScene(*(np.ascontiguousarray(sa.xy[:, k]) for k in range(4)),
                               np.ascontiguousarray(sa.kind)),
                  orc.RawTri(np.ascontiguousarray(arr.vxy[:, 0]), np.ascontiguousarray(arr.vxy[:, 1]),
                             np.ascontiguousarray(arr.v), np.ascontiguousarray(arr.nbr),
                             np.ascontiguousarray(arr.flag)))
    ref = om.trace(rays)
    for k in ("start", "seg", "steps"):
        assert np.array_equal(after[k], ref[k]), k
    assert not np.array_equal(before["steps"], after["steps"])  # the edit is visible
    assert accel.pack(tri) is p1  # unchanged content: the cache holds


def test_kd_from_given_start_leaves():
    """kd_intersect(kd, ray, start_leaf=...) (accel.py:761-771) from random
    leaves: hit and all three counters equal the reference's (kdstart.npz);
    a start index that is not a leaf is an error, and the drop-in rejects it."""
    from paper_2112_05570_b200 import _lib, accel
    from paper_2112_05570_b200.engine import DeviceKd, DeviceMesh
    g = _golden("kdstart.npz")
    mesh = DeviceMesh.from_files(*fixture_paths("lines1024", "mwt"))
    kd = DeviceKd(mesh, {k: g[k] for k in g.files if not k.startswith("out_")})
    o = kd.trace(g["rays"], g["start"])
    assert not (o["status"] & _lib.ST_ERROR).any() and not g["out_error"].any()
    for k in ("seg", "nodes", "ropes", "prims"):
        assert np.array_equal(o[k], g["out_" + k]), k
    hit = g["out_seg"] >= 0
    assert np.array_equal(o["t"][hit], g["out_t"][hit])
    internal = int(np.nonzero(g["axis"] >= 0)[0][0])
    bad = kd.trace(g["rays"][:2], np.array([internal, -1], np.int32))
    assert (bad["status"] & _lib.ST_ERROR).all()
