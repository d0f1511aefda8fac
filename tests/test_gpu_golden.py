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
    box = (0.0, 0.0, 1.0, 0.5) if cfg == "grass4096" else (0.0, 0.0, 1.0, 1.0)
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
        box = (0.0, 0.0, 1.0, 0.5) if cfg == "grass4096" else (0.0, 0.0, 1.0, 1.0)
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
