"""Parity of the CUDA engine against the C oracle (itself pinned to the
reference by tests/test_oracle_golden.py) on the five BASELINE configs.

Bar (BASELINE.json north_star): hit segment id, start triangle and step count
bit-exact; hit distance t within 1e-12 relative (the engine is in fact
bit-exact: no FMA contraction, reference operation order)."""
import numpy as np
import pytest

from conftest import CONFIGS, box_of, fixture_paths

pytestmark = pytest.mark.gpu

T_RTOL = 1e-12
LOC_BRUTE = np.uint32(256 | 2048)  # engine-only bits: own seed walk, boundary-table start


def _mesh_pair(cfg, which):
    paths = fixture_paths(cfg, which)
    if paths is None:
        pytest.skip(f"{cfg}/{which} fixture not generated")
    from paper_2112_05570_b200.engine import DeviceMesh
    from oracle import oracle as orc
    return DeviceMesh.from_files(*paths), orc.Mesh.from_files(*paths)


def _compare(got, ref, keys=("start", "seg", "steps", "status"), t_bits=False):
    ok_err = (ref["status"] & 1) == 0
    for k in keys:
        a, b = np.asarray(got[k]), np.asarray(ref[k])
        if k == "steps":
            a, b = a[ok_err], b[ok_err]
        if k == "status":
            # LOC_BRUTE marks the engine's own seed walk failing (its walk is
            # not the reference's); every other bit must agree
            a, b = a.view(np.uint32) & ~LOC_BRUTE, b.view(np.uint32) & ~LOC_BRUTE
        bad = np.nonzero(a != b)[0]
        assert len(bad) == 0, f"{k}: {len(bad)} mismatches, first {bad[:5]} got {a[bad[:5]]} ref {b[bad[:5]]}"
    hit = ref["seg"] >= 0
    t_got, t_ref = got["t"][hit], ref["t"][hit]
    if t_bits:  # (hit tests that overflow: inf / nan on both sides, bit for bit)
        assert np.array_equal(t_got.view(np.uint64), t_ref.view(np.uint64))
        return
    rel = np.abs(t_got - t_ref) / np.maximum(1.0, np.abs(t_ref))
    assert rel.max(initial=0.0) <= T_RTOL
    assert np.all(np.isnan(got["t"][~hit]))


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("which", ["cdt", "mwt"])
@pytest.mark.parametrize("mode", [0, 1])
def test_trace_with_device_locate(cfg, which, mode):
    from oracle import oracle as orc
    mesh, om = _mesh_pair(cfg, which)
    n = 1 << 16
    box = box_of(cfg)
    rays_dev = mesh.raygen_device(mode, box, 0, 12345, n)
    got = {k: v.cpu().numpy() for k, v in mesh.trace_device(rays_dev).items()}
    rays = orc.raygen(mode, box, 0, 12345, n)
    assert np.array_equal(rays_dev.cpu().numpy().view(np.uint64), rays.view(np.uint64))
    ref = om.trace(rays)
    _compare(got, ref)


@pytest.mark.parametrize("cfg", CONFIGS)
def test_trace_host_entry_point(cfg):
    from oracle import oracle as orc
    mesh, om = _mesh_pair(cfg, "mwt")
    rays = orc.raygen(0, box_of(cfg), 7, 0, 20000)
    ref = om.trace(rays)
    got = mesh.trace(rays)
    _compare(got, ref)
    got2 = mesh.trace(rays, ref["start"])  # explicit start triangles
    _compare(got2, ref)


def test_unbounded_ray_takes_the_full_rule():
    """The tight walk loop compares side_of's two products instead of
    subtracting them (exact while |o|, |d| and the mesh stay within 2^500);
    loaded rays outside that bound walk with the full rule.  Directions
    scaled by 2^600 (exact) must give the oracle's results -- and the
    unscaled rays' walk: every side value scales by the same power of two."""
    from oracle import oracle as orc
    mesh, om = _mesh_pair("floorplan64", "mwt")
    rays = orc.raygen(0, box_of("floorplan64"), 3, 0, 4096)
    big = rays.copy()
    big[:, 2:] *= 2.0 ** 600
    ref = om.trace(big)
    got = mesh.trace(big)
    _compare(got, ref)
    base = mesh.trace(rays)
    for k in ("start", "seg", "steps"):
        assert np.array_equal(got[k], base[k]), k


def test_mesh_beyond_the_bound_walks_with_the_full_rule():
    """A mesh whose coordinates exceed 2^500 (MeshDev.coord_small = 0) never
    takes the compare-form tight loop: Lines-64 scaled by 2^600 (exact), its
    box-entry rays' origins scaled alike, engine = oracle on every ray."""
    import dataclasses
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    from paper_2112_05570_b200.formats import load_scene, load_tri
    paths = fixture_paths("lines64", "mwt")
    if paths is None:
        pytest.skip("lines64/mwt fixture not generated")
    K = 2.0 ** 600
    sc, tr = load_scene(paths[0]), load_tri(paths[1])
    mesh = DeviceMesh(dataclasses.replace(sc, xy=sc.xy * K), dataclasses.replace(tr, vxy=tr.vxy * K))
    rs, rt = orc.load_scene(paths[0]), orc.load_tri(paths[1])
    om = orc.Mesh(orc.RawScene(rs.ax * K, rs.ay * K, rs.bx * K, rs.by * K, rs.kind, rs.name),
                  orc.RawTri(rt.vx * K, rt.vy * K, rt.v, rt.nbr, rt.flag))
    rays = orc.raygen(0, (0.0, 0.0, 1.0, 1.0), 5, 0, 4096)
    rays[:, :2] *= K
    # (the hit test's products exceed the double range: t is inf or nan, as in
    # the reference's Python floats -- compared bit for bit)
    _compare(mesh.trace(rays), om.trace(rays), t_bits=True)
