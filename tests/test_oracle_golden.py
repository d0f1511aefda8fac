"""Pin the C oracle (oracle/mwt_oracle.c) to the reference: every function is
checked against golden vectors recorded by running the unmodified reference
(tests/golden/make_golden.py).  CPU only."""
import os

import numpy as np
import pytest

from conftest import CONFIGS, GOLDEN, fixture_paths

orc = pytest.importorskip("oracle.oracle")
from oracle import raygen as rg  # noqa: E402


def _golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"golden file {name} not generated")
    return np.load(p)


def test_hypot_is_cpython_hypot():
    g = _golden("hypot.npz")
    got = np.array([orc.hypot(a, b) for a, b in zip(g["x"].tolist(), g["y"].tolist())])
    assert np.array_equal(got.view(np.uint64), g["h"].view(np.uint64))


@pytest.mark.parametrize("mode", [0, 1, rg.coherent(0), rg.coherent(1), rg.coherent(0, 0, 16),
                                  rg.coherent(1, 40, 1)])
def test_raygen_twins_agree(mode):
    box = (0.0, 0.0, 1.0, 0.5)
    a = rg.raygen(mode, box, 11, 1000, 50000)
    b = orc.raygen(mode, box, 11, 1000, 50000)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    # reference Ray would not renormalise (geometry.py:73)
    n = np.hypot(a[:, 2], a[:, 3])
    assert np.abs(n - 1.0).max() <= 1e-12
    if mode & 0xFF == 0:  # origin exactly on the entered side of the box
        on = (a[:, 0] == 0.0) | (a[:, 0] == 1.0) | (a[:, 1] == 0.0) | (a[:, 1] == 0.5)
        assert on.all()


def test_raygen_mode_words():
    """include/mwt.h MWT_RAYS_COHERENT: malformed words are rejected by every twin;
    cell_bits 0 is the iid generator whatever the group size."""
    for bad in (2, 0xFF, rg.coherent(0, 41, 1), rg.coherent(0, 7, 17), 1 << 24, -1):
        with pytest.raises(ValueError):
            rg.raygen(bad, (0, 0, 1, 1), 0, 0, 4)
        with pytest.raises(ValueError):
            orc.raygen(bad, (0, 0, 1, 1), 0, 0, 4)
    a = rg.raygen(rg.coherent(0, 7, 0), (0, 0, 1, 1), 5, 3, 1000)
    assert np.array_equal(a.view(np.uint64), rg.raygen(0, (0, 0, 1, 1), 5, 3, 1000).view(np.uint64))


@pytest.mark.parametrize("base", [0, 1])
def test_coherent_rays_keep_the_iid_distribution(base):
    """Each coherent ray is an exact draw of the base distribution: the rays at
    one position j of every group (independent groups) pass the same isotropy,
    uniform-offset / uniform-origin tests as the iid generator; and a group's
    rays share a cell (nearly the same line)."""
    from scipy.stats import chisquare, kstest
    box = (0.0, 0.0, 1.0, 0.5)
    mode = rg.coherent(base)
    n = 512 * 5000
    r = rg.raygen(mode, box, 21, 0, n).reshape(-1, 512, 4)
    for j in (0, 77, 300):
        s = r[:, j]
        ang = np.arctan2(s[:, 3], s[:, 2])
        counts, _ = np.histogram(ang, bins=36, range=(-np.pi, np.pi))
        assert chisquare(counts).pvalue > 1e-4
        if base == 1:
            assert kstest(s[:, 0], "uniform").pvalue > 1e-4
            assert kstest(s[:, 1] / 0.5, "uniform").pvalue > 1e-4
        else:
            nx, ny = -s[:, 3], s[:, 2]
            cx = np.array([0.0, 1.0, 1.0, 0.0])
            cy = np.array([0.0, 0.0, 0.5, 0.5])
            proj = nx[:, None] * cx[None, :] + ny[:, None] * cy[None, :]
            a, b = proj.min(1), proj.max(1)
            off = (nx * s[:, 0] + ny * s[:, 1] - a) / (b - a)
            assert kstest(off, "uniform").pvalue > 1e-4
    # coherence: most groups span a small angle
    ang = np.arctan2(r[..., 3], r[..., 2])
    spread = np.abs(np.angle(np.exp(1j * (ang - ang[:, :1])))).max(1)
    assert np.median(spread) < 0.02


def test_raygen_isotropic():
    """chi-square isotropy like test_harness.py:99-111."""
    from scipy.stats import chisquare
    r = rg.raygen(0, (0, 0, 1, 1), 3, 0, 200000)
    ang = np.arctan2(r[:, 3], r[:, 2])
    counts, _ = np.histogram(ang, bins=36, range=(-np.pi, np.pi))
    assert chisquare(counts).pvalue > 1e-4


def test_ray_segment_intersect_golden():
    g = _golden("known.npz")
    t = np.empty(len(g["rsi_rays"]))
    u = np.empty(len(g["rsi_rays"]))
    for k, (r, s) in enumerate(zip(g["rsi_rays"], g["rsi_segs"])):
        tt, uu = np.zeros(1), np.zeros(1)
        import ctypes
        ok = orc.lib().orc_ray_segment_intersect(
            np.ascontiguousarray(r).ctypes.data_as(ctypes.c_void_p),
            np.ascontiguousarray(s).ctypes.data_as(ctypes.c_void_p),
            tt.ctypes.data_as(ctypes.c_void_p), uu.ctypes.data_as(ctypes.c_void_p))
        t[k], u[k] = (tt[0], uu[0]) if ok else (np.nan, np.nan)
    ref = g["rsi_tu"]
    assert np.array_equal(np.isnan(t), np.isnan(ref[:, 0]))
    m = ~np.isnan(t)
    assert np.array_equal(t[m], ref[m, 0]) and np.array_equal(u[m], ref[m, 1])


def _known_cases():
    p = os.path.join(GOLDEN, "known.npz")
    if not os.path.exists(p):
        return []
    return [str(c) for c in np.load(p)["cases"]]


def known_mesh(g, name):
    sc = orc.RawScene(*(np.ascontiguousarray(g[f"{name}__seg_xy"][:, k]) for k in range(4)),
                      np.ascontiguousarray(g[f"{name}__seg_kind"]))
    vxy = g[f"{name}__vxy"]
    tri = orc.RawTri(np.ascontiguousarray(vxy[:, 0]), np.ascontiguousarray(vxy[:, 1]),
                     np.ascontiguousarray(g[f"{name}__v"]), np.ascontiguousarray(g[f"{name}__nbr"]),
                     np.ascontiguousarray(g[f"{name}__flag"]))
    return orc.Mesh(sc, tri)


def check_walk(out, ref, prefix=""):
    err = ref[prefix + "error"].astype(bool)
    assert np.array_equal((out["status"] & 1).astype(bool), err)
    ok = ~err
    for k in ("start", "seg", "steps"):
        a, b = out[k][ok], ref[prefix + k][ok]
        bad = np.nonzero(a != b)[0]
        assert len(bad) == 0, f"{k}: {len(bad)} mismatches e.g. {bad[:5]}"
    hit = ok & (ref[prefix + "seg"] >= 0)
    assert np.array_equal(out["t"][hit], ref[prefix + "t"][hit])


@pytest.mark.parametrize("name", _known_cases())
def test_known_cases(name):
    g = _golden("known.npz")
    m = known_mesh(g, name)
    rays = g[f"{name}__rays"]
    out = m.trace(rays)
    ref = {k[len(name) + 4:]: g[k] for k in g.files if k.startswith(f"{name}__w_")}
    check_walk(out, ref)
    tid, _ = m.locate(g[f"{name}__loc_pts"])
    assert np.array_equal(tid, g[f"{name}__loc_anchor"])
    assert np.array_equal(tid, g[f"{name}__loc_brute"])
    bf = m.brute_force(rays)
    assert np.array_equal(bf["seg"], g[f"{name}__bf_seg"])
    h = bf["seg"] >= 0
    assert np.array_equal(bf["t"][h], g[f"{name}__bf_t"][h])


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("which", ["cdt", "mwt"])
def test_config_walk_golden(cfg, which):
    g = _golden(f"config_{cfg}.npz")
    paths = fixture_paths(cfg, which)
    if paths is None or f"{which}0_seg" not in g.files:
        pytest.skip("fixture/golden not generated")
    m = orc.Mesh.from_files(*paths)
    for mode in (0, 1):
        if f"rays{mode}" not in g.files or f"{which}{mode}_seg" not in g.files:
            continue
        rays = g[f"rays{mode}"]
        box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
        assert np.array_equal(orc.raygen(mode, box, 0, 0, len(rays)).view(np.uint64), rays.view(np.uint64))
        check_walk(m.trace(rays), g, f"{which}{mode}_")
        n = len(g[f"bf{mode}_seg"])
        bf = m.brute_force(rays[:n])
        assert np.array_equal(bf["seg"], g[f"bf{mode}_seg"])


@pytest.mark.parametrize("cfg", CONFIGS[1:])
def test_structures_golden(cfg):
    g = _golden(f"struct_{cfg}.npz")
    paths = fixture_paths(cfg, "cdt")
    m = orc.Mesh.from_files(*paths)
    d = os.path.dirname(paths[0])
    for key in [k for k in g.files if k.startswith("bvh") and k.endswith("_seg")]:
        tag = key[3:-4]               # "<mode>_ct<c>"
        mode, ct = tag.split("_ct")
        rays = g[f"rays{mode}"]
        bvh = orc.Bvh(m, orc.load_npz(os.path.join(d, f"bvh_ct{ct}.npz")))
        o = bvh.trace(rays)
        assert np.array_equal(o["seg"], g[f"bvh{tag}_seg"])
        h = o["seg"] >= 0
        assert np.array_equal(o["t"][h], g[f"bvh{tag}_t"][h])
        assert np.array_equal(o["node_tests"], g[f"bvh{tag}_nodes"])
        assert np.array_equal(o["prim_tests"], g[f"bvh{tag}_prims"])
        kd = orc.Kd(m, orc.load_npz(os.path.join(d, f"kd_ct{ct}.npz")))
        o = kd.trace(rays)
        ok = g[f"kd{tag}_nodes"] >= 0
        assert np.array_equal(o["seg"][ok], g[f"kd{tag}_seg"][ok])
        assert np.array_equal(o["nodes"][ok], g[f"kd{tag}_nodes"][ok])
        assert np.array_equal(o["ropes"][ok], g[f"kd{tag}_ropes"][ok])
        assert np.array_equal(o["prims"][ok], g[f"kd{tag}_prims"][ok])
        assert np.array_equal((o["status"] & 1) == 1, ~ok)


@pytest.mark.parametrize("box", [(0.0, 0.0, 1.0, 1.0), (0.0, 0.0, 1.0, 0.5)])
def test_raygen_box_entry_is_a_uniform_line_field(box):
    """BASELINE.json's ray recipe: isotropic lines with a uniform perpendicular
    offset over the box's projected width, origin at the box entry point.
    Within each direction bin, the offset n.o (n = (-dy, dx)) normalised to the
    box's projection must be uniform, and every origin lies on the side that
    faces -d."""
    from scipy.stats import kstest
    x0, y0, x1, y1 = box
    r = rg.raygen(0, box, 11, 0, 400000)
    ox, oy, dx, dy = r.T
    on_side = ((ox == x0) & (dx > 0)) | ((ox == x1) & (dx < 0)) | ((oy == y0) & (dy > 0)) | \
        ((oy == y1) & (dy < 0))
    assert on_side.all()
    ang = np.arctan2(dy, dx)
    cx = np.array([x0, x1, x1, x0])
    cy = np.array([y0, y0, y1, y1])
    for lo in np.linspace(-np.pi, np.pi, 8, endpoint=False):
        sel = (ang >= lo) & (ang < lo + np.pi / 4)
        nx, ny = -dy[sel], dx[sel]
        s = nx * ox[sel] + ny * oy[sel]
        proj = nx[:, None] * cx[None, :] + ny[:, None] * cy[None, :]
        a, b = proj.min(1), proj.max(1)
        assert kstest((s - a) / (b - a), "uniform").pvalue > 1e-4, lo


def test_degenerate_rays_reference_walk_not_brute_force():
    """Rays where the reference's walk and its brute-force oracle disagree (its
    run_experiment raises HitMismatchError on them; found over the full
    BASELINE ray sets): the oracle reproduces the reference walk's start, hit,
    t and steps, and the reference brute force, each bit for bit."""
    g = _golden("degenerate.npz")
    k = 0
    while f"{k}_cfg" in g:
        cfg, index = str(g[f"{k}_cfg"]), int(g[f"{k}_index"])
        box = (0.0, 0.0, 1.0, 0.5) if cfg.startswith("grass") else (0.0, 0.0, 1.0, 1.0)
        ray = rg.raygen(0, box, 0, index, 1)
        assert np.array_equal(ray.view(np.uint64), g[f"{k}_ray"].view(np.uint64))
        assert bool(g[f"{k}_harness_raises"])
        for w in ("cdt", "mwt"):
            om = orc.Mesh.from_files(*fixture_paths(cfg, w))
            o = om.trace(ray)
            start, seg, steps = (int(x) for x in g[f"{k}_{w}"])
            assert (int(o["start"][0]), int(o["seg"][0]), int(o["steps"][0])) == (start, seg, steps)
            assert o["t"][0] == float(g[f"{k}_{w}_t"])
        bf = om.brute_force(ray)
        assert int(bf["seg"][0]) == int(g[f"{k}_brute"][0]) != seg
        assert bf["t"][0] == g[f"{k}_brute"][1]
        k += 1
    assert k > 0


def _branch_cases():
    p = os.path.join(GOLDEN, "branches.npz")
    return [str(c) for c in np.load(p)["cases"]] if os.path.exists(p) else []


# cases whose starts the reference located itself (TriLocator); the others
# are given start triangles (wrong starts, tangled fans)
LOCATED = ("parallel_exit", "outside_")


@pytest.mark.parametrize("name", _branch_cases())
def test_branch_fixtures(name):
    """Hand-built inputs forcing the branches random rays never reach (make_golden.py
    make_branches): the oracle reproduces the reference's recorded outcomes,
    TraversalError (both kinds) exactly on the reference's rays."""
    g = _golden("branches.npz")
    m = known_mesh(g, name)
    rays = g[f"{name}__rays"]
    ref = {k[len(name) + 4:]: g[k] for k in g.files if k.startswith(f"{name}__w_")}
    out = m.trace(rays, None if name.startswith(LOCATED) else ref["start"])
    check_walk(out, ref)
    hit = (ref["error"] == 0) & (ref["seg"] >= 0)
    # the reference returns the hit point, not u: its u is recovered from the point
    assert np.all(np.abs(out["u"][hit] - ref["u"][hit]) <= 1e-9 * np.maximum(1.0, np.abs(ref["u"][hit])))
    if f"{name}__loc_pts" in g.files:
        tid, st = m.locate(g[f"{name}__loc_pts"])
        assert np.array_equal(tid, g[f"{name}__loc_anchor"])
        assert np.array_equal(tid, g[f"{name}__loc_brute"])
        assert (st & orc.ST_LOC_OUTSIDE).all()  # every point is outside the mesh


def test_branch_fixtures_reach_every_branch():
    """Across the branch fixtures the reference raised both TraversalError kinds
    and the oracle took the fallback exit, the parallel branch at a constrained
    exit, the grazing fallback and the outside-the-mesh locate."""
    g = _golden("branches.npz")
    err = np.concatenate([g[f"{c}__w_error"] for c in _branch_cases()])
    assert (err == 1).sum() > 0 and (err == 2).sum() > 0
    bits = 0
    for name in _branch_cases():
        ref_start = None if name.startswith(LOCATED) else g[f"{name}__w_start"]
        bits |= int(np.bitwise_or.reduce(known_mesh(g, name).trace(g[f"{name}__rays"], ref_start)["status"]))
    for b in (orc.ST_ERROR, orc.ST_FALLBACK, orc.ST_PARALLEL, orc.ST_GRAZING, orc.ST_ZERO_SIDE,
              orc.ST_LOC_OUTSIDE, orc.ST_LOC_BRUTE, orc.ST_MULTI, orc.ST_LOC_TIE):
        assert bits & b, f"status bit {b} never set"


@pytest.mark.parametrize("mesh", ["mwt", "cdt"])
def test_oracle_matches_full_set_reference_digests_on_sample_chunks(mesh):
    """The reference's per-chunk digests over the full BASELINE ray sets
    (tests/golden/make_digests.py): the oracle reproduces the first, a middle
    and the last chunk of every config's parts on CPU (the GPU test covers every
    chunk on the device and with the oracle)."""
    import digests as dg
    D = dg.load(mesh)
    if D is None or not D["configs"]:
        pytest.skip(f"reference digests for {mesh} not recorded")
    chunk = D["chunk"]
    for cfg, C in D["configs"].items():
        m = orc.Mesh.from_files(*fixture_paths(cfg, mesh))
        for part in C["parts"]:
            base, n, ref_chunks = part["mode"], part["n"], part["chunks"]
            mode = rg.coherent(base)
            nc = len(ref_chunks)
            for c in sorted({0, nc // 2, nc - 1}):
                lo = c * chunk
                k = min(chunk, n - lo)
                out = m.trace(orc.raygen(mode, tuple(C["box"]), D["seed"], lo, k))
                err = (out["status"] & orc.ST_ERROR) != 0
                (dw, ds), = dg.chunk_digests(out["seg"], out["t"], out["steps"], out["start"], err, chunk)
                assert (dw, ds) == tuple(ref_chunks[c][:2]), f"{cfg} part {base} chunk {c}"
