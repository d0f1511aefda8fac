"""Full-set parity at BASELINE sizes: every ray of every config (2^20 .. 2^26,
the benchmark's coherent generator order, seed 0) through the engine, against
per-chunk digests of what the UNMODIFIED reference computed for the same rays
(tests/golden/digests_<mesh>.json, tests/golden/make_digests.py: reference
TriLocator.locate + traverse_triangulation, ~35 CPU-minutes per mesh).

Three paths are checked chunk by chunk:
  * the fused benchmark path (mwt_trace_generated_dev: rays generated, located
    and walked in one launch) -- seg / t / steps, and its histogram;
  * the explicit path (mwt_raygen_dev + mwt_trace_dev) -- also the start
    triangles and the TraversalError status;
  * the oracle (oracle/mwt_oracle.c on the host's cores) -- the pinned checker,
    which names the differing rays if a chunk ever disagrees.
"""
import os

import numpy as np
import pytest

import digests as dg
from conftest import fixture_paths

pytestmark = pytest.mark.gpu

CFGS = ["lines64", "lines1024", "grass4096", "hair512", "floorplan64", "grass4096l", "hair512r"]
COHERENT = (9, 12)


def _mode(base):
    return base | (COHERENT[0] << 8) | (COHERENT[1] << 16)


def _cases():
    out = []
    for mesh in ("mwt", "cdt"):
        d = dg.load(mesh)
        for cfg in CFGS:
            out.append((cfg, mesh))
    return out


def _explain(om, box, base, lo, n, got):
    """Oracle on one chunk: the indices where the engine differs from it."""
    from oracle import oracle as orc
    rays = orc.raygen(_mode(base), box, 0, lo, n)
    ref = om.trace(rays)
    bad = np.nonzero((ref["seg"] != got["seg"][lo:lo + n]) | (ref["steps"] != got["steps"][lo:lo + n]))[0]
    return f"oracle differs from the engine at {len(bad)} rays, first {(bad[:8] + lo).tolist()}"


@pytest.mark.parametrize("cfg,mesh", _cases())
def test_full_ray_set_matches_reference_digests(cfg, mesh):
    import torch
    from oracle import oracle as orc
    from paper_2112_05570_b200 import _lib
    from paper_2112_05570_b200.engine import DeviceMesh, new_histogram
    from paper_2112_05570_b200.sharding import histogram_host
    D = dg.load(mesh)
    if D is None or cfg not in D["configs"]:
        pytest.skip(f"reference digests for {cfg}/{mesh} not recorded")
    C = D["configs"][cfg]
    box = tuple(C["box"])
    chunk = D["chunk"]
    paths = fixture_paths(cfg, mesh)
    m = DeviceMesh.from_files(*paths)
    om = orc.Mesh.from_files(*paths)
    for part in C["parts"]:
        base, n, ref_chunks = part["mode"], part["n"], part["chunks"]
        mode = _mode(base)
        # fused benchmark path
        h = new_histogram()
        fused = m.trace_generated_device(mode, box, 0, 0, n, outputs=True, hist=h)
        # explicit path
        rays = m.raygen_device(mode, box, 0, 0, n)
        ex = m.trace_device(rays, None, want=("start", "seg", "t", "steps", "status"))
        torch.cuda.synchronize()
        for k in ("seg", "steps"):
            assert torch.equal(fused[k], ex[k]), f"{cfg}/{mesh}: fused != explicit ({k})"
        hit = ex["seg"] >= 0
        assert torch.equal(fused["t"][hit], ex["t"][hit])
        got = {k: v.cpu().numpy() for k, v in ex.items()}
        err = (got["status"].view(np.uint32) & _lib.ST_ERROR) != 0
        hd = h.cpu().numpy()
        assert np.array_equal(hd, histogram_host(got["seg"], got["steps"], got["status"].view(np.uint32)))
        del rays, ex, fused
        mine = dg.chunk_digests(got["seg"], got["t"], got["steps"], got["start"], err, chunk)
        assert len(mine) == len(ref_chunks)
        for c, ((dw, ds), r) in enumerate(zip(mine, ref_chunks)):
            lo = c * chunk
            if dw != r[0] or ds != r[1]:
                pytest.fail(f"{cfg}/{mesh} part {base} chunk {c} (rays {lo}..{lo + chunk - 1}): "
                            f"walk {'ok' if dw == r[0] else 'DIFFERS'}, start {'ok' if ds == r[1] else 'DIFFERS'}; "
                            + _explain(om, box, base, lo, min(chunk, n - lo), got))
        # the reference's per-chunk totals agree with the histogram
        assert sum(r[3] for r in ref_chunks) == int(hd[_lib.HIST_HIT])
        assert sum(r[4] for r in ref_chunks) == int(got["steps"][~err].astype(np.int64).sum())
        assert sum(r[2] for r in ref_chunks) == int(err.sum())
        # the pinned oracle, over the whole part on the host's cores
        ref = om.trace(orc.raygen(mode, box, 0, 0, n))
        oerr = (ref["status"] & orc.ST_ERROR) != 0
        theirs = dg.chunk_digests(ref["seg"], ref["t"], ref["steps"], ref["start"], oerr, chunk)
        assert [tuple(x[:2]) for x in ref_chunks] == theirs, f"{cfg}/{mesh}: oracle != reference digests"


@pytest.mark.parametrize("cfg,mesh", _cases())
def test_full_iid_ray_set_matches_oracle(cfg, mesh):
    """The iid generator order (no coherent groups) at the same BASELINE sizes:
    every ray through the fused path and the explicit path, against the
    oracle (pinned to the reference by the digests above and the goldens) on
    the host's cores -- start, seg, steps, status and t bit-exact."""
    import torch
    from oracle import oracle as orc
    from paper_2112_05570_b200.engine import DeviceMesh
    D = dg.load(mesh)
    if D is None or cfg not in D["configs"]:
        pytest.skip(f"{cfg}/{mesh}: no BASELINE sizes recorded")
    C = D["configs"][cfg]
    box = tuple(C["box"])
    paths = fixture_paths(cfg, mesh)
    m = DeviceMesh.from_files(*paths)
    om = orc.Mesh.from_files(*paths)
    orc.set_num_threads(os.cpu_count() or 1)
    step = 1 << 23
    for part in C["parts"]:
        base, n = part["mode"], part["n"]
        for lo in range(0, n, step):
            k = min(step, n - lo)
            fused = m.trace_generated_device(base, box, 0, lo, k, outputs=True, hist=None)
            rays = m.raygen_device(base, box, 0, lo, k)
            ex = m.trace_device(rays, None, want=("start", "seg", "t", "steps", "status"))
            torch.cuda.synchronize()
            got = {x: v.cpu().numpy() for x, v in ex.items()}
            for x in ("seg", "steps"):
                assert np.array_equal(fused[x].cpu().numpy(), got[x]), f"{cfg}/{mesh}: fused != explicit ({x})"
            del fused, rays, ex
            ref = om.trace(orc.raygen(base, box, 0, lo, k))
            st_bits = np.uint32(orc.ST_ERROR)
            assert np.array_equal(got["status"].view(np.uint32) & st_bits, ref["status"] & st_bits)
            ok = (ref["status"] & st_bits) == 0  # (the step count of a TraversalError is not a result)
            for x in ("start", "seg", "steps"):
                bad = np.nonzero((got[x] != ref[x]) & (ok if x == "steps" else True))[0]
                assert len(bad) == 0, f"{cfg}/{mesh} rays {lo}+{bad[:5].tolist()}: {x} differs from the oracle"
            hit = ref["seg"] >= 0
            assert np.array_equal(got["t"][hit].view(np.uint64), ref["t"][hit].view(np.uint64))
