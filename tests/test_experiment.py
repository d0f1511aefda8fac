"""The harness layer (experiment.py:29-202): the reference's ray sampler
reproduced bit-for-bit on the host, and run_experiment on the device engines
against the reference's own report (tests/golden/experiment.npz)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, fixture_paths


def _golden():
    p = os.path.join(GOLDEN, "experiment.npz")
    if not os.path.exists(p):
        pytest.skip("experiment golden not generated")
    return np.load(p)


def test_sample_rays_bit_exact():
    from paper_2112_05570_b200.experiment import sample_rays_array
    from paper_2112_05570_b200.model import Scene
    g = _golden()
    scene = Scene.load(fixture_paths("lines1024", "mwt")[0])
    for key, (count, seed) in (("rays", (3000, 11)), ("sample5000_seed5", (5000, 5))):
        got = sample_rays_array(scene, count, seed)
        assert np.array_equal(got.view(np.uint64), g[key].view(np.uint64)), key


def test_sample_rays_rejects_bad_count():
    from paper_2112_05570_b200.experiment import sample_rays_array
    from paper_2112_05570_b200.model import Scene
    with pytest.raises(ValueError):
        sample_rays_array(Scene.load(fixture_paths("lines64", "mwt")[0]), 0)


@pytest.mark.gpu
def test_run_experiment_matches_reference_report():
    from paper_2112_05570_b200.experiment import run_experiment
    from paper_2112_05570_b200.formats import load_structure
    from paper_2112_05570_b200.model import Scene, load_triangulation
    g = _golden()
    paths = fixture_paths("lines1024", "mwt")
    d = os.path.dirname(paths[0])
    scene = Scene.load(paths[0])
    tris = [load_triangulation(os.path.join(d, f"{w}.tri"), scene) for w in ("cdt", "mwt")]
    grid = (0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0)
    bvh = {c: load_structure(os.path.join(d, f"bvh_ct{c:g}.npz")) for c in grid}
    kd = {c: load_structure(os.path.join(d, f"kd_ct{c:g}.npz")) for c in grid}
    rep = run_experiment(scene, tris, g["rays"], labels=["cdt", "mwt"], ct_grid=grid,
                         bvh_structures=bvh, kd_structures=kd)
    got = json.loads(rep.to_json())
    got.pop("timing")
    ref = json.loads(str(g["report"]))
    # the scene name comes from the scene file; everything else must be identical
    got["scene"] = ref["scene"]
    for m in got["methods"] + ref["methods"]:
        m["mean_total"] = round(m["mean_total"], 9)
        m["means"] = {k: round(v, 9) for k, v in m["means"].items()}
    assert got == ref
    assert rep.to_csv().splitlines()[1:] == str(g["csv"]).splitlines()[1:] or \
        [ln.split(",")[1:] for ln in rep.to_csv().splitlines()[1:]] == \
        [ln.split(",")[1:] for ln in str(g["csv"]).splitlines()[1:]]
