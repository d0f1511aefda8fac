"""pytest plugin: run the reference's own tests with mintri.accel's query
functions routed to the B200 drop-in (paper_2112_05570_b200.accel).

Loaded with ``-p mwt_dropin_plugin`` before collection, so the reference test
modules' ``from mintri.accel import ...`` bind the drop-ins.  Patched in
mintri.accel (whose Bvh.intersect / RopedKdTree.intersect resolve these names
at call time), in the mintri package namespace and in mintri.experiment.
The builders (build_cdt, build_bvh, build_kdtree, SceneIndex, sample_rays)
stay the reference's: the drop-in takes the reference-built objects as input.
"""
import mintri
import mintri.accel as ref_accel
import mintri.experiment as ref_experiment

from paper_2112_05570_b200 import accel as dropin

QUERIES = ("traverse_triangulation", "TriLocator", "locate_triangle", "bvh_intersect", "kd_intersect",
           "brute_force_closest", "sweep_structure_params")

import collections
import functools
import sys

# the drop-in raises the reference's own exception type
dropin.TraversalError = ref_accel.TraversalError
CALLS = collections.Counter()


def _counted(name, fn):
    if isinstance(fn, type):  # TriLocator: count constructions (its locate runs on the device)
        class Counted(fn):
            def __init__(self, *a, **k):
                CALLS[name] += 1
                super().__init__(*a, **k)
        Counted.__name__ = fn.__name__
        return Counted

    @functools.wraps(fn)
    def wrapper(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)
    return wrapper


PATCHED = {name: _counted(name, getattr(dropin, name)) for name in QUERIES}
for mod in (ref_accel, mintri, ref_experiment):
    for name in QUERIES:
        if hasattr(mod, name):
            setattr(mod, name, PATCHED[name])
# the structures' own methods (Bvh.intersect / RopedKdTree.intersect) call the
# module-level names, which now resolve to the drop-ins


def pytest_configure(config):
    print(f"mwt drop-in: mintri.accel.{{{', '.join(QUERIES)}}} -> paper_2112_05570_b200.accel (B200)",
          file=sys.stderr, flush=True)


def pytest_sessionfinish(session, exitstatus):
    print("mwt drop-in calls: " + ", ".join(f"{k}={CALLS[k]}" for k in QUERIES), file=sys.stderr, flush=True)
