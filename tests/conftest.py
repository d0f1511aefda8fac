import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FIXTURES = os.path.join(ROOT, "fixtures", "data")
GOLDEN = os.path.join(ROOT, "tests", "golden")
# BASELINE.json configs[0..4], then Grass / Hair under the other crossing
# policies (fixtures/gen_fixtures.py: lane confinement, turn resampling)
CONFIGS = ["lines64", "lines1024", "grass4096", "hair512", "floorplan64", "grass4096l", "hair512r"]
BOXES = {"grass4096": (0.0, 0.0, 1.0, 0.5), "grass4096l": (0.0, 0.0, 1.0, 0.5)}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def pytest_sessionstart(session):
    """A clean checkout has no built libraries (they are not committed):
    build them once (nvcc cross-compiles for sm_100a without a GPU)."""
    libs = [os.path.join(ROOT, "paper_2112_05570_b200", "_build", "libmwt.so"),
            os.path.join(ROOT, "oracle", "_build", "libmwt_oracle.so")]
    if not all(os.path.exists(p) for p in libs):
        import __graft_entry__
        __graft_entry__.build()


def fixture_paths(cfg: str, mesh: str):
    d = os.path.join(FIXTURES, cfg)
    tri = os.path.join(d, f"{mesh}.tri")
    if not os.path.exists(tri):
        return None
    return os.path.join(d, "scene.txt"), tri


def box_of(cfg: str):
    return BOXES.get(cfg, (0.0, 0.0, 1.0, 1.0))


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
