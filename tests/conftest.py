import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FIXTURES = os.path.join(ROOT, "fixtures", "data")
GOLDEN = os.path.join(ROOT, "tests", "golden")
CONFIGS = ["lines64", "lines1024", "grass4096", "hair512", "floorplan64"]
BOXES = {"grass4096": (0.0, 0.0, 1.0, 0.5)}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


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
