"""ctypes binding of libmwt.so (include/mwt.h).

The product path has no CPU fallback: if the shared library is missing this
module raises at import, and every call that fails on the device raises
``MwtError`` with the library's message.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

LIB_PATH = os.environ.get("MWT_LIB_PATH", _build.LIB)  # override: A/B of builds

# include/mwt.h constants
ST_ERROR = 1
ST_FALLBACK = 2
ST_GRAZING = 4
ST_CANON = 8
ST_PARALLEL = 16
ST_ZERO_SIDE = 32
ST_MULTI = 64
ST_LOC_TIE = 128
ST_LOC_BRUTE = 256
ST_LOC_OUTSIDE = 512
ST_OVERFLOW = 1024
ST_BOUNDARY = 2048
# bits the engine sets about its own strategy (not reference semantics)
ST_ENGINE_ONLY = ST_LOC_BRUTE | ST_BOUNDARY
STATUS_NAMES = ("error", "fallback", "grazing", "canonical", "parallel", "zero_side", "multi",
                "locate_tie", "locate_brute", "locate_outside", "overflow", "boundary_start")

RAYS_BOX_ENTRY = 0
RAYS_INTERIOR = 1


def rays_coherent(base: int, group_log2: int = 9, cell_bits: int = 12) -> int:
    """MWT_RAYS_COHERENT(base, group_log2, cell_bits) of include/mwt.h."""
    return base | (group_log2 << 8) | (cell_bits << 16)


RAYS_BOX_ENTRY_COHERENT = rays_coherent(RAYS_BOX_ENTRY)  # MWT_RAYS_BOX_ENTRY_COHERENT
RAYS_INTERIOR_COHERENT = rays_coherent(RAYS_INTERIOR)

HIST_STEP_BINS = 1024
HIST_HIT = 1024
HIST_MISS = 1025
HIST_STEPS_SUM = 1026
HIST_STATUS0 = 1027
HIST_LEN = 1040

ABI_VERSION = 3


class MwtError(RuntimeError):
    pass


class MeshInfo(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_int32), ("num_triangles", ctypes.c_int32),
                ("num_segments", ctypes.c_int32), ("anchor_res", ctypes.c_int32),
                ("anchors_not_strict", ctypes.c_int32), ("device", ctypes.c_int32),
                ("device_bytes", ctypes.c_int64), ("walk_record_bytes", ctypes.c_int64),
                ("walk_smem_bytes", ctypes.c_int64)]


# (name, restype, argtypes); every symbol declared in include/mwt.h
P = ctypes.c_void_p
I32, I64, U64, INT = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
SIGNATURES = {
    "mwt_abi_version": (INT, []),
    "mwt_last_error": (ctypes.c_char_p, []),
    "mwt_build_id": (ctypes.c_char_p, []),
    "mwt_device_count": (INT, [P]),
    "mwt_probe_l2_read": (INT, [INT, I64, INT, P]),
    "mwt_set_tuning": (INT, [INT, INT, INT]),
    "mwt_mesh_create": (INT, [P, P, I32, P, P, P, I32, P, P, I32, INT, P]),
    "mwt_mesh_destroy": (INT, [P]),
    "mwt_pack_dry_run": (INT, [P, P, I32, P, P, P, I32, P, P, I32, P, P, P, P]),
    "mwt_mesh_info_get": (INT, [P, P]),
    "mwt_mesh_anchors": (INT, [P, P]),
    "mwt_raygen_dev": (INT, [INT, P, U64, U64, I64, P, P]),
    "mwt_locate_dev": (INT, [P, P, I64, P, P, P]),
    "mwt_locate_brute_dev": (INT, [P, P, I64, P, P, P]),
    "mwt_trace_dev": (INT, [P, P, P, I64, P, P, P, P, P, P, P]),
    "mwt_trace_chain_dev": (INT, [P, P, P, I64, P, P, P, P, P, P, P]),
    "mwt_trace_host": (INT, [P, P, P, I64, P, P, P, P, P, P]),
    "mwt_trace_generated_dev": (INT, [P, INT, P, U64, U64, I64, P, P, P, P, P]),
    "mwt_histogram_dev": (INT, [P, P, P, I64, P, P]),
    "mwt_bvh_create": (INT, [P, I32, P, P, P, P, P, I32, P, P]),
    "mwt_bvh_destroy": (INT, [P]),
    "mwt_bvh_trace_dev": (INT, [P, P, I64, P, P, P, P, P, P, P]),
    "mwt_kd_create": (INT, [P, I32, I32, P, P, P, P, P, P, P, P, P, I32, P, P]),
    "mwt_kd_destroy": (INT, [P]),
    "mwt_kd_trace_dev": (INT, [P, P, P, I64, P, P, P, P, P, P, P, P]),
    "mwt_brute_force_dev": (INT, [P, P, I64, P, P, P, P]),
    "mwt_trace_generated_sharded": (INT, [P, INT, INT, P, U64, U64, I64, P]),
    "mwt_trace_host_sharded": (INT, [P, INT, P, P, I64, P, P, P, P, P, P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libmwt.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'` "
            "-- there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mwt_abi_version() != ABI_VERSION:
        raise ImportError("libmwt.so ABI version mismatch; rebuild")
    return lib


lib = _load()


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib.mwt_last_error().decode(errors="replace")
        raise MwtError(f"{what}: {msg} (code {rc})" if what else f"{msg} (code {rc})")


def ptr(a) -> ctypes.c_void_p | None:
    """Address of a numpy array or torch tensor (None passes NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)
