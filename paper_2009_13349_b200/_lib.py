"""ctypes binding of libtccd.so (include/tccd.h).

The shared library is built in-tree (``make -C paper_2009_13349_b200/csrc``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or fails to load, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCCD_LIB") or os.path.join(_HERE, "libtccd.so")  # override: experiments only

ABI_VERSION = 3
FLAG_HEAVY_ONLY = 1
FLAG_NO_LANE = 2

# solver stages per chunk, in launch order (TCCD_STAGE_*)
STAGES = ("prologue", "lane", "light", "medium", "giant")

# diagnostic counters (TCCD_STAT_*, include/tccd.h)
NUM_STATS = 32
STAT_GIANT_QUERIES = 0
STAT_ROUNDS = 1
STAT_DEFERRALS = 2
STAT_MEDIUM_QUERIES = 3
STAT_BOXES = 4          # [4..6]
STAT_LANE_QUERIES = 7
STAT_CLS = 8            # [8..13]
STAT_LANE_CLS = 14      # [14..15]
STAT_LANE_CHECKS = 16   # [16..17]
STAT_LANE_DONE = 18     # [18..19]
STAT_LANE_EVICTED = 20
STAT_LANE_WASTED = 21
STAT_POOL_DEMAND = 22   # [22..23]
STAT_RESTARTS = 24      # [24..25]
STAT_TIER_CHECKS = 26   # [26..28]
STAT_PROLOGUE_DONE = 29
STAT_LANE_HANDED = 30
STAT_CHUNKS = 31

STATUS_FREE = 0
STATUS_HIT = 1
STATUS_ERR_SEPARATION = 2
STATUS_ERR_NONFINITE = 3
STATUS_ERR_PARAM = 4

_vp = ctypes.c_void_p


class TccdBatch(ctypes.Structure):
    """Mirror of ``struct tccd_batch`` (include/tccd.h)."""

    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("flags", ctypes.c_uint32),
        ("n", ctypes.c_int64),
        ("points", _vp),
        ("kind", _vp),
        ("kind_all", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
        ("delta", _vp),
        ("delta_all", ctypes.c_double),
        ("max_checks", _vp),
        ("max_checks_all", ctypes.c_int64),
        ("max_checks_max", ctypes.c_int64),
        ("separation", _vp),
        ("separation_all", ctypes.c_double),
        ("t_max", _vp),
        ("t_max_all", ctypes.c_double),
        ("eps", _vp),
        ("status", _vp),
        ("toi", _vp),
        ("tol", _vp),
        ("codom", _vp),
        ("checks", _vp),
        ("early", _vp),
        ("witness", _vp),
        ("level", _vp),
        ("workspace", _vp),
        ("workspace_bytes", ctypes.c_size_t),
        ("heavy_blocks", ctypes.c_int32),
        ("device_sms", ctypes.c_int32),
        ("stats", _vp),
        ("events", _vp),
        ("event_stage", _vp),
        ("n_events", ctypes.c_int32),
        ("events_used", ctypes.c_int32),
        ("input_events", _vp),
        ("input_chunk", ctypes.c_int64),
        ("n_input_events", ctypes.c_int32),
        ("reserved1", ctypes.c_int32),
        ("hit_index", _vp),
        ("hit_toi", _vp),
        ("hit_count", _vp),
        ("hit_capacity", ctypes.c_int64),
        ("hit_index_base", ctypes.c_int64),
        ("pool_boxes", ctypes.c_int64),
        ("launches", ctypes.c_int64),
    ]


class TccdMesh(ctypes.Structure):
    """Mirror of ``struct tccd_mesh`` (include/tccd.h)."""

    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("n_vertices", ctypes.c_int64),
        ("n_triangles", ctypes.c_int64),
        ("n_edges", ctypes.c_int64),
        ("x0", _vp),
        ("x1", _vp),
        ("triangles", _vp),
        ("edges", _vp),
    ]


EXPORTS = (
    "tccd_abi_version",
    "tccd_error_string",
    "tccd_workspace_bytes",
    "tccd_workspace_bytes_ex",
    "tccd_solve_batch",
    "tccd_solve_kernel",
    "tccd_broad_create",
    "tccd_broad_emit",
    "tccd_broad_destroy",
    "tccd_copy_to_host",
    "tccd_copy_counted_to_host",
    "tccd_release_cached",
    "tccd_box_hulls",
    "tccd_kappas",
    "tccd_irf_workspace_bytes",
    "tccd_irf_batch",
)

_lib = None


class TccdError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: tccd error {code}: {error_string(code)}")
        self.code = code


def lib() -> ctypes.CDLL:
    """Load libtccd.so (raises if it is missing: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not built; run `make -C {_HERE}/csrc` or __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.tccd_abi_version.restype = ctypes.c_int
        L.tccd_abi_version.argtypes = []
        L.tccd_error_string.restype = ctypes.c_char_p
        L.tccd_error_string.argtypes = [ctypes.c_int]
        L.tccd_workspace_bytes.restype = ctypes.c_size_t
        L.tccd_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32]
        L.tccd_workspace_bytes_ex.restype = ctypes.c_size_t
        L.tccd_workspace_bytes_ex.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                              ctypes.c_int64]
        L.tccd_release_cached.restype = None
        L.tccd_release_cached.argtypes = []
        L.tccd_box_hulls.restype = ctypes.c_int
        L.tccd_box_hulls.argtypes = [_vp, _vp, ctypes.c_int, _vp, ctypes.c_int64, _vp, _vp, _vp]
        L.tccd_kappas.restype = ctypes.c_int
        L.tccd_kappas.argtypes = [_vp, _vp, ctypes.c_int, _vp, ctypes.c_double, ctypes.c_int64,
                                  _vp, _vp]
        L.tccd_solve_batch.restype = ctypes.c_int
        L.tccd_solve_batch.argtypes = [ctypes.POINTER(TccdBatch), _vp]
        L.tccd_solve_kernel.restype = ctypes.c_int
        L.tccd_solve_kernel.argtypes = [
            _vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int64,
            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp]
        L.tccd_broad_create.restype = ctypes.c_int
        L.tccd_broad_create.argtypes = [ctypes.POINTER(TccdMesh), ctypes.c_double,
                                        ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_int64), _vp]
        L.tccd_broad_emit.restype = ctypes.c_int
        L.tccd_broad_emit.argtypes = [_vp, _vp, _vp, _vp]
        L.tccd_broad_destroy.restype = None
        L.tccd_broad_destroy.argtypes = [_vp]
        L.tccd_irf_workspace_bytes.restype = ctypes.c_size_t
        L.tccd_irf_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32]
        L.tccd_irf_batch.restype = ctypes.c_int
        L.tccd_irf_batch.argtypes = [ctypes.POINTER(TccdBatch), _vp]
        L.tccd_copy_to_host.restype = ctypes.c_int
        L.tccd_copy_to_host.argtypes = [_vp, _vp, ctypes.c_int64, _vp]
        L.tccd_copy_counted_to_host.restype = ctypes.c_int
        L.tccd_copy_counted_to_host.argtypes = [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                                _vp, _vp]
        v = L.tccd_abi_version()
        if v != ABI_VERSION:
            raise RuntimeError(f"libtccd ABI {v} != expected {ABI_VERSION}")
        _lib = L
    return _lib


def error_string(code: int) -> str:
    return lib().tccd_error_string(int(code)).decode()


def check(code: int, where: str) -> None:
    if code != 0:
        raise TccdError(code, where)
