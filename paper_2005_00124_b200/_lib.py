"""ctypes binding of the C ABI declared in include/wagma_b200.h.

The library is built in-tree by `_build.build()` (``__graft_entry__.build``).
There is no fallback: if the shared library is missing or cannot be loaded,
importing the device path raises immediately.
"""

from __future__ import annotations

import ctypes
import os

from . import _build

(WG_OK, WG_EINVAL, WG_EVERSION, WG_ESTALE, WG_EPROTO, WG_ETIMEOUT, WG_ECUDA, WG_ENOMEM, WG_EDIVERGE,
 WG_ESYNC) = range(10)
WG_RULE_EXAMPLE, WG_RULE_LITERAL = 0, 1
WG_F32, WG_F64 = 0, 1
WG_JOB_STEP, WG_JOB_SYNC_STEP, WG_JOB_LOCAL_STEP, WG_JOB_GROUP_SUM, WG_JOB_SYNC_SUM = range(5)
WG_UPDATE_SGD, WG_UPDATE_MOMENTUM = 0, 1

RULES = {"example": WG_RULE_EXAMPLE, "literal": WG_RULE_LITERAL}


class WgConfig(ctypes.Structure):
    _fields_ = [
        ("P", ctypes.c_int32), ("S", ctypes.c_int32), ("n_gpus", ctypes.c_int32),
        ("gpu_index", ctypes.c_int32), ("device", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("mask_rule", ctypes.c_int32), ("activation_enabled", ctypes.c_int32),
        ("n", ctypes.c_int64), ("tau", ctypes.c_int64), ("staleness_bound", ctypes.c_int64),
        ("ring_depth", ctypes.c_int32), ("version_ring", ctypes.c_int32),
        ("grace_ns", ctypes.c_int64), ("timeout_ns", ctypes.c_int64),
    ]


class WgJob(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32), ("kind", ctypes.c_int32), ("version", ctypes.c_int64),
        ("update_rule", ctypes.c_int32), ("pad", ctypes.c_int32),
        ("eta", ctypes.c_double), ("beta", ctypes.c_double),
        ("W", ctypes.c_void_p), ("m", ctypes.c_void_p), ("g", ctypes.c_void_p),
        ("fresh", ctypes.c_void_p), ("acc_out", ctypes.c_void_p),
    ]


class WgJobStatus(ctypes.Structure):
    _fields_ = [
        ("version", ctypes.c_int64), ("contrib_stamp", ctypes.c_int64),
        ("timely", ctypes.c_int32), ("activator", ctypes.c_int32),
        ("error", ctypes.c_int32), ("root", ctypes.c_int32),
    ]


_I = ctypes.c_int
_I64 = ctypes.c_int64
_PI = ctypes.POINTER(ctypes.c_int)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_VP = ctypes.c_void_p

# every symbol of include/wagma_b200.h with its ctypes signature
SIGNATURES = {
    "wg_check_params": (_I, [_I, _I, _I64]),
    "wg_phase_masks": (_I, [_I, _I, _I64, _I, _PI, _PI]),
    "wg_compute_groups": (_I, [_I, _I, _I64, _I, _PI, _PI, _PI]),
    "wg_group_of": (_I, [_I, _I, _I64, _I, _I, _PI, _PI]),
    "wg_peer": (_I, [_I, _I, _I, _PI]),
    "wg_mixing_reachable": (_I, [_I, _I, _I64, _I, _I, _PI]),
    "wg_tree_leaves": (_I, [_I, _I, _I64, _I, _I, _PI, _PI]),
    "wg_ctx_create": (_I, [ctypes.POINTER(WgConfig), ctypes.POINTER(_VP)]),
    "wg_ctx_destroy": (_I, [_VP]),
    "wg_ctx_export": (_I, [_VP, _VP, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "wg_ctx_import_peer": (_I, [_VP, _I, _VP, ctypes.c_size_t]),
    "wg_ctx_set_initial_model": (_I, [_VP, _I, _VP, _VP]),
    "wg_install": (_I, [_VP, _I, _I64, _VP, _VP]),
    "wg_ctx_slot": (_I, [_VP, _I, _I64, ctypes.POINTER(_VP), _PI64]),
    "wg_launch": (_I, [_VP, ctypes.POINTER(WgJob), _I, _PI64, _PI64, _I, _VP]),
    "wg_launch_status": (_I, [_VP, _I, ctypes.POINTER(WgJobStatus)]),
    "wg_query_version": (_I, [_VP, _I64, _PI64, _PI]),
    "wg_ctx_error": (_I, [_VP, _PI, _PI64]),
    "wg_ctx_error_async": (_I, [_VP, _PI, _PI64]),
    "wg_ctx_clear_error": (_I, [_VP]),
    "wg_delay": (_I, [_VP, _I64, _VP]),
    "wg_replicas_sum": (_I, [_VP, ctypes.POINTER(_VP), _I, _VP, _VP]),
    "wg_replicas_spread": (_I, [_VP, ctypes.POINTER(_VP), _I, _VP, _VP, _VP]),
    "wg_ctx_set_profile": (_I, [_VP, _VP]),
    "wg_ctx_geometry": (_I, [_VP, _PI64, _PI64, _PI, _PI]),
    "wg_strerror": (ctypes.c_char_p, [_I]),
    "wg_last_error_message": (ctypes.c_char_p, []),
}

_lib = None


def lib_path() -> str:
    # WAGMA_B200_LIB: load an alternative build (A/B kernel experiments)
    return os.environ.get("WAGMA_B200_LIB", _build.LIB_PATH)


def load(build_if_missing: bool = False) -> ctypes.CDLL:
    """Load libwagma_b200.so (fail loudly if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing:
            raise ImportError(
                f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                "There is no CPU fallback for the WAGMA hot path.")
        _build.build()
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None and "WAGMA_B200_LIB" in os.environ:
            continue  # older experimental build without this entry point
        if fn is None:
            raise ImportError(f"{path} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().wg_last_error_message()
    return msg.decode() if msg else ""
