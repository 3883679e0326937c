"""ctypes binding of the in-tree C ABI libraries.

* ``libcosched_b200.so``  -- sm_100a sweep kernels (include/cosched_b200.h),
  built from ``csrc/sweep.cu`` with ``-gencode arch=compute_100a,code=sm_100a``.
* ``libcosched_train.so`` -- sm_100a device-side trainer (include/cosched_train.h),
  built from ``csrc/train.cu``.
* ``libcosched_match.so`` -- host C++ Edmonds matching (include/cosched_match.h).

All live next to this file (built by ``__graft_entry__.build()``).  There is
no fallback: a missing library raises ``NativeLibraryError`` with the build
command, so a GPU box never silently runs a CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
SWEEP_LIB = os.path.join(_HERE, "libcosched_b200.so")
MATCH_LIB = os.path.join(_HERE, "libcosched_match.so")
TRAIN_LIB = os.path.join(_HERE, "libcosched_train.so")

MAX_BUDGETS = 8
KERNEL_AUTO, KERNEL_TCGEN05, KERNEL_SIMT = 0, 1, 2
_lock = threading.Lock()
_libs: dict = {}


class NativeLibraryError(RuntimeError):
    """The compiled extension is missing or failed to load."""


# ---- structs (must match include/cosched_b200.h) --------------------------
c_double_p = ctypes.POINTER(ctypes.c_double)
c_float_p = ctypes.POINTER(ctypes.c_float)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_uint32_p = ctypes.POINTER(ctypes.c_uint32)
c_uint8_p = ctypes.POINTER(ctypes.c_uint8)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_ull_p = ctypes.POINTER(ctypes.c_ulonglong)


class CsNetwork(ctypes.Structure):
    _fields_ = [("w1", c_double_p), ("b1", c_double_p), ("w2", c_double_p), ("b2", c_double_p),
                ("w_out", c_double_p), ("b_out", c_double_p), ("feature_bounds", c_double_p)]


class CsGrid(ctypes.Structure):
    _fields_ = [("n_grid", ctypes.c_int32), ("knob1", c_double_p), ("knob2", c_double_p),
                ("mask", c_uint32_p), ("n_budgets", ctypes.c_int32),
                ("n_configs", ctypes.c_int32 * MAX_BUDGETS),
                ("solo_offsets", ctypes.c_int32 * (MAX_BUDGETS + 1)),
                ("solo_knob", c_double_p)]


class CsTables(ctypes.Structure):
    _fields_ = [("n_apps", ctypes.c_int32), ("n_grid", ctypes.c_int32), ("n_solo", ctypes.c_int32),
                ("w2_tile", ctypes.c_void_p), ("app_a32", c_float_p), ("app_b32", c_float_p),
                ("app_a64", c_double_p), ("app_b64", c_double_p),
                ("knob1_32", c_float_p), ("knob2_32", c_float_p),
                ("knob1_64", c_double_p), ("knob2_64", c_double_p), ("solo64", c_double_p),
                ("net_image", c_double_p), ("split_scratch", c_float_p),
                ("split_cnt", c_uint32_p), ("split_slots", ctypes.c_int32)]


class CsPairOut(ctypes.Structure):
    _fields_ = [("corun_grid_index", c_int32_p), ("corun_time", c_double_p),
                ("corun_chosen", c_uint8_p), ("weight", c_double_p)]


class CsSoloOut(ctypes.Structure):
    _fields_ = [("solo_time", c_double_p), ("solo_split", c_int32_p), ("solo_clamps", c_int32_p)]


# cs_counters (include/cosched_b200.h): 4 u32
COUNTERS_BYTES = 4 * 4


SWEEP_SYMBOLS = {
    # name: (restype, argtypes)
    "cs_version": (ctypes.c_char_p, []),
    "cs_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "cs_tables_bytes": (ctypes.c_size_t, [ctypes.c_int32] * 3),
    "cs_tables_bind": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(CsTables)]),
    "cs_build_tables": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.POINTER(CsGrid), ctypes.POINTER(CsTables),
                                       ctypes.c_void_p]),
    "cs_tables_set_network": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                             ctypes.c_void_p]),
    "cs_prepare": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int32, ctypes.POINTER(CsGrid), ctypes.POINTER(CsTables),
                                  CsSoloOut, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_solo": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                               ctypes.POINTER(CsGrid), ctypes.c_void_p, CsSoloOut, ctypes.c_void_p]),
    "cs_pair_sweep": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                     ctypes.POINTER(CsGrid), ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_double, CsPairOut, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_pair_sweep_ex": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                        ctypes.POINTER(CsGrid), ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_double, CsPairOut, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_void_p]),
    "cs_pair_screen": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                      ctypes.POINTER(CsGrid), ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_double, CsPairOut, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_void_p]),
    "cs_pair_sweep_fused": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                           ctypes.POINTER(CsGrid), ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_double, CsPairOut,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "cs_pair_screen_fused": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                            ctypes.POINTER(CsGrid), ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_double, CsPairOut,
                                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "cs_resolve_fused": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                        ctypes.POINTER(CsGrid), ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        CsPairOut, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_resolve": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsTables),
                                  ctypes.POINTER(CsGrid), ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.c_int64, CsPairOut, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p]),
    "cs_pair_decide": (ctypes.c_int, [ctypes.POINTER(CsGrid), ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, CsPairOut,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_scatter_weights": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_wire_records_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32]),
    "cs_pack_records": (ctypes.c_int, [CsPairOut, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "cs_unpack_gathered": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                          CsPairOut, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_analytic_sweep": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, c_double_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_int32, CsPairOut,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "cs_forward_rows": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "cs_device_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "cs_device_free": (ctypes.c_int, [ctypes.c_void_p]),
    "cs_workspace_retain": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t]),
    "cs_workspace_release": (ctypes.c_int, [ctypes.c_void_p]),
    "cs_build_graph_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.POINTER(CsGrid)]),
    "cs_build_graph_host": (ctypes.c_int, [ctypes.POINTER(CsNetwork), ctypes.POINTER(CsGrid),
                                           c_double_p, c_double_p, ctypes.c_int32,
                                           ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t,
                                           c_double_p, CsPairOut, CsSoloOut, c_ull_p,
                                           ctypes.c_void_p]),
}

TRAIN_SYMBOLS = {
    "ct_version": (ctypes.c_char_p, []),
    "ct_backward": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ct_train_sgd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                    ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32,
                                    ctypes.c_int32, ctypes.c_double, ctypes.c_int32, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
}

MATCH_SYMBOLS = {
    "cm_version": (ctypes.c_char_p, []),
    "cm_max_weight_matching": (ctypes.c_int, [c_double_p, ctypes.c_int32, c_int32_p]),
    "cm_min_weight_perfect_matching": (ctypes.c_int, [c_double_p, ctypes.c_int32, c_int32_p]),
    "cm_min_weight_perfect_matching_k": (ctypes.c_int, [c_double_p, ctypes.c_int32, ctypes.c_int32,
                                                        c_int32_p]),
    "cm_min_weight_perfect_matching_pot": (ctypes.c_int, [c_double_p, ctypes.c_int32, c_double_p,
                                                          ctypes.c_int32, c_int32_p]),
}


def _load(path: str, symbols: dict, what: str):
    with _lock:
        if path in _libs:
            return _libs[path]
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{what} not built: {path} is missing. Run `python -c \"import __graft_entry__ as g; "
                f"g.build()\"` from the repo root (nvcc for sm_100a / g++).")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in symbols.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _libs[path] = lib
        return lib


def sweep_lib():
    return _load(SWEEP_LIB, SWEEP_SYMBOLS, "CUDA sweep extension")


def match_lib():
    return _load(MATCH_LIB, MATCH_SYMBOLS, "C++ matching library")


def train_lib():
    return _load(TRAIN_LIB, TRAIN_SYMBOLS, "CUDA training extension")


def check(rc: int, what: str) -> None:
    """Map a CS_ERR_* code to the reference's exception types."""
    if rc == 0:
        return
    from .core import ValidationError
    msg = sweep_lib().cs_error_string(rc).decode()
    if rc in (-1, -2, -3):
        raise ValidationError(f"{what}: {msg}")
    if rc == -5:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (code {rc})")


def ptr(arr, ctype=c_double_p):
    """Pointer to a C-contiguous numpy array (kept alive by the caller)."""
    return arr.ctypes.data_as(ctype)
