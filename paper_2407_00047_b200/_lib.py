"""ctypes declarations of include/qlm.h (argument marshalling only).

Loads the in-tree ``libqlm.so``; there is no fallback: if the library is
missing or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("QLM_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                          "libqlm.so")

QLM_OK, QLM_EINVAL, QLM_ENOMEM, QLM_ECUDA, QLM_ENCCL, QLM_EBADORDER, QLM_ERANGE = 0, 1, 2, 3, 4, 5, 6
COMM_ID_BYTES = 128
OVERRIDE = {"no_ws": 1, "no_ws2": 2, "no_two_phase": 4, "no_wide": 8, "no_tier_warp": 16, "no_graph": 32, "no_large": 64}
CAND_EXPLICIT, CAND_RANDOM, CAND_ENUM, CAND_NEIGHBOR = 0, 1, 2, 3
MAX_MOVES = 8

# numpy mirrors of the C structs (layout asserted in tests/test_abi.py)
GROUP_DTYPE = np.dtype([("model", "<i4"), ("n_req", "<i4"), ("slo_s", "<f8"), ("mu_out", "<f8"),
                        ("var_out", "<f8"), ("dist_id", "<i4"), ("reserved", "<i4")], align=True)
QUEUE_DTYPE = np.dtype([("device", "<i4"), ("resident_model", "<i4"),
                        ("backlog_mean_s", "<f8"), ("backlog_var_s2", "<f8")], align=True)


class Profile(C.Structure):
    _fields_ = [("D", C.c_int32), ("M", C.c_int32), ("theta", C.c_void_p),
                ("prefill_s", C.c_void_p), ("eps", C.c_void_p), ("decode_s", C.c_void_p),
                ("max_out", C.c_void_p), ("swap_s", C.c_void_p)]


class LenTables(C.Structure):
    _fields_ = [("K", C.c_int32), ("n_tables", C.c_int32), ("len", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("z_clamp", C.c_double), ("alpha", C.c_double), ("device", C.c_int32),
                ("reserved", C.c_int32)]


class Record(C.Structure):
    _fields_ = [("key", C.c_uint64), ("index", C.c_int64)]


class Candidates(C.Structure):
    _fields_ = [("kind", C.c_int32), ("token_bytes", C.c_int32), ("rows", C.c_void_p),
                ("stride", C.c_int64), ("seed", C.c_uint64), ("first", C.c_int64),
                ("count", C.c_int64), ("first_from", C.c_void_p), ("moves", C.c_int32),
                ("reserved", C.c_int32)]


class Tiers(C.Structure):
    _fields_ = [("model_mem", C.c_void_p), ("cpu_cap", C.c_void_p), ("load_s", C.c_void_p)]


class Requests(C.Structure):
    _fields_ = [("n", C.c_int32), ("dims", C.c_int32), ("model", C.c_void_p), ("slo_s", C.c_void_p),
                ("out_tokens", C.c_void_p), ("feat", C.c_void_p)]


class Best(C.Structure):
    _fields_ = [("index", C.c_int64), ("s1", C.c_float), ("s2", C.c_float),
                ("n_over", C.c_int32), ("reserved", C.c_int32)]


# name -> (restype, argtypes)
_vp, _i32, _i64, _u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
SIGNATURES = {
    "qlm_create": (C.c_int, [_vp, _i32, _vp, _i32, C.POINTER(Profile), C.POINTER(LenTables),
                             C.POINTER(Options), C.POINTER(C.c_void_p)]),
    "qlm_destroy": (None, [_vp]),
    "qlm_last_error": (C.c_char_p, []),
    "qlm_update_groups": (C.c_int, [_vp, _vp, _vp]),
    "qlm_score_orderings": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp, _vp]),
    "qlm_best_ordering_async": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp]),
    "qlm_reduce_records": (C.c_int, [_vp, _vp, _i32, _vp, _vp]),
    "qlm_best_ordering": (C.c_int, [_vp, C.POINTER(Candidates), C.POINTER(Best), _vp, _vp, _vp]),
    "qlm_rwt_estimate": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp, _vp]),
    "qlm_score_estimate": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                     _vp]),
    "qlm_mc_estimate": (C.c_int, [_vp, C.POINTER(Candidates), _u64, _i64, _i64, _vp, _vp]),
    "qlm_mc_sample": (C.c_int, [_vp, _u64, _i64, _i64, _vp]),
    "qlm_mc_count": (C.c_int, [_vp, C.POINTER(Candidates), _i64, _vp, _vp]),
    "qlm_decode": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp]),
    "qlm_rows": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp]),
    "qlm_check_rows": (C.c_int, [_vp, C.POINTER(Candidates), C.POINTER(C.c_int64), _vp]),
    "qlm_dims": (C.c_int, [_vp] + [C.POINTER(C.c_int32)] * 5),
    "qlm_kernel_launches": (C.c_int64, []),
    "qlm_adopt_best": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp]),
    "qlm_request_violations": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp]),
    "qlm_local_search": (C.c_int, [_vp, _vp, _i32, _i32, _i64, _i32, _u64, _vp, _vp]),
    "qlm_abi_version": (C.c_int, []),
    "qlm_set_tiers": (C.c_int, [_vp, C.POINTER(Tiers)]),
    "qlm_tiered_mc_count": (C.c_int, [_vp, C.POINTER(Candidates), _i64, _vp, _vp]),
    "qlm_form_groups": (C.c_int, [C.POINTER(Requests), _i32, _vp, _i32, _i32, _vp, _vp, _vp, _i32,
                                  C.POINTER(C.c_int32), C.POINTER(C.c_int32), _i32, _vp]),
    "qlm_tiered_score_estimate": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp, _vp, _vp, _vp,
                                            _vp, _vp]),
    "qlm_comm_unique_id": (C.c_int, [_vp]),
    "qlm_comm_attach": (C.c_int, [_vp, _vp, _i32, _i32]),
    "qlm_comm_detach": (C.c_int, [_vp]),
    "qlm_comm_info": (C.c_int, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "qlm_set_kernel_overrides": (C.c_int, [C.c_uint32, _i64]),
    "qlm_winner": (C.c_int, [_vp, C.POINTER(Candidates), _vp, _vp, _vp, _vp]),
}

_lib = None


def lib():
    """Load libqlm.so (in-tree).  Raises if it is missing -- no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; "
                               "g.build()'` (nvcc, sm_100a)")
        lib_ = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib_, name)
            f.restype = res
            f.argtypes = args
        _lib = lib_
    return _lib


class QlmError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = lib().qlm_last_error().decode(errors="replace")
        super().__init__(f"{where} failed with status {code}: {msg}")
        self.code = code


def check(code: int, where: str):
    if code != QLM_OK:
        raise QlmError(code, where)
