"""ctypes binding of libpbnsim (include/pbnsim.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module
only converts Python / numpy / torch objects into the C structs.  There is
no CPU fallback: if the extension is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpbnsim.so")
# experiments only: an alternative in-tree build (e.g. libpbnsim_u16.so) by file name
if os.environ.get("PBN_LIB_VARIANT"):
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), os.environ["PBN_LIB_VARIANT"])

# status codes
PBN_OK = 0
PBN_E_INVALID = 1
PBN_E_USAGE = 2
PBN_E_DEGENERATE = 3
PBN_E_NOT_CONVERGED = 4
PBN_E_IO = 5
PBN_E_CUDA = 6
PBN_E_NOMEM = 7
STATUS_NAMES = {0: "PBN_OK", 1: "PBN_E_INVALID", 2: "PBN_E_USAGE", 3: "PBN_E_DEGENERATE",
                4: "PBN_E_NOT_CONVERGED", 5: "PBN_E_IO", 6: "PBN_E_CUDA", 7: "PBN_E_NOMEM"}

PBN_PERTURB_VECTOR = 0
PBN_PERTURB_PER_NODE = 1
PBN_PERTURB_GEOMETRIC = 2
PBN_LAYOUT_AUTO = 0
PBN_LAYOUT_CHAIN_LANES = 1
PBN_LAYOUT_NODE_LANES = 2
PBN_METHOD_TWO_STATE = 0
PBN_METHOD_SKART = 1


class PbnError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")


class pbn_model_desc(C.Structure):
    _fields_ = [("n", C.c_int32), ("fn_off", C.POINTER(C.c_int32)), ("par_off", C.POINTER(C.c_int32)),
                ("parents", C.POINTER(C.c_uint16)), ("tbl_off", C.POINTER(C.c_int32)),
                ("tables", C.POINTER(C.c_uint32)), ("sel_prob", C.POINTER(C.c_double)),
                ("p", C.c_double), ("flags", C.c_uint32)]


class pbn_model_info(C.Structure):
    _fields_ = [("n", C.c_int32), ("nf", C.c_int32), ("n_parents", C.c_int64), ("density", C.c_double),
                ("T_p", C.c_uint32), ("flags", C.c_uint32), ("max_ell", C.c_int32),
                ("max_theta", C.c_int32), ("image_bytes", C.c_int64)]


class pbn_predicate(C.Structure):
    _fields_ = [("k", C.c_int32), ("node", C.POINTER(C.c_uint16)), ("value", C.POINTER(C.c_uint8))]


class pbn_sim_args(C.Structure):
    _fields_ = [("n_chains", C.c_int64), ("chain_base", C.c_int64), ("step0", C.c_int64),
                ("burn_in", C.c_int64), ("steps", C.c_int64), ("batch", C.c_int64),
                ("seed", C.c_uint64), ("pred", pbn_predicate), ("init", C.c_int32),
                ("emit_bits", C.c_int32), ("bits_offset", C.c_int64), ("bits_row_words", C.c_int64),
                ("groups_per_cta", C.c_int32), ("warps_per_group", C.c_int32),
                ("schedule", C.c_int32), ("chunk_steps", C.c_int64), ("n_props", C.c_int32),
                ("props", C.c_void_p), ("cluster_size", C.c_int32), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_int64), ("layout", C.c_int32), ("chains_per_cluster", C.c_int32)]


class pbn_sim_out(C.Structure):
    _fields_ = [("state", C.c_void_p), ("c1", C.c_void_p), ("n01", C.c_void_p), ("n10", C.c_void_p),
                ("first_last", C.c_void_p), ("batch_sums", C.c_void_p), ("bits", C.c_void_p),
                ("totals", C.c_void_p)]


class pbn_two_state_result(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("M_raw", C.c_double),
                ("N_raw", C.c_double), ("M", C.c_int64), ("N", C.c_int64)]


class pbn_skart_ci(C.Structure):
    _fields_ = [("mu", C.c_double), ("var", C.c_double), ("phi", C.c_double), ("skew", C.c_double),
                ("ci_lo", C.c_double), ("ci_hi", C.c_double), ("H", C.c_double), ("batches", C.c_int64)]


class pbn_skart_result(C.Structure):
    _fields_ = [("estimate", C.c_double), ("ci_lo", C.c_double), ("ci_hi", C.c_double), ("H", C.c_double),
                ("skew", C.c_double), ("kappa", C.c_int64), ("batches", C.c_int64), ("spacer", C.c_int64),
                ("eta", C.c_int64), ("need_per_chain", C.c_int64), ("randomness_tests", C.c_int32)]


class pbn_run_args(C.Structure):
    _fields_ = [("method", C.c_int32), ("omega", C.c_int64), ("psi0", C.c_int64),
                ("rhat_threshold", C.c_double), ("r", C.c_double), ("s", C.c_double),
                ("eps", C.c_double), ("h_star", C.c_double), ("alpha_conf", C.c_double),
                ("seed", C.c_uint64), ("pred", pbn_predicate), ("max_steps", C.c_int64)]


class pbn_prop_result(C.Structure):
    _fields_ = [("estimate", C.c_double), ("rhat", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("M", C.c_int64), ("N", C.c_int64), ("status", C.c_int32)]


class pbn_run_result(C.Structure):
    _fields_ = [("estimate", C.c_double), ("ci_lo", C.c_double), ("ci_hi", C.c_double),
                ("rhat", C.c_double), ("psi", C.c_int64), ("sample_size", C.c_int64),
                ("steps_per_chain", C.c_int64), ("gr_iterations", C.c_int64),
                ("extensions", C.c_int64), ("M", C.c_int64), ("N", C.c_int64),
                ("alpha", C.c_double), ("beta", C.c_double)]


# symbol -> (restype, argtypes); the exact list include/pbnsim.h declares
SIGNATURES = {
    "pbn_validate": (C.c_int, [C.POINTER(pbn_model_desc), C.c_char_p, C.c_size_t]),
    "pbn_load": (C.c_int, [C.POINTER(pbn_model_desc), C.c_int, C.POINTER(C.c_void_p), C.c_char_p,
                           C.c_size_t]),
    "pbn_free": (None, [C.c_void_p]),
    "pbn_get_model_info": (C.c_int, [C.c_void_p, C.POINTER(pbn_model_info)]),
    "pbn_simulate": (C.c_int, [C.c_void_p, C.POINTER(pbn_sim_args), C.POINTER(pbn_sim_out), C.c_void_p]),
    "pbn_simulate_workspace_size": (C.c_int, [C.c_void_p, C.POINTER(pbn_sim_args), C.POINTER(C.c_int64)]),
    "pbn_recount": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p]),
    "pbn_gelman_rubin": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "pbn_two_state": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                C.c_double, C.c_double, C.POINTER(pbn_two_state_result)]),
    "pbn_inv_norm_cdf": (C.c_double, [C.c_double]),
    "pbn_t_quantile": (C.c_double, [C.c_double, C.c_double]),
    "pbn_skart_ci_from_batches": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                            C.POINTER(pbn_skart_ci)]),
    "pbn_skart": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                            C.POINTER(pbn_skart_result), C.c_void_p]),
    "pbn_run": (C.c_int, [C.c_void_p, C.POINTER(pbn_run_args), C.POINTER(pbn_run_result), C.c_void_p,
                          C.c_char_p, C.c_size_t]),
    "pbn_run_multi": (C.c_int, [C.c_void_p, C.POINTER(pbn_run_args), C.c_void_p, C.c_int32,
                                C.POINTER(pbn_run_result), C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t]),
    "pbn_run_sharded": (C.c_int, [C.c_void_p, C.POINTER(pbn_run_args), C.c_int64, C.c_int64, C.c_void_p,
                                  C.c_void_p, C.POINTER(pbn_run_result), C.c_void_p, C.c_char_p, C.c_size_t]),
    "pbn_version": (C.c_char_p, []),
    "pbn_last_kernel": (C.c_char_p, []),
}

# int (*)(uint64_t* values, int32_t count, void* ctx): in-place sum over shards
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_uint64), C.c_int32, C.c_void_p)

_lib = None


def lib():
    """Load libpbnsim.so (built by __graft_entry__.build()).  Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libpbnsim.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, err: bytes | None = None):
    if status != PBN_OK:
        raise PbnError(status, (err or b"").split(b"\0", 1)[0].decode(errors="replace"))


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))
