"""ctypes binding of include/pisa_b200.h (lib/libpisa_b200.so).

Loads the in-tree library and fails loudly when it is missing: there is no CPU
or eager fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libpisa_b200.so")

i64 = C.c_int64


class AttnDesc(C.Structure):
    _fields_ = [
        ("batch", i64), ("heads", i64), ("seq_len", i64), ("head_dim", i64),
        ("q_strides", i64 * 3), ("k_strides", i64 * 3), ("v_strides", i64 * 3),
        ("o_strides", i64 * 3),
        ("block_size", C.c_int32), ("group_size", C.c_int32),
        ("scale", C.c_double), ("sparsity", C.c_double), ("topk", i64),
        ("variant", C.c_int32), ("router", C.c_int32), ("force_diagonal", C.c_int32),
        ("literal_phase3", C.c_int32), ("ragged", C.c_int32), ("out_dtype", C.c_int32),
        ("check_finite", C.c_int32), ("row_level", C.c_int32), ("epsilon", C.c_double),
    ]


class Diag(C.Structure):
    _fields_ = [("row_max", C.c_void_p), ("ell", C.c_void_p), ("ell_tail", C.c_void_p),
                ("selected", C.c_void_p)]


# every symbol include/pisa_b200.h declares (tests check they are exported)
EXPORTED = [
    "pisa_b200_create", "pisa_b200_destroy", "pisa_b200_last_error", "pisa_b200_abi_version",
    "pisa_b200_sparsity_to_k", "pisa_b200_resolve", "pisa_b200_fwd", "pisa_b200_fwd_host",
    "pisa_b200_fwd_qrange", "pisa_b200_set_pairing", "pisa_b200_block_stats", "pisa_b200_select", "pisa_b200_block_norms",
    "pisa_b200_select_cov", "pisa_b200_attention",
    "pisa_b200_last_launch_count", "pisa_b200_kernel_name", "pisa_b200_selftest_mma",
    "pisa_b200_set_profiling", "pisa_b200_read_profile", "pisa_b200_fused_tiles",
    "pisa_b200_debug_trace", "pisa_b200_block_stats_host", "pisa_b200_block_norms_host",
    "pisa_b200_select_host", "pisa_b200_attention_host", "pisa_b200_gen_gaussian",
    "pisa_b200_gen_clustered",
]

_lib = None


def load(build_if_missing: bool = False):
    """Returns the loaded C-ABI library; raises if the sm_100a build is absent.
    PISA_B200_LIB overrides the path (e.g. the PISA_TRACE debug build)."""
    global _lib, LIB_PATH
    if _lib is not None:
        return _lib
    LIB_PATH = os.environ.get("PISA_B200_LIB", LIB_PATH)
    if not os.path.exists(LIB_PATH):
        if build_if_missing:
            from . import build as _b
            _b.build()
        else:
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -m paper_2602_01077_b200.build` "
                "(the CUDA extension is required; there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.pisa_b200_create.argtypes = [C.POINTER(vp), C.c_int]
    L.pisa_b200_destroy.argtypes = [vp]
    L.pisa_b200_destroy.restype = None
    L.pisa_b200_last_error.argtypes = [vp]
    L.pisa_b200_last_error.restype = C.c_char_p
    L.pisa_b200_abi_version.restype = C.c_int
    L.pisa_b200_sparsity_to_k.argtypes = [C.c_double, i64, C.POINTER(i64), C.POINTER(C.c_double)]
    L.pisa_b200_resolve.argtypes = [C.POINTER(AttnDesc), C.POINTER(i64), C.POINTER(i64),
                                    C.POINTER(C.c_double)]
    L.pisa_b200_fwd.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, C.POINTER(Diag), vp]
    L.pisa_b200_fwd_host.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, C.POINTER(Diag)]
    L.pisa_b200_fwd_qrange.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, i64, i64, C.POINTER(Diag), vp]
    L.pisa_b200_set_pairing.argtypes = [vp, C.c_int]
    L.pisa_b200_block_stats.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp, vp, vp]
    L.pisa_b200_select.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, vp]
    L.pisa_b200_block_norms.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, vp]
    L.pisa_b200_select_cov.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp]
    L.pisa_b200_attention.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp, vp, vp,
                                      C.POINTER(Diag), vp]
    L.pisa_b200_last_launch_count.argtypes = [vp]
    L.pisa_b200_last_launch_count.restype = i64
    L.pisa_b200_kernel_name.argtypes = [C.c_int]
    L.pisa_b200_kernel_name.restype = C.c_char_p
    L.pisa_b200_selftest_mma.argtypes = [vp, vp, vp, vp, vp]
    L.pisa_b200_set_profiling.argtypes = [vp, C.c_int]
    L.pisa_b200_debug_trace.argtypes = [vp, vp, C.c_int]
    L.pisa_b200_debug_trace.restype = C.c_int
    L.pisa_b200_read_profile.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(i64)]
    L.pisa_b200_fused_tiles.argtypes = [vp, C.POINTER(i64)]
    L.pisa_b200_fused_tiles.restype = C.c_int
    L.pisa_b200_block_stats_host.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp, vp]
    L.pisa_b200_block_norms_host.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp]
    L.pisa_b200_select_host.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp]
    L.pisa_b200_attention_host.argtypes = [vp, C.POINTER(AttnDesc), vp, vp, vp, vp, vp, vp, vp, vp,
                                           C.POINTER(Diag)]
    L.pisa_b200_gen_gaussian.argtypes = [C.c_uint64, i64, i64, i64, C.c_double, C.c_int32, vp, vp, vp,
                                         C.c_int]
    L.pisa_b200_gen_clustered.argtypes = [C.c_uint64, i64, i64, i64, i64, C.c_double, C.c_double,
                                          C.c_int32, vp, vp, vp, C.c_int]
    for name in ("pisa_b200_block_stats_host", "pisa_b200_block_norms_host", "pisa_b200_select_host",
                 "pisa_b200_attention_host", "pisa_b200_gen_gaussian", "pisa_b200_gen_clustered",
                 "pisa_b200_set_profiling", "pisa_b200_read_profile", "pisa_b200_create", "pisa_b200_sparsity_to_k", "pisa_b200_resolve",
                 "pisa_b200_fwd", "pisa_b200_fwd_host", "pisa_b200_fwd_qrange", "pisa_b200_set_pairing",
                 "pisa_b200_block_stats", "pisa_b200_select", "pisa_b200_block_norms", "pisa_b200_select_cov",
                 "pisa_b200_attention", "pisa_b200_selftest_mma"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L
