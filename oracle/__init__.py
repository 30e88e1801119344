"""ctypes bindings for the CPU checker (TEST INFRASTRUCTURE ONLY).

Two libraries live here:
  * ``liboracle.so``            -- the restatement (oracle/pisa_oracle.cpp)
  * ``_ref/libpisa_ref*.so``    -- the unmodified reference, compiled from
                                   /root/reference by oracle/Makefile

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import this
package. The product package (paper_2602_01077_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64 = C.c_int64


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return " avx512f " in f.read()
    except OSError:
        return False


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.oracle_rng_u64.argtypes = [C.c_uint64, _u64p, i64]
        L.oracle_rng_gaussian.argtypes = [C.c_uint64, _f64p, i64]
        L.oracle_gen_gaussian.argtypes = [C.c_uint64, i64, i64, i64, C.c_double, _f32p, _f32p, _f32p]
        L.oracle_gen_gaussian_head.argtypes = [C.c_uint64, i64, i64, i64, C.c_double, i64, i64, _f32p,
                                               _f32p, _f32p]
        L.oracle_gen_clustered.argtypes = [C.c_uint64, i64, i64, i64, i64, C.c_double, C.c_double,
                                           _f32p, _f32p, _f32p]
        L.oracle_round_bf16.argtypes = [_f32p, i64]
        L.oracle_sparsity_to_k.argtypes = [C.c_double, i64, C.POINTER(i64), C.POINTER(C.c_double)]
        L.oracle_block_stats.argtypes = [_f32p, _f32p, i64, i64, i64, _f64p, _f64p, _f64p, _f64p]
        L.oracle_query_means.argtypes = [_f32p, i64, i64, i64, _f64p]
        L.oracle_select_plain.argtypes = [_f64p, _f64p, i64, i64, i64, i64, C.c_double, C.c_int,
                                          _i32p, C.c_void_p]
        L.oracle_select_cov.argtypes = [_f64p, _f64p, _f64p, i64, i64, i64, i64, C.c_double,
                                        C.c_double, C.c_int, _i32p, C.c_void_p]
        L.oracle_select_rowmax.argtypes = [_f32p, _f64p, C.c_void_p, i64, i64, i64, i64, i64,
                                           C.c_double, C.c_double, _i32p, C.c_void_p]
        L.oracle_block_norms.argtypes = [_f32p, _f32p, i64, i64, i64, _f64p, C.c_void_p, C.c_int]
        L.oracle_pisa_attention.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, _i32p, i64, _f64p,
                                            _f64p, _f64p, _f64p, C.c_double, C.c_int, C.c_int,
                                            i64, i64, C.c_int, _f64p, _f64p, _f64p, _f64p]
        L.oracle_dense.argtypes = [_f32p, _f32p, _f32p, i64, i64, C.c_double, i64, i64, C.c_int,
                                   _f64p]
        L.oracle_multihead.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, i64, C.c_double, i64,
                                       C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _f64p,
                                       _i32p, _f64p, _f64p, _f64p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libpisa_ref.so"))


def ref():
    """The unmodified reference library (AVX-512 build when the host has it)."""
    global _ref
    if _ref is None:
        name = "libpisa_ref_v4.so" if _cpu_has_avx512() else "libpisa_ref.so"
        path = os.path.join(HERE, "_ref", name)
        if not os.path.exists(path):
            path = os.path.join(HERE, "_ref", "libpisa_ref.so")
        R = C.CDLL(path)
        R.ref_rng_u64.argtypes = [C.c_uint64, _u64p, i64]
        R.ref_rng_gaussian.argtypes = [C.c_uint64, _f64p, i64]
        R.ref_gen.argtypes = [C.c_int, C.c_uint64, i64, i64, i64, C.c_double, i64, C.c_double,
                              C.c_double, _f32p, _f32p, _f32p]
        R.ref_sparsity_to_k.argtypes = [C.c_double, i64, C.POINTER(i64), C.POINTER(C.c_double)]
        R.ref_block_stats.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, _f64p, _f64p, _f64p,
                                      _f64p, _f64p]
        R.ref_select_plain.argtypes = [_f64p, _f64p, i64, i64, i64, i64, C.c_double, C.c_int, _i32p]
        R.ref_block_norms.argtypes = [_f32p, _f32p, i64, i64, i64, _f64p, C.c_void_p]
        R.ref_select_cov.argtypes = [_f64p, _f64p, _f64p, i64, i64, i64, i64, C.c_double, C.c_double,
                                     C.c_int, _i32p]
        R.ref_select_rowmax.argtypes = [_f32p, _f64p, C.c_void_p, i64, i64, i64, i64, i64, C.c_double,
                                        C.c_double, _i32p]
        R.ref_pqkv_write.argtypes = [C.c_char_p, C.c_int, _f64p, _f64p, _f64p, i64, i64, i64,
                                     C.POINTER(i64)]
        R.ref_pqkv_read.argtypes = [C.c_char_p, C.POINTER(i64), C.c_void_p, i64, C.c_char_p, i64]
        R.ref_flop_model.argtypes = [i64, i64, i64, i64, C.c_int, _f64p]
        R.ref_theorem1.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, i64, _i32p, _f64p, _f64p]
        R.ref_multihead.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, C.c_double, C.c_int,
                                    C.c_int, i64, i64, C.c_double, C.c_int, C.c_int, C.c_int,
                                    C.c_uint, _f32p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        R.ref_bench_sample.argtypes = [_f32p, _f32p, _f32p, i64, i64, C.c_double, i64, i64,
                                       C.c_uint, _f32p, _f64p]
        R.ref_dense_online.argtypes = [_f32p, _f32p, _f32p, i64, i64, C.c_int, C.c_uint, _f32p]
        R.ref_head_parity.argtypes = [_f32p, _f32p, _f32p, i64, i64, C.c_double, C.c_int, i64,
                                      C.c_void_p, C.c_void_p, C.c_int, C.c_uint, _i32p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
        R._path = path
        _ref = R
    return _ref


# ----------------------------------------------------------------- helpers --
class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: status {status}")
        self.status = status


def _check(st: int, where: str) -> None:
    if st != 0:
        raise OracleError(st, where)


def round_bf16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32).copy()
    lib().oracle_round_bf16(x, x.size)
    return x


def gen(kind: str, seed: int, heads: int, L: int, d: int, std: float = 1.0, clusters: int = 16,
        concentration: float = 2.0, noise_std: float = 0.15, bf16: bool = True):
    """Synthetic Q/K/V exactly as the reference generates them ([H][L][d] float32),
    optionally rounded to bf16 (RNE) so the GPU and the oracle see the same values."""
    n = heads * L * d
    q = np.empty(n, np.float32)
    k = np.empty(n, np.float32)
    v = np.empty(n, np.float32)
    if kind == "gaussian":
        _check(lib().oracle_gen_gaussian(seed, heads, L, d, std, q, k, v), "gen_gaussian")
    else:
        _check(lib().oracle_gen_clustered(seed, heads, L, d, clusters, concentration, noise_std,
                                          q, k, v), "gen_clustered")
    out = [a.reshape(heads, L, d) for a in (q, k, v)]
    if bf16:
        out = [round_bf16(a) for a in out]
    return out


def gen_gaussian_head(seed: int, heads: int, L: int, d: int, head: int, rows: int | None = None,
                      std: float = 1.0, bf16: bool = True):
    """Rows [0, rows) of head `head` of gen_gaussian(seed, heads, L, d, std), without
    generating the other heads ([rows][d] float32 q, k, v; bf16-rounded by default)."""
    rows = L if rows is None else rows
    out = [np.empty((rows, d), np.float32) for _ in range(3)]
    _check(lib().oracle_gen_gaussian_head(seed, heads, L, d, std, head, rows, *out), "gen_gaussian_head")
    return [round_bf16(x) for x in out] if bf16 else out


def sparsity_to_k(r: float, n: int):
    k = i64()
    real = C.c_double()
    _check(lib().oracle_sparsity_to_k(r, n, C.byref(k), C.byref(real)), "sparsity_to_k")
    return k.value, real.value


def block_stats(k: np.ndarray, v: np.ndarray, B: int = 64):
    L, d = k.shape
    N = (L + B - 1) // B
    kb = np.empty((N, d)); vh = np.empty((N, d)); hb = np.empty((d, d)); kg = np.empty(d)
    _check(lib().oracle_block_stats(np.ascontiguousarray(k, np.float32),
                                    np.ascontiguousarray(v, np.float32), L, d, B, kb, vh, hb, kg),
           "block_stats")
    return kb, vh, hb, kg


def query_means(q: np.ndarray, B: int = 64):
    L, d = q.shape
    N = (L + B - 1) // B
    qb = np.empty((N, d))
    _check(lib().oracle_query_means(np.ascontiguousarray(q, np.float32), L, d, B, qb), "query_means")
    return qb


def select_plain(qbar, kbar, k: int, scale: float, force_diagonal: bool = False,
                 return_scores: bool = False):
    nq, d = qbar.shape
    n = kbar.shape[0]
    sel = np.empty((nq, k), np.int32)
    scores = np.empty((nq, n)) if return_scores else None
    _check(lib().oracle_select_plain(np.ascontiguousarray(qbar), np.ascontiguousarray(kbar), nq, n,
                                     d, k, scale, int(force_diagonal), sel,
                                     scores.ctypes.data if scores is not None else None),
           "select_plain")
    return (sel, scores) if return_scores else sel


def block_norms(k: np.ndarray, v: np.ndarray, B: int = 64, threads: int = 0):
    """M_j = ||H_j - H_bar||_2 per key block (compute_global_stats with norms,
    block_stats.hpp:207-241; Jacobi spectral norm, :42-94). Ragged-aware."""
    L, d = k.shape
    N = (L + B - 1) // B
    m = np.empty(N)
    _check(lib().oracle_block_norms(np.ascontiguousarray(k, np.float32),
                                    np.ascontiguousarray(v, np.float32), L, d, B, m, None, threads),
           "block_norms")
    return m


def select_cov(qbar, kbar, m, k: int, scale: float, eps: float = 1e-6, force_diagonal=False,
               return_scores: bool = False):
    """select_topk_covariance (router.hpp:157-193)."""
    nq, d = qbar.shape
    n = kbar.shape[0]
    sel = np.empty((nq, k), np.int32)
    scores = np.empty((nq, n)) if return_scores else None
    _check(lib().oracle_select_cov(np.ascontiguousarray(qbar), np.ascontiguousarray(kbar),
                                   np.ascontiguousarray(m, np.float64), nq, n, d, k, scale, eps,
                                   int(force_diagonal), sel,
                                   scores.ctypes.data if scores is not None else None),
           "select_cov")
    return (sel, scores) if return_scores else sel


def select_rowmax(q, kbar, k: int, scale: float, m=None, eps: float = 1e-6, B: int = 64,
                  return_scores: bool = False):
    """select_topk_rowmax (router.hpp:198-233); m = None for the plain score."""
    L, d = q.shape
    n = kbar.shape[0]
    nq = (L + B - 1) // B
    sel = np.empty((nq, k), np.int32)
    scores = np.empty((nq, n)) if return_scores else None
    mm = None if m is None else np.ascontiguousarray(m, np.float64)
    _check(lib().oracle_select_rowmax(np.ascontiguousarray(q, np.float32), np.ascontiguousarray(kbar),
                                      mm.ctypes.data if mm is not None else None, L, n, d, B, k,
                                      scale, eps, sel,
                                      scores.ctypes.data if scores is not None else None),
           "select_rowmax")
    return (sel, scores) if return_scores else sel


VARIANTS = {"sparse_only": 0, "zeroth": 1, "block_first": 2, "hybrid": 3, "global_centroid": 4}


def pisa_attention(q, k, v, selected, stats, scale: float, variant="hybrid", literal_phase3=False,
                   qb0: int = 0, qb1: int | None = None, B: int = 64, threads: int = 0):
    L, d = q.shape
    N = (L + B - 1) // B
    qb1 = N if qb1 is None else qb1
    kb, vh, hb, kg = stats
    out = np.zeros((L, d)); m = np.zeros(L); ell = np.zeros(L); et = np.zeros(L)
    sel = np.ascontiguousarray(selected, np.int32)
    _check(lib().oracle_pisa_attention(np.ascontiguousarray(q, np.float32),
                                       np.ascontiguousarray(k, np.float32),
                                       np.ascontiguousarray(v, np.float32), L, d, B, sel,
                                       sel.shape[1], kb, vh, hb, kg, scale,
                                       VARIANTS[variant], int(literal_phase3), qb0, qb1, threads,
                                       out, m, ell, et), "pisa_attention")
    return out, m, ell, et


def dense(q, k, v, scale: float, r0: int = 0, r1: int | None = None, threads: int = 0):
    L, d = q.shape
    r1 = L if r1 is None else r1
    out = np.zeros((L, d))
    _check(lib().oracle_dense(np.ascontiguousarray(q, np.float32), np.ascontiguousarray(k, np.float32),
                              np.ascontiguousarray(v, np.float32), L, d, scale, r0, r1, threads, out),
           "dense")
    return out


def multihead(q, k, v, r: float = 0.875, ksel: int = 0, variant="hybrid", force_diagonal=False,
              scale: float = 0.0, literal_phase3=False, B: int = 64, threads: int = 0):
    H, L, d = q.shape
    N = (L + B - 1) // B
    kk = ksel if ksel > 0 else sparsity_to_k(r, N)[0]
    out = np.zeros((H, L, d)); sel = np.zeros((H, N, kk), np.int32)
    m = np.zeros((H, L)); ell = np.zeros((H, L)); et = np.zeros((H, L))
    _check(lib().oracle_multihead(np.ascontiguousarray(q, np.float32),
                                  np.ascontiguousarray(k, np.float32),
                                  np.ascontiguousarray(v, np.float32), H, L, d, B, r, kk,
                                  VARIANTS[variant], int(force_diagonal), scale,
                                  int(literal_phase3), threads, out, sel, m, ell, et), "multihead")
    return dict(out=out, selected=sel, row_max=m, ell=ell, ell_tail=et, k=kk)


# ------------------------------------------------------ reference wrappers --
def ref_gen(kind: str, seed: int, heads: int, L: int, d: int, std=1.0, clusters=16,
            concentration=2.0, noise_std=0.15):
    n = heads * L * d
    q = np.empty(n, np.float32); k = np.empty(n, np.float32); v = np.empty(n, np.float32)
    _check(ref().ref_gen(int(kind == "clustered"), seed, heads, L, d, std, clusters, concentration,
                         noise_std, q, k, v), "ref_gen")
    return [a.reshape(heads, L, d) for a in (q, k, v)]


def ref_block_stats(q, k, v, B: int = 64):
    L, d = k.shape
    N = L // B
    kb = np.empty((N, d)); vh = np.empty((N, d)); hb = np.empty((d, d)); qb = np.empty((N, d))
    kg = np.empty(d)
    _check(ref().ref_block_stats(np.ascontiguousarray(q, np.float32),
                                 np.ascontiguousarray(k, np.float32),
                                 np.ascontiguousarray(v, np.float32), L, d, B, kb, vh, hb, qb, kg),
           "ref_block_stats")
    return kb, vh, hb, qb, kg


def ref_select_plain(qbar, kbar, k: int, scale: float, force_diagonal=False):
    nq, d = qbar.shape
    sel = np.empty((nq, k), np.int32)
    _check(ref().ref_select_plain(np.ascontiguousarray(qbar), np.ascontiguousarray(kbar), nq,
                                  kbar.shape[0], d, k, scale, int(force_diagonal), sel),
           "ref_select_plain")
    return sel


def ref_block_norms(k, v, B: int = 64):
    L, d = k.shape
    m = np.empty(L // B)
    _check(ref().ref_block_norms(np.ascontiguousarray(k, np.float32),
                                 np.ascontiguousarray(v, np.float32), L, d, B, m, None),
           "ref_block_norms")
    return m


def ref_select_cov(qbar, kbar, m, k: int, scale: float, eps=1e-6, force_diagonal=False):
    nq, d = qbar.shape
    sel = np.empty((nq, k), np.int32)
    _check(ref().ref_select_cov(np.ascontiguousarray(qbar), np.ascontiguousarray(kbar),
                                np.ascontiguousarray(m, np.float64), nq, kbar.shape[0], d, k, scale,
                                eps, int(force_diagonal), sel), "ref_select_cov")
    return sel


def ref_select_rowmax(q, kbar, k: int, scale: float, m=None, eps=1e-6, B: int = 64):
    L, d = q.shape
    sel = np.empty((L // B, k), np.int32)
    mm = None if m is None else np.ascontiguousarray(m, np.float64)
    _check(ref().ref_select_rowmax(np.ascontiguousarray(q, np.float32), np.ascontiguousarray(kbar),
                                   mm.ctypes.data if mm is not None else None, L, kbar.shape[0], d,
                                   B, k, scale, eps, sel), "ref_select_rowmax")
    return sel


def ref_pqkv_write(path: str, q, k, v, dtype: str = "f32") -> int:
    """The reference's write_bundle_file (io.hpp:102-126) on [H][L][d] arrays."""
    H, L, d = q.shape
    nb = i64()
    _check(ref().ref_pqkv_write(path.encode(), 1 if dtype == "f32" else 2,
                                *(np.ascontiguousarray(x, np.float64) for x in (q, k, v)), H, L, d,
                                C.byref(nb)), "ref_pqkv_write")
    return nb.value


def ref_pqkv_read(path: str):
    """The reference's read_bundle_file (io.hpp:180-221): (q, k, v, dtype_tag) or
    raises OracleError whose message starts with the reference error class."""
    sd = (i64 * 4)()
    err = C.create_string_buffer(512)
    st = ref().ref_pqkv_read(path.encode(), sd, None, 0, err, 512)
    if st != 0:
        e = OracleError(st, err.value.decode())
        e.message = err.value.decode()
        raise e
    H, L, d, tag = (int(x) for x in sd)
    buf = np.empty(3 * H * L * d)
    st = ref().ref_pqkv_read(path.encode(), sd, buf.ctypes.data, buf.size, err, 512)
    _check(st, "ref_pqkv_read")
    buf = buf.reshape(3, H, L, d)
    return buf[0], buf[1], buf[2], tag


def ref_flop_model(L, d, b, k, variant="hybrid"):
    out = np.empty(6)
    _check(ref().ref_flop_model(L, d, b, k, VARIANTS[variant], out), "ref_flop_model")
    return dict(zip(["dense_flops", "sparse_flops", "pisa_flops", "sparse_ratio", "pisa_ratio",
                     "overhead_ratio"], out.tolist()))


def ref_theorem1(q, k, v, ksel: int, B: int = 64):
    """The reference's theorem1_check + jensen_check (analysis.hpp:86-223) for one
    head (Plain router, norms by the exact solver): dict with the plan, per-row
    arrays and the report scalars."""
    L, d = q.shape
    N = L // B
    plan = np.empty((N, ksel), np.int32)
    rows = np.empty((5, L))
    scal = np.empty(6)
    _check(ref().ref_theorem1(*(np.ascontiguousarray(x, np.float32) for x in (q, k, v)), L, d, B, ksel,
                              plan, rows, scal), "ref_theorem1")
    return dict(plan=plan, actual_err=rows[0], bound=rows[1], rho=rows[2], alpha_sum=rows[3],
                jensen_rhs=rows[4], c_q=scal[0], m_max=scal[1], violations=int(scal[2]),
                jensen_violations=int(scal[3]), max_slack_ratio=scal[4], jensen_check=int(scal[5]))


def ref_head_parity(q, k, v, r: float, blocks=(), force_diagonal=False, accum_f64=True, threads=0,
                    B: int = 64, sub_plan=None):
    """One head through the reference's own pipeline (engine.hpp:437-461): the full
    plan [N][k], the fp64 q_bar / k_bar [N][d], and pisa_streaming's output rows
    of the query blocks `blocks` ([len(blocks)*B][d] float32; None without
    blocks). `sub_plan` ([len(blocks)][k]) replaces the reference's plan rows of
    those blocks in the streaming step (e.g. the GPU's plan). L % 64 == 0."""
    L, d = q.shape
    N = L // B
    kk, _ = sparsity_to_k(r, N)
    sel = np.empty((N, kk), np.int32)
    qb = np.empty((N, d)); kb = np.empty((N, d))
    blk = np.ascontiguousarray(np.asarray(blocks, np.int64))
    sp = None if sub_plan is None else np.ascontiguousarray(sub_plan, np.int32)
    out = np.empty((max(1, len(blk)) * B, d), np.float32)
    _check(ref().ref_head_parity(np.ascontiguousarray(q, np.float32), np.ascontiguousarray(k, np.float32),
                                 np.ascontiguousarray(v, np.float32), L, d, r, int(force_diagonal), len(blk),
                                 blk.ctypes.data, None if sp is None else sp.ctypes.data, int(accum_f64),
                                 threads, sel, qb.ctypes.data, kb.ctypes.data, out.ctypes.data), "ref_head_parity")
    return sel, qb, kb, (out[:len(blk) * B] if len(blk) else None)


def ref_multihead(q, k, v, r=0.875, variant="hybrid", force_diagonal=False, B=64, group=8,
                  scale=0.0, accum_f64=True, streaming=True, literal_phase3=False, threads=0,
                  router="plain", row_level=False):
    """pisa_multihead of the unmodified reference; router "plain" | "covariance"
    (RouterOptions, engine.hpp:385-390, epsilon 1e-6)."""
    H, L, d = q.shape
    N = L // B
    kk, _ = sparsity_to_k(r, N)
    out = np.zeros((H, L, d), np.float32)
    sel = np.zeros((H, N, kk), np.int32)
    denom = np.zeros((H, L)); tm = np.zeros((H, L)); et = np.zeros((H, L)); rm = np.zeros((H, L))
    times = np.zeros(3)
    kout = i64()
    _check(ref().ref_multihead(np.ascontiguousarray(q, np.float32),
                               np.ascontiguousarray(k, np.float32),
                               np.ascontiguousarray(v, np.float32), H, L, d, r, VARIANTS[variant],
                               int(force_diagonal) | (2 if router == "covariance" else 0)
                               | (4 if row_level else 0), B, group, scale, int(accum_f64),
                               int(streaming), int(literal_phase3), threads, out,
                               sel.ctypes.data, denom.ctypes.data, tm.ctypes.data, et.ctypes.data,
                               rm.ctypes.data, times.ctypes.data, C.byref(kout)), "ref_multihead")
    return dict(out=out, selected=sel, denom=denom, tail_mass=tm, ell_tail=et, row_max=rm,
                times_ms=times, k=kout.value)
