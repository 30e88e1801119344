"""B200-native PISA (Piecewise Sparse Attention, arXiv 2602.01077) forward.

The product is the C-ABI library lib/libpisa_b200.so (include/pisa_b200.h),
built from csrc/ for sm_100a. This package is the Python host mirror of the
reference's operator interface (``pisa::`` in /root/reference/proj/include).
"""
from .pisa import (  # noqa: F401
    AccumDtype, AttentionConfig, BlockDivisibility, BlockStatistics, Context, CudaError,
    DegenerateScale, EmptySelection, Error, ErrorKind, InvalidDimension, InvalidEpsilon,
    InvalidSparsity, MultiheadResult, NumericalOverflow, PisaOutput, PisaVariant,
    RouterOptions, RouterStrategy, SelectionPlan, SparsityResolution, TensorBundle,
    Unsupported, compute_prepare, fwd, fwd_host, kernel_names, make_desc, pisa_attention,
    pisa_multihead, pisa_reference, pisa_streaming, resolve, select_topk_plain, selftest_mma,
    block_norms, select_topk_covariance, BadMagic, IoError, IoFailure, MalformedFile,
    NonFiniteValue, UnsupportedDtype, UnsupportedVersion,
    sparsity_to_k, variant_name, dense_online,
)

from . import dit  # noqa: F401,E402  (DiT integration surface: warmup policy, joint attention)
from .dit import PRESETS, PisaAttention, WarmupPolicy  # noqa: F401,E402
from . import pqkv  # noqa: F401,E402  (PQKV tensor files, io.hpp)
from . import analysis  # noqa: F401,E402  (theory checks on GPU outputs, analysis.hpp)
from .generate import gen_clustered, gen_gaussian  # noqa: F401,E402  (generate.hpp fixtures)

__all__ = [n for n in dir() if not n.startswith("_")]
