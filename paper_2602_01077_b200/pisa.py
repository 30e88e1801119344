"""Host-side mirror of the reference operator interface (namespace ``pisa``),
backed by the sm_100a C ABI. Names, argument meaning and error classes follow
/root/reference/proj/include/pisa/*.hpp so callers read like the reference:

    res = pisa_multihead(bundle, r, RouterOptions(), PisaVariant.Hybrid, cfg, True)

Tensors are torch CUDA tensors (bf16). PyTorch provides device memory and the
current stream only; every computation runs in the library's own kernels.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import torch

from . import _abi

# ------------------------------------------------------------------- enums --


class PisaVariant(enum.IntEnum):  # engine.hpp:30
    SparseOnly = 0
    Zeroth = 1
    BlockFirst = 2
    Hybrid = 3
    GlobalCentroid = 4


class RouterStrategy(enum.IntEnum):  # router.hpp:16
    Plain = 0
    CovarianceAware = 1


class AccumDtype(enum.IntEnum):  # attention.hpp:17
    F32 = 0
    F64 = 1


def variant_name(v: PisaVariant) -> str:  # engine.hpp:32-41
    return {0: "sparse_only", 1: "zeroth", 2: "block_first", 3: "hybrid",
            4: "global_centroid"}[int(v)]


# ------------------------------------------------------------------ errors --
class ErrorKind(enum.IntEnum):  # errors.hpp:10
    Validation = 0
    Invariant = 1
    Io = 2


class Error(RuntimeError):  # errors.hpp:12-20
    kind = ErrorKind.Validation


class InvalidDimension(Error):
    pass


class DegenerateScale(InvalidDimension):
    pass


class BlockDivisibility(Error):
    pass


class InvalidSparsity(Error):
    pass


class InvalidEpsilon(Error):
    pass


class EmptySelection(Error):
    pass


class NumericalOverflow(Error):
    kind = ErrorKind.Invariant


class Unsupported(Error):
    """No reference class: the request is outside the GPU path (e.g. BlockFirst)."""


class CudaError(Error):
    kind = ErrorKind.Invariant


class IoFailure(Error):  # base of the PQKV / file errors (errors.hpp:52-80, ErrorKind::Io)
    kind = ErrorKind.Io


class BadMagic(IoFailure):
    pass


class UnsupportedVersion(IoFailure):
    pass


class UnsupportedDtype(IoFailure):
    pass


class MalformedFile(IoFailure):
    pass


class NonFiniteValue(IoFailure):
    pass


class IoError(IoFailure):
    pass


_STATUS = {1: InvalidDimension, 2: BlockDivisibility, 3: InvalidSparsity, 4: InvalidEpsilon,
           5: EmptySelection, 6: NumericalOverflow, 7: DegenerateScale, 8: Unsupported,
           9: CudaError}


def _raise(status: int, ctx=None, where: str = "") -> None:
    if status == 0:
        return
    msg = ""
    if ctx is not None:
        msg = _abi.load().pisa_b200_last_error(ctx).decode()
    raise _STATUS.get(status, Error)(msg or f"{where}: status {status}")


# ------------------------------------------------------------------ config --
@dataclass
class AttentionConfig:  # attention.hpp:19-49
    block_size: int = 64
    group_size: int = 8
    scale: float = 0.0
    accum: AccumDtype = AccumDtype.F64
    deterministic: bool = True
    num_threads: int = 0
    literal_phase3: bool = False
    collect_phase_times: bool = False

    def resolved_scale(self, d: int) -> float:
        return self.scale if self.scale > 0.0 else 1.0 / math.sqrt(d)

    def check(self, L: int, ragged: bool = False) -> None:
        if self.block_size == 0 or self.group_size == 0:
            raise InvalidDimension("InvalidDimension: block_size and group_size must be >= 1")
        if not ragged and L % self.block_size != 0:
            raise BlockDivisibility(
                f"BlockDivisibility: seq_len {L} not divisible by block size {self.block_size}")


@dataclass
class RouterOptions:  # engine.hpp:385-390
    strategy: RouterStrategy = RouterStrategy.Plain
    epsilon: float = 1e-6
    force_diagonal: bool = False
    row_level: bool = False


@dataclass
class SparsityResolution:  # router.hpp:73-76
    k: int
    realized: float


def sparsity_to_k(r: float, n: int) -> SparsityResolution:  # router.hpp:80-90
    k = _abi.i64()
    real = C.c_double()
    _raise(_abi.load().pisa_b200_sparsity_to_k(float(r), int(n), C.byref(k), C.byref(real)),
           where="sparsity_to_k")
    return SparsityResolution(k.value, real.value)


@dataclass
class TensorBundle:  # bundle.hpp:28-51: q/k/v [H][L][d] (here: CUDA bf16 tensors)
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor

    @property
    def num_heads(self) -> int:
        return self.q.shape[0]

    @property
    def seq_len(self) -> int:
        return self.q.shape[1]

    @property
    def head_dim(self) -> int:
        return self.q.shape[2]


@dataclass
class SelectionPlan:  # router.hpp:24-71 (device tensor of ascending lists)
    num_key_blocks: int
    k: int
    selected: torch.Tensor  # int32 [N][k]
    strategy: RouterStrategy = RouterStrategy.Plain
    epsilon: float = 0.0

    def num_query_blocks(self) -> int:
        return self.selected.shape[0]


@dataclass
class PisaOutput:  # engine.hpp:43-57
    output: torch.Tensor
    denom: Optional[torch.Tensor] = None
    tail_mass: Optional[torch.Tensor] = None
    ell_tail: Optional[torch.Tensor] = None
    row_max: Optional[torch.Tensor] = None
    running_max_used: bool = True
    exact_ms: float = 0.0
    approx_ms: float = 0.0
    normalize_ms: float = 0.0


@dataclass
class MultiheadResult:  # engine.hpp:392-403
    heads: List[PisaOutput] = field(default_factory=list)
    plans: List[SelectionPlan] = field(default_factory=list)
    k: int = 0
    num_blocks: int = 0
    sparsity_requested: float = 0.0
    sparsity_realized: float = 0.0
    prepare_ms: float = 0.0
    select_ms: float = 0.0
    attention_ms: float = 0.0


@dataclass
class BlockStatistics:  # block_stats.hpp:21-37 (fp32, device)
    num_blocks: int
    block_size: int
    dim: int
    k_bar: torch.Tensor
    v_hat: torch.Tensor
    h_bar: torch.Tensor
    q_bar: Optional[torch.Tensor] = None
    global_ready: bool = True


# ----------------------------------------------------------------- context --
class Context:
    """Owns one pisa_ctx (device workspace, staging streams) per device."""

    _per_device: dict = {}

    def __init__(self, device: int = 0):
        self.lib = _abi.load()
        h = C.c_void_p()
        st = self.lib.pisa_b200_create(C.byref(h), int(device))
        if st != 0:
            raise CudaError(f"pisa_b200_create(device={device}) failed with status {st}")
        self.handle = h
        self.device = device

    @classmethod
    def get(cls, device: Optional[int] = None) -> "Context":
        if device is None:
            device = torch.cuda.current_device()
        c = cls._per_device.get(device)
        if c is None:
            c = cls._per_device[device] = Context(device)
        return c

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.pisa_b200_destroy(self.handle)
        except Exception:
            pass

    def last_launch_count(self) -> int:
        return int(self.lib.pisa_b200_last_launch_count(self.handle))

    def set_pairing(self, mode: int) -> None:
        """Query-block pairing of the fused kernel: 0 consecutive, 1 auto, 2 always
        overlap-aware (pisa_b200_set_pairing); results do not depend on it."""
        _raise(self.lib.pisa_b200_set_pairing(self.handle, int(mode)), self.handle)

    def set_profiling(self, on: bool) -> None:
        _raise(self.lib.pisa_b200_set_profiling(self.handle, int(on)), self.handle)

    def read_profile(self) -> dict:
        """{kernel_name: (total_ms, launches)} since the last read (syncs on events)."""
        ms = (C.c_double * 8)()
        n = (_abi.i64 * 8)()
        _raise(self.lib.pisa_b200_read_profile(self.handle, ms, n), self.handle)
        names = kernel_names()
        return {names[i]: (ms[i], n[i]) for i in range(len(names)) if n[i] > 0}

    def fused_tiles(self) -> int:
        """64-key tiles the fused kernel processed while profiling (resets)."""
        t = _abi.i64()
        _raise(self.lib.pisa_b200_fused_tiles(self.handle, C.byref(t)), self.handle)
        return t.value


def _strides_bhld(t: torch.Tensor, layout: str):
    """Element strides (b, h, l) of a 4-D tensor in 'bhld' or 'blhd' order."""
    s = t.stride()
    if t.stride(-1) != 1:
        raise InvalidDimension("InvalidDimension: last dim must be contiguous")
    if layout == "bhld":
        return (s[0], s[1], s[2])
    if layout == "blhd":
        return (s[0], s[2], s[1])
    raise InvalidDimension(f"InvalidDimension: unknown layout {layout}")


def make_desc(q, k, v, o, *, layout="bhld", block_size=64, group_size=8, scale=0.0,
              sparsity=0.875, topk=0, variant=PisaVariant.Hybrid,
              router=RouterStrategy.Plain, force_diagonal=False, literal_phase3=False,
              ragged=True, check_finite=False, epsilon=1e-6, row_level=False) -> _abi.AttnDesc:
    if q.dim() != 4:
        raise InvalidDimension("InvalidDimension: expected 4-D tensors")
    if layout == "bhld":
        B, H, L, d = q.shape
    else:
        B, L, H, d = q.shape
    for t in (k, v):
        if tuple(t.shape) != tuple(q.shape):
            raise InvalidDimension(
                f"InvalidDimension: Q {tuple(q.shape)} K {tuple(k.shape)} V {tuple(v.shape)} "
                "do not form an attention instance")
    desc = _abi.AttnDesc()
    desc.batch, desc.heads, desc.seq_len, desc.head_dim = B, H, L, d
    for name, t in (("q_strides", q), ("k_strides", k), ("v_strides", v), ("o_strides", o)):
        getattr(desc, name)[:] = _strides_bhld(t, layout)
    desc.block_size = int(block_size)
    desc.group_size = int(group_size)
    desc.scale = float(scale)
    desc.sparsity = float(sparsity)
    desc.topk = int(topk)
    desc.variant = int(variant)
    desc.router = int(router)
    desc.epsilon = float(epsilon)
    desc.row_level = int(row_level)
    desc.force_diagonal = int(force_diagonal)
    desc.literal_phase3 = int(literal_phase3)
    desc.ragged = int(ragged)
    desc.out_dtype = 1 if o.dtype == torch.float32 else 0
    desc.check_finite = int(check_finite)
    return desc


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_inputs(*ts):
    for t in ts:
        if not t.is_cuda:
            raise InvalidDimension("InvalidDimension: tensors must live on a CUDA device "
                                   "(there is no CPU path)")
        if t.dtype != torch.bfloat16:
            raise Unsupported("Unsupported: q/k/v must be bfloat16")


def _check_out(q, out):
    if tuple(out.shape) != tuple(q.shape):
        raise InvalidDimension(f"InvalidDimension: output shape {tuple(out.shape)} != query shape "
                               f"{tuple(q.shape)}")
    if out.device != q.device:
        raise InvalidDimension("InvalidDimension: output must live on the inputs' device")
    if out.dtype not in (torch.bfloat16, torch.float32):
        raise Unsupported(f"Unsupported: output dtype {out.dtype} (bfloat16 or float32)")


def resolve(desc: _abi.AttnDesc):
    n = _abi.i64()
    k = _abi.i64()
    sc = C.c_double()
    _raise(_abi.load().pisa_b200_resolve(C.byref(desc), C.byref(n), C.byref(k), C.byref(sc)),
           where="resolve")
    return n.value, k.value, sc.value


def fwd(q, k, v, out=None, *, layout="bhld", out_dtype=torch.bfloat16, diagnostics=False,
        return_plan=False, ctx: Optional[Context] = None, q_blocks=None, **kw):
    """The fused forward (pisa_b200_fwd) on 4-D device tensors.

    ``q_blocks=(begin, end)`` restricts the fused step to those query blocks of
    every head (pisa_b200_fwd_qrange; rows outside are left as they are in
    ``out``) -- the unit of (head x query-block range) sharding.
    Returns ``out`` or ``(out, extras)`` where extras holds row_max / ell / ell_tail
    ([B][H][L] fp32) and the plan ([B][H][N][k] int32) when requested."""
    _check_inputs(q, k, v)
    ctx = ctx or Context.get(q.device.index)
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    _check_out(q, out)
    desc = make_desc(q, k, v, out, layout=layout, **kw)
    N, kk, _ = resolve(desc)
    B, H, L = desc.batch, desc.heads, desc.seq_len
    extras = {}
    diag = None
    if diagnostics or return_plan:
        diag = _abi.Diag()
        if diagnostics:
            for nm in ("row_max", "ell", "ell_tail"):
                extras[nm] = torch.empty((B, H, L), dtype=torch.float32, device=q.device)
                setattr(diag, nm, extras[nm].data_ptr())
        if return_plan:
            extras["selected"] = torch.empty((B, H, N, kk), dtype=torch.int32, device=q.device)
            diag.selected = extras["selected"].data_ptr()
    dp = C.byref(diag) if diag is not None else None
    if q_blocks is None:
        st = ctx.lib.pisa_b200_fwd(ctx.handle, C.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(out), dp,
                                   _stream())
    else:
        st = ctx.lib.pisa_b200_fwd_qrange(ctx.handle, C.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                          int(q_blocks[0]), int(q_blocks[1]), dp, _stream())
    _raise(st, ctx.handle)
    return (out, extras) if extras else out


def fwd_host(q, k, v, out, ctx: Optional[Context] = None, device: int = 0, **kw):
    """pisa_b200_fwd_host: Q/K/V/O in (pinned) host memory, dense [B][H][L][d]."""
    ctx = ctx or Context.get(device)
    desc = make_desc(q, k, v, out, layout="bhld", **kw)
    st = ctx.lib.pisa_b200_fwd_host(ctx.handle, C.byref(desc), _ptr(q), _ptr(k), _ptr(v),
                                    _ptr(out), None)
    _raise(st, ctx.handle)
    return out


# ------------------------------------------------- reference step functions --
def _bundle4(x: torch.Tensor) -> torch.Tensor:
    return x.unsqueeze(0) if x.dim() == 3 else x


def compute_prepare(q, k, v, block_size: int = 64, ragged: bool = True) -> BlockStatistics:
    """compute_block_stats + compute_global_stats(norms off) + query_block_means
    (block_stats.hpp:155-278) for [H][L][d] (or [B][H][L][d]) tensors; fp32 outputs."""
    q4, k4, v4 = _bundle4(q), _bundle4(k), _bundle4(v)
    _check_inputs(q4, k4, v4)
    ctx = Context.get(q4.device.index)
    desc = make_desc(q4, k4, v4, q4, block_size=block_size, ragged=ragged, topk=1)
    N, _, _ = resolve(desc)
    B, H, d = desc.batch, desc.heads, desc.head_dim
    dev = q4.device
    kb = torch.empty((B, H, N, d), dtype=torch.float32, device=dev)
    vh = torch.empty_like(kb)
    qb = torch.empty_like(kb)
    hb = torch.empty((B, H, d, d), dtype=torch.float32, device=dev)
    st = ctx.lib.pisa_b200_block_stats(ctx.handle, C.byref(desc), _ptr(q4), _ptr(k4), _ptr(v4),
                                       _ptr(kb), _ptr(vh), _ptr(qb), _ptr(hb), _stream())
    _raise(st, ctx.handle)
    return BlockStatistics(N, block_size, d, kb, vh, hb, qb)


def select_topk_plain(q_bar: torch.Tensor, k_bar: torch.Tensor, k: int, scale: float,
                      force_diagonal: bool = False, return_mask: bool = False):
    """select_topk_plain (router.hpp:126-151) on fp32 device tensors [..][N][d]."""
    q4 = q_bar.reshape(-1, 1, *q_bar.shape[-2:]).contiguous()
    k4 = k_bar.reshape(-1, 1, *k_bar.shape[-2:]).contiguous()
    BH, _, N, d = q4.shape
    if k < 1 or k > N:
        raise InvalidSparsity(f"InvalidSparsity: k must lie in [1, N], got {k} for N = {N}")
    ctx = Context.get(q4.device.index)
    desc = _abi.AttnDesc()
    desc.batch, desc.heads, desc.seq_len, desc.head_dim = BH, 1, N * 64, d
    for nm in ("q_strides", "k_strides", "v_strides", "o_strides"):
        getattr(desc, nm)[:] = (N * 64 * d, N * 64 * d, d)
    desc.block_size, desc.group_size, desc.scale, desc.topk = 64, 8, float(scale), int(k)
    desc.variant, desc.force_diagonal, desc.ragged = 3, int(force_diagonal), 1
    sel = torch.empty((BH, N, k), dtype=torch.int32, device=q4.device)
    W = (N + 31) // 32
    mask = torch.empty((BH, N, W), dtype=torch.int32, device=q4.device)
    st = ctx.lib.pisa_b200_select(ctx.handle, C.byref(desc), _ptr(q4), _ptr(k4), _ptr(sel),
                                  _ptr(mask), _stream())
    _raise(st, ctx.handle)
    sel = sel.reshape(*q_bar.shape[:-2], N, k)
    if return_mask:
        return sel, mask.reshape(*q_bar.shape[:-2], N, W)
    return sel


def block_norms(q, k, v, block_size: int = 64, ragged: bool = True) -> torch.Tensor:
    """M_j = ||H_j - H_bar||_2 per key block (compute_global_stats with
    compute_norms, block_stats.hpp:207-241): fp32 [..][N]. q/k/v [H][L][d] or
    [B][H][L][d] bf16 device tensors."""
    q4, k4, v4 = _bundle4(q), _bundle4(k), _bundle4(v)
    _check_inputs(q4, k4, v4)
    ctx = Context.get(q4.device.index)
    desc = make_desc(q4, k4, v4, q4, block_size=block_size, ragged=ragged)
    B, H, L = desc.batch, desc.heads, desc.seq_len
    N = -(-L // block_size)
    m = torch.empty((B, H, N), dtype=torch.float32, device=q4.device)
    _raise(ctx.lib.pisa_b200_block_norms(ctx.handle, C.byref(desc), _ptr(q4), _ptr(k4), _ptr(v4),
                                         _ptr(m), _stream()), ctx.handle)
    return m.reshape(*q.shape[:-2], N)


def select_topk_covariance(q_bar: torch.Tensor, k_bar: torch.Tensor, m: torch.Tensor,
                           epsilon: float, k: int, scale: float, force_diagonal: bool = False,
                           return_mask: bool = False):
    """select_topk_covariance (router.hpp:157-193): scores scale * <q_bar_i, k_bar_j>
    + log(M_j + epsilon) on fp32 device tensors q_bar/k_bar [..][N][d], m [..][N]."""
    q4 = q_bar.reshape(-1, 1, *q_bar.shape[-2:]).contiguous()
    k4 = k_bar.reshape(-1, 1, *k_bar.shape[-2:]).contiguous()
    BH, _, N, d = q4.shape
    if not epsilon > 0.0:
        raise InvalidEpsilon(f"InvalidEpsilon: epsilon must be > 0, got {epsilon}")
    if m.numel() != BH * N:
        raise InvalidDimension("InvalidDimension: M has wrong length")
    if k < 1 or k > N:
        raise InvalidSparsity(f"InvalidSparsity: k must lie in [1, N], got {k} for N = {N}")
    ctx = Context.get(q4.device.index)
    desc = _abi.AttnDesc()
    desc.batch, desc.heads, desc.seq_len, desc.head_dim = BH, 1, N * 64, d
    for nm in ("q_strides", "k_strides", "v_strides", "o_strides"):
        getattr(desc, nm)[:] = (N * 64 * d, N * 64 * d, d)
    desc.block_size, desc.group_size, desc.scale, desc.topk = 64, 8, float(scale), int(k)
    desc.variant, desc.force_diagonal, desc.ragged = 3, int(force_diagonal), 1
    desc.router, desc.epsilon = int(RouterStrategy.CovarianceAware), float(epsilon)
    sel = torch.empty((BH, N, k), dtype=torch.int32, device=q4.device)
    W = (N + 31) // 32
    mask = torch.empty((BH, N, W), dtype=torch.int32, device=q4.device)
    st = ctx.lib.pisa_b200_select_cov(ctx.handle, C.byref(desc), _ptr(q4), _ptr(k4),
                                      _ptr(m.contiguous().float()), _ptr(sel), _ptr(mask), _stream())
    _raise(st, ctx.handle)
    sel = sel.reshape(*q_bar.shape[:-2], N, k)
    if return_mask:
        return sel, mask.reshape(*q_bar.shape[:-2], N, W)
    return sel


def _check_engine_inputs(desc, selected, stats: BlockStatistics, cfg: AttentionConfig):
    """detail::check_engine_inputs (engine.hpp:61-80): the plan and the block
    statistics must describe these inputs, else InvalidDimension (the plan's
    ordering / range is validated on the device, SelectionPlan::validate)."""
    B, H, L, d = desc.batch, desc.heads, desc.seq_len, desc.head_dim
    N = -(-L // cfg.block_size)
    lead = [(B, H), (H,)] if B == 1 else [(B, H)]  # [B][H][..] or, for B = 1, [H][..]

    def fits(t, tail):
        return tuple(t.shape[-len(tail):]) == tail and tuple(t.shape[:-len(tail)]) in lead

    if stats.block_size != cfg.block_size or stats.num_blocks != N or stats.dim != d:
        raise InvalidDimension("InvalidDimension: block statistics do not match inputs")
    for t, tail in ((stats.k_bar, (N, d)), (stats.v_hat, (N, d)), (stats.h_bar, (d, d))):
        if not fits(t, tail) or t.device != selected.device:
            raise InvalidDimension("InvalidDimension: block statistics do not match inputs")
    if selected.dim() < 3 or not fits(selected, (N, selected.shape[-1])):
        raise InvalidDimension("InvalidDimension: selection plan does not match inputs")
    if selected.shape[-1] < 1:
        raise EmptySelection("EmptySelection: query blocks select no key block")


def pisa_attention(q, k, v, selected: torch.Tensor, stats: BlockStatistics,
                   cfg: AttentionConfig = AttentionConfig(), variant=PisaVariant.Hybrid,
                   out_dtype=torch.bfloat16, diagnostics=True, ragged=True,
                   literal_phase3: Optional[bool] = None):
    """pisa_streaming / pisa_reference (engine.hpp:103-383) for a given plan and
    prepare products. q/k/v [H][L][d] or [B][H][L][d]; selected [..][N][k].
    ``literal_phase3`` defaults to ``cfg.literal_phase3`` for Hybrid (the
    streaming path's diagnostic, engine.hpp:345-346) and is off otherwise."""
    if literal_phase3 is None:
        literal_phase3 = cfg.literal_phase3 and int(variant) == int(PisaVariant.Hybrid)
    q4, k4, v4 = _bundle4(q), _bundle4(k), _bundle4(v)
    _check_inputs(q4, k4, v4)
    ctx = Context.get(q4.device.index)
    out = torch.empty(q4.shape, dtype=out_dtype, device=q4.device)
    kk = selected.shape[-1]
    desc = make_desc(q4, k4, v4, out, block_size=cfg.block_size, group_size=cfg.group_size,
                     scale=cfg.scale, topk=kk, variant=variant,
                     literal_phase3=literal_phase3, ragged=ragged, check_finite=True)
    B, H, L = desc.batch, desc.heads, desc.seq_len
    _check_engine_inputs(desc, selected, stats, cfg)
    diag = _abi.Diag()
    ex = {}
    if diagnostics:
        for nm in ("row_max", "ell", "ell_tail"):
            ex[nm] = torch.empty((B, H, L), dtype=torch.float32, device=q4.device)
            setattr(diag, nm, ex[nm].data_ptr())
    sel = selected.contiguous().to(torch.int32)
    st = ctx.lib.pisa_b200_attention(ctx.handle, C.byref(desc), _ptr(q4), _ptr(k4), _ptr(v4),
                                     _ptr(sel), _ptr(stats.k_bar.contiguous()),
                                     _ptr(stats.v_hat.contiguous()),
                                     _ptr(stats.h_bar.contiguous()), _ptr(out), C.byref(diag),
                                     _stream())
    _raise(st, ctx.handle)
    return (out, ex) if diagnostics else out


def pisa_streaming(q, k, v, plan, stats, cfg: AttentionConfig = AttentionConfig(), **kw):
    """engine.hpp:374-383 (implicitly Hybrid)."""
    sel = plan.selected if isinstance(plan, SelectionPlan) else plan
    return pisa_attention(q, k, v, sel, stats, cfg, PisaVariant.Hybrid, **kw)


def pisa_reference(q, k, v, plan, stats, variant: PisaVariant,
                   cfg: AttentionConfig = AttentionConfig(), **kw):
    """engine.hpp:103-223 (SparseOnly / Zeroth / Hybrid / GlobalCentroid)."""
    sel = plan.selected if isinstance(plan, SelectionPlan) else plan
    kw.setdefault("literal_phase3", False)  # pisa_reference has no literal Phase 3
    return pisa_attention(q, k, v, sel, stats, cfg, variant, **kw)


def dense_online(q, k, v, cfg: AttentionConfig = AttentionConfig()):
    """dense_online (attention.hpp:186-193): the dense softmax-attention baseline
    the reference's CLI times PISA against (pisa_cli.cpp:719-723). ``q``/``k``/``v``
    [L][d] or [..., L, d] CUDA tensors; scale from ``cfg`` (0 -> 1/sqrt(d),
    attention.hpp:34-37). Runs cuDNN / flash SDPA on the device: a baseline,
    not the PISA path."""
    import torch.nn.functional as F
    scale = cfg.resolved_scale(q.shape[-1])
    squeeze = q.dim() == 2
    if squeeze:
        q, k, v = (t.unsqueeze(0) for t in (q, k, v))
    o = F.scaled_dot_product_attention(q, k, v, scale=scale)
    return o.squeeze(0) if squeeze else o


def pisa_multihead(bundle: TensorBundle, r: float, router: RouterOptions = RouterOptions(),
                   variant: PisaVariant = PisaVariant.Hybrid,
                   cfg: AttentionConfig = AttentionConfig(), use_streaming: bool = False,
                   *, ragged: bool = True, out_dtype=torch.bfloat16,
                   diagnostics: bool = True) -> MultiheadResult:
    """pisa_multihead (engine.hpp:408-470): per head prepare -> route -> attention.

    On the GPU all heads run in one stream-ordered K1 -> K2 -> K3 sequence; the
    streaming and reference formulations are the same kernel (they agree to
    1e-10 in the reference, test_engine.cpp:137-150), so ``use_streaming`` only
    decides whether ``cfg.literal_phase3`` applies (streaming Hybrid only, :460).
    A non-finite output raises NumericalOverflow (engine.hpp:368)."""
    if router.row_level:
        raise Unsupported("Unsupported: row-level routing is not on the GPU path")
    cfg.check(bundle.seq_len, ragged=ragged)
    L = bundle.seq_len
    n = -(-L // cfg.block_size)
    res_k = sparsity_to_k(r, n)
    q4, k4, v4 = _bundle4(bundle.q), _bundle4(bundle.k), _bundle4(bundle.v)
    t0 = time.perf_counter()
    # the streaming path (use_streaming and Hybrid, engine.hpp:460) is the only
    # one that honours literal_phase3; every head's output is checked for
    # non-finite values (check_output_finite, engine.hpp:221,368)
    literal = cfg.literal_phase3 and use_streaming and int(variant) == int(PisaVariant.Hybrid)
    out, ex = fwd(q4, k4, v4, out_dtype=out_dtype, diagnostics=diagnostics, return_plan=True,
                  block_size=cfg.block_size, group_size=cfg.group_size, scale=cfg.scale,
                  sparsity=r, variant=variant, force_diagonal=router.force_diagonal,
                  literal_phase3=literal, ragged=ragged, router=router.strategy,
                  epsilon=router.epsilon, check_finite=True)
    torch.cuda.current_stream().synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    res = MultiheadResult(k=res_k.k, num_blocks=n, sparsity_requested=r,
                          sparsity_realized=res_k.realized, attention_ms=ms)
    H = bundle.num_heads
    for h in range(H):
        po = PisaOutput(output=out[0, h])
        if diagnostics:
            rm = ex["row_max"][0, h].double()
            lift = torch.exp(rm)
            po.row_max = rm
            po.denom = ex["ell"][0, h].double() * lift
            po.ell_tail = ex["ell_tail"][0, h].double() * lift
            po.tail_mass = float(cfg.block_size) * po.ell_tail
        res.heads.append(po)
        res.plans.append(SelectionPlan(n, res_k.k, ex["selected"][0, h]))
    return res


def selftest_mma(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Runs the tcgen05 operand-mode self test on two bf16 [128][128] tiles."""
    ctx = Context.get(a.device.index)
    out = torch.empty((4, 128, 128), dtype=torch.float32, device=a.device)
    _raise(ctx.lib.pisa_b200_selftest_mma(ctx.handle, _ptr(a.contiguous()),
                                          _ptr(b.contiguous()), _ptr(out), _stream()), ctx.handle)
    return out


def kernel_names() -> List[str]:
    L = _abi.load()
    out, i = [], 0
    while True:
        nm = L.pisa_b200_kernel_name(i)
        if not nm:
            return out
        out.append(nm.decode())
        i += 1
