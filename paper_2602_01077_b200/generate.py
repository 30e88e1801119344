"""The reference's synthetic inputs (generate.hpp:29-116), bit-identical, from
the C ABI's generators (pisa_b200_gen_gaussian / pisa_b200_gen_clustered,
csrc/generate.cu): the fixtures bench.py feeds both arms and the parity harness
feeds the GPU and the reference. Host tensors [heads][L][d]."""
from __future__ import annotations

import torch

from . import _abi
from .pisa import _raise

_DT = {torch.bfloat16: 0, torch.float32: 1, torch.float64: 2}


def _alloc(heads, L, d, dtype, pin):
    if dtype not in _DT:
        raise TypeError(f"dtype must be one of {list(_DT)}")
    return [torch.empty((heads, L, d), dtype=dtype, pin_memory=pin) for _ in range(3)]


def gen_gaussian(seed: int, heads: int, L: int, d: int, std: float = 1.0, *, dtype=torch.bfloat16,
                 pin_memory: bool = False, threads: int = 0):
    """gen_gaussian<float>(seed, heads, L, d, std) (generate.hpp:29-49); bf16 is the
    RNE rounding of the float values. Returns host (q, k, v)."""
    q, k, v = _alloc(heads, L, d, dtype, pin_memory)
    _raise(_abi.load().pisa_b200_gen_gaussian(int(seed), int(heads), int(L), int(d), float(std), _DT[dtype],
                                              q.data_ptr(), k.data_ptr(), v.data_ptr(), int(threads)),
           where="gen_gaussian")
    return q, k, v


def gen_clustered(seed: int, heads: int, L: int, d: int, n_clusters: int = 16, concentration: float = 2.0,
                  noise_std: float = 0.15, *, dtype=torch.bfloat16, pin_memory: bool = False, threads: int = 0):
    """gen_clustered<float>(seed, heads, L, d, n_clusters, concentration, noise_std)
    (generate.hpp:57-116; defaults = the CLI's, pisa_cli.cpp:27-39). Host (q, k, v)."""
    q, k, v = _alloc(heads, L, d, dtype, pin_memory)
    _raise(_abi.load().pisa_b200_gen_clustered(int(seed), int(heads), int(L), int(d), int(n_clusters),
                                               float(concentration), float(noise_std), _DT[dtype],
                                               q.data_ptr(), k.data_ptr(), v.data_ptr(), int(threads)),
           where="gen_clustered")
    return q, k, v
