"""PQKV tensor files: the reference's on-disk Q/K/V bundle (io.hpp:17-221).

Layout (little-endian), header exactly 24 bytes:

    offset size field
    0      4    magic "PQKV"
    4      4    version   u32
    8      4    dtype     u32 (1 = f32, 2 = f64; 3 = bf16, version 2 only)
    12     4    num_heads u32
    16     4    head_dim  u32
    20     4    seq_len   u32   (the reference's SPEC.md:100 says u64; the code
                                 and its files use u32 at offset 20, io.hpp:25,125)
    24     -    Q, K, V payloads back to back, each row-major [heads][L][d]

Version 1 is the reference format, read and written bit-compatibly. Version 2
adds the bf16 dtype tag (3), the element type of the GPU path, so a bundle can
round-trip at the precision the kernels compute in; the
reference rejects it with UnsupportedVersion, as it should.

Errors mirror the reference (errors.hpp:52-80, ErrorKind::Io): BadMagic,
UnsupportedVersion, UnsupportedDtype, MalformedFile (truncated header or
payload, trailing bytes), NonFiniteValue (first non-finite entry with its
head / row / col), IoError (open / write failures).
"""
from __future__ import annotations

import os
import struct
from typing import Tuple

import numpy as np
import torch

from .pisa import (BadMagic, IoError, MalformedFile, NonFiniteValue, UnsupportedDtype,
                   UnsupportedVersion)

MAGIC = b"PQKV"
HEADER_BYTES = 24
DTYPES = {1: np.dtype("<f4"), 2: np.dtype("<f8"), 3: np.dtype("<u2")}  # 3: bf16 bit patterns
TAG_OF = {"f32": 1, "f64": 2, "bf16": 3}


def _to_numpy(x, tag: int) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach()
        if tag == 3:
            return x.to(torch.bfloat16).cpu().view(torch.int16).numpy().view("<u2")
        return x.to(torch.float32 if tag == 1 else torch.float64).cpu().numpy()
    x = np.asarray(x)
    if tag == 3:
        t = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16)
        return t.view(torch.int16).numpy().view("<u2")
    return x.astype(DTYPES[tag])


def write_bundle(path: str, q, k, v, dtype: str = "f32") -> int:
    """write_bundle_file (io.hpp:102-126, :207-214); q/k/v [H][L][d]. Returns bytes."""
    if dtype not in TAG_OF:
        raise UnsupportedDtype(f"UnsupportedDtype: {dtype}")
    tag = TAG_OF[dtype]
    arrs = [_to_numpy(x, tag) for x in (q, k, v)]
    shape = tuple(arrs[0].shape)
    if len(shape) != 3 or any(tuple(a.shape) != shape for a in arrs):
        from .pisa import InvalidDimension
        raise InvalidDimension("InvalidDimension: bundle payload size does not match its shape")
    H, L, d = shape
    version = 2 if tag == 3 else 1
    header = MAGIC + struct.pack("<5I", version, tag, H, d, L)
    try:
        with open(path, "wb") as f:
            f.write(header)
            for a in arrs:
                f.write(np.ascontiguousarray(a).tobytes())
    except OSError as e:
        raise IoError(f"IoError: cannot open {path} for writing ({e})") from None
    return HEADER_BYTES + 3 * H * L * d * DTYPES[tag].itemsize


def read_bundle(path: str) -> Tuple[np.ndarray, np.ndarray, np.ndarray, str]:
    """read_bundle_file (io.hpp:180-221): returns (q, k, v, dtype_name); bf16
    bundles come back as float32 arrays holding the exact bf16 values."""
    try:
        size = os.path.getsize(path)
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"IoError: cannot open {path} for reading ({e})") from None
    with f:
        header = f.read(HEADER_BYTES)
        if len(header) != HEADER_BYTES:
            raise MalformedFile(f"MalformedFile: header truncated: expected {HEADER_BYTES} bytes, "
                                f"got {len(header)}")
        if header[:4] != MAGIC:
            raise BadMagic('BadMagic: first 4 bytes are not "PQKV"')
        version, tag, H, d, L = struct.unpack("<5I", header[4:])
        if version not in (1, 2):
            raise UnsupportedVersion(f"UnsupportedVersion: version {version}, expected 1")
        if tag not in DTYPES or (tag == 3 and version != 2):
            raise UnsupportedDtype(f"UnsupportedDtype: dtype tag {tag}")
        dt = DTYPES[tag]
        n = H * L * d
        expected = 3 * n * dt.itemsize
        payload = f.read(expected)
        if len(payload) != expected:
            raise MalformedFile(f"MalformedFile: payload truncated: expected {expected} bytes, "
                                f"got {len(payload)}")
        if size != HEADER_BYTES + expected:
            raise MalformedFile(f"MalformedFile: payload longer than expected {expected} bytes")
    raw = np.frombuffer(payload, dtype=dt).reshape(3, H, L, d)
    if tag == 3:
        vals = torch.from_numpy(raw.view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    else:
        vals = raw.astype(np.float64 if tag == 2 else np.float32)
    for idx, name in enumerate("QKV"):  # check_finite (io.hpp:84-101): first offender
        bad = np.flatnonzero(~np.isfinite(vals[idx]))
        if bad.size:
            i = int(bad[0])
            raise NonFiniteValue(f"NonFiniteValue: {name} head {i // (L * d)} row {(i // d) % L} "
                                 f"col {i % d}")
    name = {1: "f32", 2: "f64", 3: "bf16"}[tag]
    return vals[0], vals[1], vals[2], name
