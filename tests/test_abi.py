"""The C-ABI library loads on a CPU-only host, exports every symbol
include/pisa_b200.h declares, and its host-side validation mirrors the
reference's error classes (no device calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_01077_b200 import _abi, build
    build.build()
    return _abi.load()


def _declared():
    with open(os.path.join(ROOT, "include", "pisa_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(pisa_b200_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    from paper_2602_01077_b200 import _abi
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_abi.EXPORTED)


def test_abi_version(lib):
    assert lib.pisa_b200_abi_version() == 3  # v3: host-buffer step entries + reference generators


def test_kernel_names(lib):
    import paper_2602_01077_b200 as P
    names = P.kernel_names()
    assert names[:4] == ["block_stats_kernel", "hbar_reduce_kernel", "select_kernels",
                         "fused_attn_kernel"]


@pytest.mark.parametrize("r,n,k", [(0.875, 512, 64), (0.0, 17, 17), (0.99, 8, 1), (0.3, 10, 7),
                                   (0.875, 1182, 148), (0.875, 1857, 232)])
def test_sparsity_to_k_matches_reference(lib, r, n, k):
    import paper_2602_01077_b200 as P
    res = P.sparsity_to_k(r, n)
    assert res.k == k and res.realized == pytest.approx((n - k) / n)


def test_sparsity_to_k_errors(lib):
    import paper_2602_01077_b200 as P
    with pytest.raises(P.InvalidSparsity):
        P.sparsity_to_k(1.0, 8)
    with pytest.raises(P.InvalidSparsity):
        P.sparsity_to_k(-0.1, 8)


def _desc(**kw):
    from paper_2602_01077_b200 import _abi
    d = _abi.AttnDesc()
    B, H, L, D = kw.get("B", 1), kw.get("H", 2), kw.get("L", 4096), kw.get("D", 128)
    d.batch, d.heads, d.seq_len, d.head_dim = B, H, L, D
    for nm in ("q_strides", "k_strides", "v_strides", "o_strides"):
        getattr(d, nm)[:] = (H * L * D, L * D, D)
    d.block_size, d.group_size = kw.get("block", 64), kw.get("group", 8)
    d.scale, d.sparsity, d.topk = kw.get("scale", 0.0), kw.get("r", 0.875), kw.get("topk", 0)
    d.variant, d.router = kw.get("variant", 3), kw.get("router", 0)
    d.epsilon, d.row_level = kw.get("eps", 1e-6), kw.get("row_level", 0)
    d.ragged = kw.get("ragged", 1)
    return d


def _resolve(lib, d):
    from paper_2602_01077_b200 import _abi
    n, k, sc = _abi.i64(), _abi.i64(), C.c_double()
    st = lib.pisa_b200_resolve(C.byref(d), C.byref(n), C.byref(k), C.byref(sc))
    return st, n.value, k.value, sc.value


def test_resolve_wan14b(lib):
    st, n, k, sc = _resolve(lib, _desc(H=40, L=75600))
    assert (st, n, k) == (0, 1182, 148)
    assert sc == pytest.approx(128 ** -0.5)


@pytest.mark.parametrize("kw,status", [
    (dict(L=75600, ragged=0), 2),         # BlockDivisibility (attention.hpp:43-47)
    (dict(block=0), 1),                   # InvalidDimension (attention.hpp:40-42)
    (dict(group=0), 1),
    (dict(r=1.0), 3),                     # InvalidSparsity (router.hpp:81-84)
    (dict(topk=65, L=4096), 3),           # k > N
    (dict(variant=2), 8),                 # BlockFirst: not on the GPU path
    (dict(router=1, eps=0.0), 4),         # InvalidEpsilon (router.hpp:164-166)
    (dict(router=1, eps=-1.0), 4),
    (dict(router=2), 1),                  # unknown router
    (dict(row_level=1), 8),               # row-level routing: not on the GPU path
    (dict(block=32), 8),
    (dict(D=96), 8),
    (dict(L=0), 1),
])
def test_resolve_errors(lib, kw, status):
    assert _resolve(lib, _desc(**kw))[0] == status


def test_covariance_router_resolves(lib):
    st, n, k, _ = _resolve(lib, _desc(router=1, eps=1e-6, L=1000))
    assert (st, n, k) == (0, 16, 2)


def test_explicit_topk_and_scale(lib):
    st, n, k, sc = _resolve(lib, _desc(topk=5, scale=0.5, L=1000))
    assert (st, n, k, sc) == (0, 16, 5, 0.5)


def test_python_api_requires_cuda_tensors(lib):
    import torch

    import paper_2602_01077_b200 as P
    x = torch.zeros((1, 1, 128, 64), dtype=torch.bfloat16)
    with pytest.raises(P.InvalidDimension):
        P.fwd(x, x, x)


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2602_01077_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "import oracle" not in src and "liboracle" not in src, f
                assert "pisa_oracle" not in src, f


def test_cpp_shim_header_compiles(tmp_path):
    """include/pisa_b200.hpp + a reference-style caller build with plain g++."""
    import subprocess
    obj = tmp_path / "shim.o"
    subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-Wall", "-Werror", "-I",
                    os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp")],
                   check=True)
    subprocess.run(["gcc", "-std=c99", "-fsyntax-only", "-Wall", "-Werror", "-x", "c",
                    os.path.join(ROOT, "include", "pisa_b200.h")], check=True)
    del obj
