"""The product's generators (csrc/generate.cu) against the reference's own
gen_gaussian / gen_clustered (oracle/_ref, the unmodified library): every
value bit-identical, for any thread count and output dtype. CPU only."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2602_01077_b200 as P

SHAPES = [(1, 64, 64), (3, 1000, 128), (2, 777, 64), (1, 33, 3), (2, 130, 7)]


@pytest.mark.parametrize("kind", ["gaussian", "clustered"])
@pytest.mark.parametrize("H,L,d", SHAPES)
def test_generators_bit_identical_to_reference(kind, H, L, d):
    ref = O.ref_gen(kind, 11, H, L, d)
    fn = P.gen_gaussian if kind == "gaussian" else P.gen_clustered
    for threads in (1, 3, 16):
        got = fn(11, H, L, d, dtype=torch.float32, threads=threads)
        for g, r in zip(got, ref):
            assert np.array_equal(g.numpy(), r), (kind, threads)
        bf = fn(11, H, L, d, dtype=torch.bfloat16, threads=threads)
        for g, r in zip(bf, ref):
            assert np.array_equal(g.float().numpy(), O.round_bf16(r)), (kind, threads)


def test_f64_and_reference_golden_values():
    # test_generate.cpp:13-24: Rng(0).gaussian() = -0.65426512664059489...
    q, _, _ = P.gen_gaussian(0, 1, 1, 2, dtype=torch.float64)
    assert q[0, 0, 0].item() == pytest.approx(-0.65426512664059489, abs=1e-16)
    g64 = O.ref_gen("gaussian", 5, 1, 100, 4)
    q64, k64, _ = P.gen_gaussian(5, 1, 100, 4, dtype=torch.float64)
    assert np.array_equal(q64.numpy().astype(np.float32), g64[0])
    assert np.array_equal(k64.numpy().astype(np.float32), g64[1])


def test_generator_errors():
    with pytest.raises(P.DegenerateScale):
        P.gen_gaussian(0, 1, 4, 4, std=0.0)
    with pytest.raises(P.InvalidDimension):
        P.gen_gaussian(0, 0, 4, 4)
    with pytest.raises(P.InvalidDimension):
        P.gen_clustered(0, 1, 4, 4, n_clusters=5)
    with pytest.raises(P.DegenerateScale):
        P.gen_clustered(0, 1, 4, 4, n_clusters=2, noise_std=-1.0)
