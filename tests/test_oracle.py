"""The CPU oracle (oracle/pisa_oracle.cpp) pinned against the reference's own
golden vectors and tests and against the unmodified
reference library compiled here (oracle/_ref) or its committed outputs
(tests/golden/*.npz, made by tests/golden/make_golden.py)."""
import glob
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# ---------------------------------------------------------------- KATs ----
def test_rng_golden_sequence(oracle_mod):
    # test_generate.cpp:13-24
    O = oracle_mod
    u = np.empty(4, np.uint64)
    O.lib().oracle_rng_u64(42, u, 4)
    assert [int(x) for x in u] == [0xd0764d4f4476689f, 0x519e4174576f3791,
                                   0xfbe07cfb0c24ed8c, 0xb37d9f600cd835b8]
    g = np.empty(4)
    O.lib().oracle_rng_gaussian(0, g, 4)
    np.testing.assert_allclose(g, [-0.65426512664059489, 0.59729745601051942,
                                   0.94168378000437492, 0.067896945646594112], rtol=0, atol=1e-15)


def test_rng_matches_reference_fixture(oracle_mod):
    f = np.load(os.path.join(GOLDEN, "rng.npz"))
    u = np.empty(8, np.uint64)
    oracle_mod.lib().oracle_rng_u64(42, u, 8)
    assert np.array_equal(u, f["u64_seed42"])
    g = np.empty(8)
    oracle_mod.lib().oracle_rng_gaussian(0, g, 8)
    assert np.array_equal(g, f["gauss_seed0"])


@pytest.mark.parametrize("r,n,k,realized", [(0.875, 512, 64, 0.875), (0.0, 17, 17, 0.0),
                                            (0.99, 8, 1, 7 / 8), (0.3, 10, 7, 0.3),
                                            (0.875, 1182, 148, (1182 - 148) / 1182)])
def test_sparsity_to_k(oracle_mod, r, n, k, realized):
    # test_router.cpp:14-24 (+ the Wan2.1-14B shape)
    kk, real = oracle_mod.sparsity_to_k(r, n)
    assert kk == k and real == pytest.approx(realized, abs=1e-15)


@pytest.mark.parametrize("r", [1.0, -0.1, float("nan")])
def test_sparsity_to_k_rejects(oracle_mod, r):
    with pytest.raises(oracle_mod.OracleError) as e:
        oracle_mod.sparsity_to_k(r, 8)
    assert e.value.status == 3  # InvalidSparsity


def test_topk_all_zero_ties_to_low_index(oracle_mod):
    # test_router.cpp:26-32
    sel = oracle_mod.select_plain(np.zeros((3, 4)), np.zeros((8, 4)), 3, 1.0)
    assert (sel == [0, 1, 2]).all()


def test_topk_constructed_tie(oracle_mod):
    # test_router.cpp:167-177
    sel = oracle_mod.select_plain(np.array([[1.0]]), np.array([[5.0], [2.0], [1.0], [2.0]]), 2, 1.0)
    assert sel.tolist() == [[0, 1]]


def test_force_diagonal(oracle_mod):
    # test_router.cpp:179-193
    qb = np.ones((4, 1))
    kb = np.array([[10.0], [9.0], [8.0], [7.0]])
    sel = oracle_mod.select_plain(qb, kb, 2, 1.0, force_diagonal=True)
    for i in range(4):
        assert i in sel[i] and len(sel[i]) == 2 and sorted(sel[i]) == list(sel[i])


def test_topk_matches_argsort(oracle_mod):
    # test_router.cpp:44-58: against a full stable argsort
    O = oracle_mod
    rng = np.random.default_rng(0)
    qb = rng.standard_normal((16, 16))
    kb = rng.standard_normal((40, 16))
    sel, sc = O.select_plain(qb, kb, 7, 0.25, return_scores=True)
    for i in range(16):
        order = np.argsort(-sc[i], kind="stable")[:7]
        assert np.array_equal(np.sort(order), sel[i])


# -------------------------------------------------- against the reference --
def _fixtures():
    return sorted(glob.glob(os.path.join(GOLDEN, "*_h*_l*.npz")))


@pytest.mark.parametrize("path", _fixtures(), ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_matches_reference_fixture(oracle_mod, path):
    """Plan bit-exact, prepare products 1e-12, outputs of every variant within fp32
    output rounding of the reference's pisa_multihead (T = float)."""
    O = oracle_mod
    f = np.load(path)
    q, k, v = f["q"], f["k"], f["v"]
    H, L, d = q.shape
    fd = bool(f["force_diagonal"])
    for h in range(H):
        kb, vh, hb, _ = O.block_stats(k[h], v[h])
        np.testing.assert_allclose(kb, f["k_bar"][h], rtol=0, atol=1e-12)
        np.testing.assert_allclose(vh, f["v_hat"][h], rtol=0, atol=1e-12)
        np.testing.assert_allclose(hb, f["h_bar"][h], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(O.query_means(q[h]), f["q_bar"][h], rtol=0, atol=1e-12)
    for variant in ("hybrid", "zeroth", "sparse_only", "global_centroid"):
        res = O.multihead(q, k, v, r=float(f["r"]), variant=variant, force_diagonal=fd)
        assert np.array_equal(res["selected"], f["selected"]), variant
        ref = f[f"out_{variant}"].astype(np.float64)
        err = np.abs(res["out"] - ref).max()
        assert err <= 2e-6 * max(1.0, np.abs(ref).max()), (variant, err)
        denom = res["ell"] * np.exp(res["row_max"])
        np.testing.assert_allclose(denom, f[f"denom_{variant}"], rtol=1e-9)


@pytest.mark.parametrize("kind,seed,H,L,d,r", [("gaussian", 3, 2, 1024, 64, 0.75),
                                               ("clustered", 4, 1, 2048, 128, 0.875),
                                               ("clustered", 5, 2, 640, 16, 0.5)])
def test_oracle_matches_live_reference(oracle_mod, ref_available, kind, seed, H, L, d, r):
    if not ref_available:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    O = oracle_mod
    q, k, v = O.gen(kind, seed, H, L, d)
    ref = O.ref_multihead(q, k, v, r=r, accum_f64=True, streaming=True)
    res = O.multihead(q, k, v, r=r)
    assert np.array_equal(res["selected"], ref["selected"])
    assert np.abs(res["out"] - ref["out"]).max() <= 2e-6
    np.testing.assert_allclose(res["ell_tail"] * np.exp(res["row_max"]), ref["ell_tail"], rtol=1e-9)


# --------------------------------------- covariance-aware / row-level router --
@pytest.mark.parametrize("path", _fixtures(), ids=lambda p: os.path.basename(p)[:-4])
def test_covariance_router_matches_reference_fixture(oracle_mod, path):
    """M_j (Jacobi spectral norms) 1e-10, covariance plan bit-exact, Hybrid output
    with that plan within fp32 rounding of the reference's pisa_multihead with
    RouterOptions{CovarianceAware} (engine.hpp:439-453)."""
    O = oracle_mod
    f = np.load(path)
    q, k, v = f["q"], f["k"], f["v"]
    H, L, d = q.shape
    fd = bool(f["force_diagonal"])
    kk, scale = int(f["topk"]), 1.0 / np.sqrt(d)
    for h in range(H):
        m = O.block_norms(k[h], v[h])
        np.testing.assert_allclose(m, f["m_norms"][h], rtol=1e-10)
        st = O.block_stats(k[h], v[h])
        sel = O.select_cov(O.query_means(q[h]), st[0], m, kk, scale, 1e-6, fd)
        assert np.array_equal(sel, f["selected_cov"][h])
        out = O.pisa_attention(q[h], k[h], v[h], sel, st, scale, "hybrid")[0]
        ref = f["out_hybrid_cov"][h].astype(np.float64)
        assert np.abs(out - ref).max() <= 2e-6 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("kind,seed,L,d", [("gaussian", 7, 1024, 64), ("clustered", 8, 768, 128),
                                           ("clustered", 9, 512, 16)])
def test_router_variants_match_live_reference(oracle_mod, ref_available, kind, seed, L, d):
    """select_topk_covariance / select_topk_rowmax (plain and rectified) and the
    spectral norms against the unmodified reference (router.hpp:157-233)."""
    if not ref_available:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    O = oracle_mod
    q, k, v = (x[0] for x in O.gen(kind, seed, 1, L, d))
    m = O.block_norms(k, v)
    np.testing.assert_allclose(m, O.ref_block_norms(k, v), rtol=1e-12)
    kb = O.block_stats(k, v)[0]
    qb = O.query_means(q)
    N, scale = kb.shape[0], 1.0 / np.sqrt(d)
    for kk in (1, N // 4, N - 1):
        for fd in (False, True):
            assert np.array_equal(O.select_cov(qb, kb, m, kk, scale, 1e-6, fd),
                                  O.ref_select_cov(qb, kb, m, kk, scale, 1e-6, fd))
        for eps in (1e-6, 0.5):
            assert np.array_equal(O.select_rowmax(q, kb, kk, scale, m=m, eps=eps),
                                  O.ref_select_rowmax(q, kb, kk, scale, m=m, eps=eps))
        assert np.array_equal(O.select_rowmax(q, kb, kk, scale), O.ref_select_rowmax(q, kb, kk, scale))


def test_covariance_router_rejects_epsilon(oracle_mod):
    # router.hpp:164-166: epsilon must be > 0 -> InvalidEpsilon
    O = oracle_mod
    with pytest.raises(O.OracleError) as e:
        O.select_cov(np.zeros((2, 4)), np.zeros((2, 4)), np.ones(2), 1, 1.0, 0.0)
    assert e.value.status == 4


def test_block_norms_of_identical_blocks_vanish(oracle_mod):
    # every block equal -> H_j == H_bar -> M_j == 0 (the all-zero matrix path of
    # spectral_norm_exact, block_stats.hpp:58-60)
    O = oracle_mod
    rng = np.random.default_rng(0)
    kb = rng.standard_normal((64, 32)).astype(np.float32)
    vb = rng.standard_normal((64, 32)).astype(np.float32)
    m = O.block_norms(np.tile(kb, (4, 1)), np.tile(vb, (4, 1)))
    assert np.all(m == 0.0)


# ------------------------------------------------ invariants of the math --
def test_full_coverage_equals_dense(oracle_mod):
    # test_engine.cpp:52-66 (r = 0: every variant = dense), incl. a ragged L
    O = oracle_mod
    for L in (256, 200):
        q, k, v = O.gen("gaussian", 0, 1, L, 16, bf16=False)
        dense = O.dense(q[0], k[0], v[0], 0.25)
        for variant in ("sparse_only", "zeroth", "hybrid", "global_centroid"):
            res = O.multihead(q, k, v, r=0.0, variant=variant)
            assert np.abs(res["out"][0] - dense).max() <= 1e-10
            assert np.abs(res["ell_tail"]).max() == 0.0


def test_constant_key_blocks_make_tail_exact(oracle_mod):
    # test_engine.cpp:68-99: constant key blocks -> Zeroth/Hybrid = dense
    O = oracle_mod
    L, d, B = 512, 16, 64
    q, k, v = O.gen("gaussian", 0, 1, L, d, bf16=False)
    rng = np.random.default_rng(100)
    for j in range(L // B):
        k[0, j * B:(j + 1) * B] = rng.standard_normal(d)
    dense = O.dense(q[0], k[0], v[0], 0.25)
    st = O.block_stats(k[0], v[0])
    sel = O.select_plain(O.query_means(q[0]), st[0], 2, 0.25)
    for variant in ("zeroth", "hybrid"):
        out, *_ = O.pisa_attention(q[0], k[0], v[0], sel, st, 0.25, variant)
        assert np.abs(out - dense).max() <= 1e-6


def test_literal_phase3_scales_correction_by_B(oracle_mod):
    # test_engine.cpp:192-209: (default - zeroth) == B * (literal - zeroth)
    O = oracle_mod
    q, k, v = O.gen("clustered", 4, 1, 512, 16, bf16=False)
    st = O.block_stats(k[0], v[0])
    sel = O.select_plain(O.query_means(q[0]), st[0], 4, 0.25)
    z, *_ = O.pisa_attention(q[0], k[0], v[0], sel, st, 0.25, "zeroth")
    dflt, *_ = O.pisa_attention(q[0], k[0], v[0], sel, st, 0.25, "hybrid")
    lit, *_ = O.pisa_attention(q[0], k[0], v[0], sel, st, 0.25, "hybrid", literal_phase3=True)
    np.testing.assert_allclose(dflt - z, 64.0 * (lit - z), rtol=1e-9, atol=1e-12)


def test_diagnostics_contract(oracle_mod):
    # test_engine.cpp:118-135
    O = oracle_mod
    q, k, v = O.gen("clustered", 1, 1, 512, 16, bf16=False)
    res = O.multihead(q, k, v, r=0.75)
    assert (res["ell"] > 0).all() and (res["ell_tail"] > 0).all()
    sp = O.multihead(q, k, v, r=0.75, variant="sparse_only")
    assert (sp["ell_tail"] == 0).all() and (sp["ell"] > 0).all()


def test_ragged_reduces_to_reference_when_divisible(oracle_mod):
    """The ragged extension is the same code path; at L % 64 == 0 it is the
    reference (pinned above). With a ragged tail, the partial block's centroid
    weight is n_last: check D_t = sum over all keys of the piecewise weights
    by comparing against an explicit per-row evaluation."""
    O = oracle_mod
    L, d = 200, 16  # 3 full blocks + 8 rows
    q, k, v = O.gen("gaussian", 7, 1, L, d, bf16=False)
    st = O.block_stats(k[0], v[0])
    kb = st[0]
    assert np.allclose(kb[3], k[0, 192:200].mean(0))
    sel = np.array([[0], [1], [2], [3]], np.int32)
    out, m, ell, et = O.pisa_attention(q[0], k[0], v[0], sel, st, 0.25, "zeroth")
    t = 5  # a row of query block 0: exact block 0, centroids 1, 2, 3 (weights 64, 64, 8)
    s_exact = 0.25 * k[0, :64].astype(np.float64) @ q[0, t]
    s_c = 0.25 * kb[1:] @ q[0, t].astype(np.float64)
    mx = max(s_exact.max(), s_c.max())
    den = np.exp(s_exact - mx).sum() + (np.array([64, 64, 8]) * np.exp(s_c - mx)).sum()
    assert ell[t] == pytest.approx(den, rel=1e-12)
    assert et[t] == pytest.approx(np.exp(s_c - mx).sum(), rel=1e-12)


def test_oracle_rejects_block_first(oracle_mod):
    O = oracle_mod
    q, k, v = O.gen("gaussian", 0, 1, 128, 8, bf16=False)
    st = O.block_stats(k[0], v[0])
    with pytest.raises(O.OracleError) as e:
        O.pisa_attention(q[0], k[0], v[0], np.array([[0], [1]], np.int32), st, 0.5, "block_first")
    assert e.value.status == 8


# ------------------------------------------- parity harness (oracle/parity.py) --
def test_ref_head_parity_is_the_reference_pipeline(oracle_mod, ref_available):
    """ref_head_parity = the reference's own per-head pipeline: its plan equals
    pisa_multihead's, and pisa_streaming on gathered query blocks equals the
    same rows of the full-head output (query blocks are independent)."""
    if not ref_available:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    from oracle import parity
    O = oracle_mod
    q, k, v = O.gen("clustered", 3, 1, 1024, 64)
    blocks = parity.sample_blocks(16, 8, run=2)
    sel, qb, kb, out = O.ref_head_parity(q[0], k[0], v[0], 0.75, blocks=blocks)
    # the same with the plan rows given explicitly: identical
    out2 = O.ref_head_parity(q[0], k[0], v[0], 0.75, blocks=blocks, sub_plan=sel[blocks])[3]
    assert np.array_equal(out, out2)
    full = O.ref_multihead(q, k, v, r=0.75, accum_f64=True, streaming=True)
    assert np.array_equal(sel, full["selected"][0])
    rows = np.concatenate([np.arange(i * 64, (i + 1) * 64) for i in blocks])
    assert np.abs(out - full["out"][0][rows]).max() <= 1e-6
    np.testing.assert_allclose(kb, O.ref_block_stats(q[0], k[0], v[0])[0], rtol=0, atol=0)
    # the classifier: identical plans -> nothing; a swap across the k-th score -> non-tie
    assert parity.classify_rows(sel, sel, qb, kb, 4, 0.125) == (0, 0, 0, [])
    bad = sel.copy()
    N = sel.shape[0]
    s = 0.125 * (kb @ qb[3])
    worst = np.argsort(-s)[N - 1]  # the lowest-scoring block replaces a selected one
    bad[3, 0] = worst
    nb, near, pairs, non = parity.classify_rows(bad, sel, qb, kb, 4, 0.125)
    assert nb == 1 and near == 0 and non == [3]
    assert list(parity.runs_of(np.array([0, 1, 2, 7, 8, 15]))) == [(0, 3), (7, 9), (15, 16)]
    assert parity.sample_blocks(1182, 64)[-1] == 1181 and len(parity.sample_blocks(1182, 64)) == 64
