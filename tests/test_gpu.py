"""GPU parity: the sm_100a path through the C ABI against the oracle (which is
pinned to the reference in test_oracle.py) and the reference's own golden outputs.

Tolerances (north_star): routing index sets bit-exact (near-tie swaps counted
and reported where the fp64 gap is below 1e-6 |score|), outputs max-abs <= 2e-2
and cosine >= 0.999 against the fp64 / fp32 reference output. Outputs are taken
as fp32 from the kernel (parity mode) unless a test says otherwise.
"""
import glob
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ATOL = 2e-2
COS = 0.999


@pytest.fixture(scope="module")
def P():
    import paper_2602_01077_b200 as P
    return P


def dev_bf16(x, unsqueeze=True):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()
    return t.unsqueeze(0) if unsqueeze else t


def cosine(a, b):
    a = a.ravel().astype(np.float64)
    b = b.ravel().astype(np.float64)
    return float(a @ b / np.sqrt((a @ a) * (b @ b)))


def check_close(got, ref, atol=ATOL, cos=COS):
    err = float(np.abs(got - ref).max())
    c = cosine(got, ref)
    assert err <= atol and c >= cos, f"max abs {err:.3e}, cosine {c:.7f}"
    return err, c


def run_fwd(P, q, k, v, **kw):
    import torch
    out, ex = P.fwd(dev_bf16(q), dev_bf16(k), dev_bf16(v), out_dtype=torch.float32,
                    diagnostics=True, return_plan=True, **kw)
    torch.cuda.synchronize()
    return out[0].cpu().numpy(), {n: t[0].cpu().numpy() for n, t in ex.items()}


# ------------------------------------------------------------- building blocks
def test_tcgen05_operand_modes(P):
    import torch
    g = torch.Generator().manual_seed(0)
    a = (torch.randn(128, 128, generator=g) * 0.5).to(torch.bfloat16)
    b = (torch.randn(128, 128, generator=g) * 0.5).to(torch.bfloat16)
    out = P.selftest_mma(a.cuda(), b.cuda()).cpu()
    A, B = a.float(), b.float()
    refs = [A @ B[:64].T, A[:64].T @ B[:64], A[:, :64] @ B[:64], A @ B]
    for i, (ref, n) in enumerate(zip(refs, [64, 128, 128, 128])):
        assert (out[i, :, :n] - ref).abs().max().item() < 1e-3, i


@pytest.mark.parametrize("kind,H,L,d", [("gaussian", 2, 1024, 128), ("clustered", 2, 1000, 64),
                                        ("clustered", 1, 4160, 128)])
def test_prepare_matches_oracle(P, oracle_mod, kind, H, L, d):
    O = oracle_mod
    q, k, v = O.gen(kind, 0, H, L, d)
    st = P.compute_prepare(dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False))
    kb, vh, qb, hb = (t[0].cpu().numpy() for t in (st.k_bar, st.v_hat, st.q_bar, st.h_bar))
    for h in range(H):
        okb, ovh, ohb, _ = O.block_stats(k[h], v[h])
        np.testing.assert_allclose(kb[h], okb, rtol=0, atol=1e-6)
        np.testing.assert_allclose(vh[h], ovh, rtol=0, atol=1e-5)
        np.testing.assert_allclose(qb[h], O.query_means(q[h]), rtol=0, atol=1e-6)
        assert np.abs(hb[h] - ohb).max() <= 1e-4 * max(1.0, np.abs(ohb).max())


def _near_tie_swaps(O, qb64, kb64, sel_gpu, k, scale):
    """Rows whose GPU index set differs from the fp64 reference; returns (rows, non-tie rows)."""
    ref, sc = O.select_plain(qb64, kb64, k, scale, return_scores=True)
    bad = np.where((sel_gpu != ref).any(1))[0]
    non_tie = []
    for i in bad:
        kth = np.sort(sc[i])[::-1][k - 1]
        diff = set(sel_gpu[i]) ^ set(ref[i])
        if any(abs(sc[i][j] - kth) > 1e-6 * abs(kth) for j in diff):
            non_tie.append(int(i))
    return len(bad), non_tie


@pytest.mark.parametrize("kind,L,d,r,fd", [("gaussian", 4096, 128, 0.875, False),
                                           ("clustered", 8192, 128, 0.75, False),
                                           ("gaussian", 2000, 64, 0.5, True),
                                           ("clustered", 3000, 128, 0.9, True)])
def test_select_index_sets_exact(P, oracle_mod, kind, L, d, r, fd):
    O = oracle_mod
    q, k, v = O.gen(kind, 1, 1, L, d)
    N = (L + 63) // 64
    kk = O.sparsity_to_k(r, N)[0]
    scale = d ** -0.5
    st = P.compute_prepare(dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False))
    sel = P.select_topk_plain(st.q_bar[0, 0], st.k_bar[0, 0], kk, scale, force_diagonal=fd)
    sel = sel.cpu().numpy()
    okb = O.block_stats(k[0], v[0])[0]
    oqb = O.query_means(q[0])
    ref = O.select_plain(oqb, okb, kk, scale, force_diagonal=fd)
    if fd:
        assert all(i in sel[i] for i in range(N))
    nbad, non_tie = _near_tie_swaps(O, oqb, okb, sel, kk, scale) if not fd else (
        int((sel != ref).any(1).sum()), [])
    assert not non_tie, f"index sets differ beyond near-ties in rows {non_tie}"
    assert nbad <= max(1, N // 1000), f"{nbad} near-tie rows"


@pytest.mark.parametrize("kind,H,L,d,r,fd", [("gaussian", 2, 40000, 128, 0.875, False),
                                              ("clustered", 3, 33000, 64, 0.75, True),
                                              ("clustered", 1, 118800, 128, 0.9, False),
                                              ("gaussian", 1, 262144, 64, 0.99, True)])
@pytest.mark.parametrize("mode", ["1", "stream"])
def test_fused_select_equals_two_kernel_select(P, kind, H, L, d, r, fd, mode, monkeypatch):
    """From N = 512 key blocks the forward scores with the pipelined select
    kernel (q_bar split in TMEM, K1's k_bar splits by TMA, double-buffered
    accumulators): by default ("stream") it writes the row-major keys and
    topk_kernel selects; with PISA_B200_FUSED_SELECT=1 (opt-in one launch,
    keys in an L2 scratch, top-k in the same CTA; slower at Wan2.1-14B,
    profiles/r02c_ab_select.log). Either way the plans equal the tile select
    (score_kernel + topk_kernel, the step entry's path) on the same statistics
    bit for bit, for the plain and the covariance router, d = 64 / 128, up to
    N = 4096."""
    import torch
    if mode == "1":
        monkeypatch.setenv("PISA_B200_FUSED_SELECT", "1")
    else:
        monkeypatch.delenv("PISA_B200_FUSED_SELECT", raising=False)
    gen = P.gen_gaussian if kind == "gaussian" else P.gen_clustered
    q, k, v = (x.reshape(1, H, L, d).cuda() for x in gen(7, H, L, d))
    N = -(-L // 64)
    kk = P.sparsity_to_k(r, N).k
    st = P.compute_prepare(q[0], k[0], v[0])
    for router in (P.RouterStrategy.Plain, P.RouterStrategy.CovarianceAware):
        _, ex = P.fwd(q, k, v, return_plan=True, sparsity=r, force_diagonal=fd, router=router, epsilon=1e-6)
        if router == P.RouterStrategy.Plain:
            ref = P.select_topk_plain(st.q_bar, st.k_bar, kk, d ** -0.5, force_diagonal=fd)
        else:
            m = P.block_norms(q[0], k[0], v[0])
            ref = P.select_topk_covariance(st.q_bar, st.k_bar, m, 1e-6, kk, d ** -0.5, force_diagonal=fd)
        torch.cuda.synchronize()
        assert torch.equal(ex["selected"], ref), router
    del q, k, v
    torch.cuda.empty_cache()


# ------------------------------------------- covariance-aware router (§8f #1) --
@pytest.mark.parametrize("kind,H,L,d", [("gaussian", 1, 1024, 64), ("clustered", 2, 1000, 128),
                                        ("gaussian", 1, 4096, 128)])
def test_block_norms_match_oracle(P, oracle_mod, kind, H, L, d):
    """M_j = ||H_j - H_bar||_2 (Lanczos, fp32) against the fp64 Jacobi oracle
    (pinned to the reference's compute_global_stats in test_oracle.py)."""
    O = oracle_mod
    q, k, v = O.gen(kind, 2, H, L, d)
    m = P.block_norms(dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False)).cpu().numpy()
    for h in range(H):
        ref = O.block_norms(k[h], v[h])
        rel = np.abs(m[h] - ref) / np.maximum(ref, 1e-30)
        assert rel.max() <= 2e-5, f"head {h}: max rel err {rel.max():.3e}"


@pytest.mark.parametrize("d", [64, 128])
def test_block_norms_keys_with_large_mean(P, oracle_mod, d):
    """Keys with a large common offset (|mean| >> spread, as real key
    projections often have): the deviation norms are computed from centred keys,
    so no precision is lost to cancellation."""
    import torch
    O = oracle_mod
    q, k, v = O.gen("gaussian", 4, 1, 2048, d)
    off = np.linspace(-12.0, 12.0, d)[None, None, :]
    k = torch.from_numpy(k + off).to(torch.bfloat16).float().numpy()  # bf16-exact inputs
    m = P.block_norms(dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False)).cpu().numpy()
    ref = O.block_norms(k[0].astype(np.float64), v[0])
    rel = np.abs(m[0] - ref) / np.maximum(ref, 1e-30)
    assert rel.max() <= 2e-5, f"max rel err {rel.max():.3e}"


def _cov_swaps(O, qb64, kb64, m64, sel_gpu, k, scale, fd):
    ref, sc = O.select_cov(qb64, kb64, m64, k, scale, 1e-6, fd, return_scores=True)
    bad = np.where((sel_gpu != ref).any(1))[0]
    non_tie = []
    for i in bad:
        kth = np.sort(sc[i])[::-1][k - 1]
        diff = set(sel_gpu[i]) ^ set(ref[i])
        # GPU scores carry the fp32 rectifier (M_j ~1e-6 relative) on top of fp32 dots
        if any(abs(sc[i][j] - kth) > 1e-5 * max(1.0, abs(kth)) for j in diff):
            non_tie.append(int(i))
    return len(bad), non_tie


@pytest.mark.parametrize("kind,L,d,r,fd", [("gaussian", 4096, 128, 0.875, False),
                                           ("clustered", 3000, 128, 0.75, True)])
def test_covariance_select_index_sets(P, oracle_mod, kind, L, d, r, fd):
    import torch
    O = oracle_mod
    q, k, v = O.gen(kind, 3, 1, L, d)
    N = (L + 63) // 64
    kk = O.sparsity_to_k(r, N)[0]
    scale = d ** -0.5
    qd, kd, vd = dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False)
    st = P.compute_prepare(qd, kd, vd)
    m_gpu = P.block_norms(qd, kd, vd)
    sel = P.select_topk_covariance(st.q_bar[0, 0], st.k_bar[0, 0], m_gpu[0], 1e-6, kk, scale,
                                   force_diagonal=fd).cpu().numpy()
    okb = O.block_stats(k[0], v[0])[0]
    oqb = O.query_means(q[0])
    om = O.block_norms(k[0], v[0])
    nbad, non_tie = _cov_swaps(O, oqb, okb, om, sel, kk, scale, fd)
    assert not non_tie, f"index sets differ beyond near-ties in rows {non_tie}"
    assert nbad <= max(1, N // 200), f"{nbad} near-tie rows"
    # the fused forward with the covariance router routes identically
    out, ex = P.fwd(qd.unsqueeze(0), kd.unsqueeze(0), vd.unsqueeze(0), return_plan=True,
                    sparsity=r, force_diagonal=fd, router=P.RouterStrategy.CovarianceAware,
                    epsilon=1e-6)
    torch.cuda.synchronize()
    assert np.array_equal(ex["selected"][0, 0].cpu().numpy(), sel)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*_h*_l*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
def test_covariance_router_matches_reference_golden(P, path):
    """pisa_multihead with RouterOptions{CovarianceAware}: plan and Hybrid output
    against the unmodified reference's (fixtures from oracle/_ref)."""
    f = np.load(path)
    out, ex = run_fwd(P, f["q"], f["k"], f["v"], sparsity=float(f["r"]),
                      variant=P.PisaVariant.Hybrid, force_diagonal=bool(f["force_diagonal"]),
                      router=P.RouterStrategy.CovarianceAware, epsilon=1e-6)
    assert np.array_equal(ex["selected"], f["selected_cov"])
    check_close(out, f["out_hybrid_cov"].astype(np.float64))


def test_covariance_multihead_api(P):
    import torch
    H, L, d = 2, 768, 64
    g = torch.Generator().manual_seed(0)
    x = [torch.randn(H, L, d, generator=g).to(torch.bfloat16).cuda() for _ in range(3)]
    res = P.pisa_multihead(P.TensorBundle(*x), 0.75,
                           P.RouterOptions(strategy=P.RouterStrategy.CovarianceAware), P.PisaVariant.Hybrid,
                           P.AttentionConfig(), True)
    assert len(res.plans) == H and res.k == 3
    with pytest.raises(P.InvalidEpsilon):
        P.pisa_multihead(P.TensorBundle(*x), 0.75,
                         P.RouterOptions(strategy=P.RouterStrategy.CovarianceAware, epsilon=0.0),
                         P.PisaVariant.Hybrid, P.AttentionConfig(), True)


def test_select_edge_cases(P):
    import torch
    import torch.nn.functional as F

    def sel_of(qb, kb, k, fd=False):
        # zero-padded to the GPU head dim (dots unchanged); the GPU router is
        # self-attention (as many query blocks as key blocks): pad the query list
        nq = len(qb)
        qb = qb + [qb[-1]] * (len(kb) - nq)
        qb = F.pad(torch.tensor(qb, dtype=torch.float32), (0, 64 - len(qb[0]))).cuda()[None]
        kb = F.pad(torch.tensor(kb, dtype=torch.float32), (0, 64 - len(kb[0]))).cuda()[None]
        return P.select_topk_plain(qb, kb, k, 1.0, force_diagonal=fd).cpu().numpy()[0][:nq]

    assert (sel_of([[0.0]] * 3, [[0.0]] * 8, 3) == [0, 1, 2]).all()    # ties -> lowest index
    assert sel_of([[1.0]], [[5.0], [2.0], [1.0], [2.0]], 2).tolist() == [[0, 1]]
    sel = sel_of([[1.0]] * 4, [[10.0], [9.0], [8.0], [7.0]], 2, fd=True)  # router.hpp:146-148
    assert all(i in sel[i] for i in range(4)) and sel.shape == (4, 2)
    assert (sel_of([[1.0]] * 4, [[10.0], [9.0], [8.0], [7.0]], 4) == [0, 1, 2, 3]).all()  # k = N
    assert (sel_of([[-1.0]] * 2, [[0.0], [-0.0], [3.0], [-2.0]], 2) == [0, 3]).all()  # -0 == +0
    with pytest.raises(P.InvalidSparsity):
        sel_of([[1.0]] * 4, [[1.0]] * 4, 5)


@pytest.mark.parametrize("N", [200, 700, 1500, 2100])
@pytest.mark.parametrize("fd", [False, True])
def test_select_heavy_ties(P, oracle_mod, N, fd):
    """Integer-valued q_bar / k_bar make every score an exact small integer, so
    rows carry long runs of equal keys: the top-k (register form up to 256 key
    blocks, shared-memory form above, both with the radix early exit, and the
    plain form past 2048) must equal the oracle's select_plain exactly -- ties
    to the lower index (router.hpp:96-108), force_block (:111-121)."""
    import torch
    rng = np.random.default_rng(N + fd)
    d = 64
    qb = rng.integers(-2, 3, size=(N, d)).astype(np.float64)
    kb = rng.integers(-1, 2, size=(N, d)).astype(np.float64)
    kb[rng.random(N) < 0.5] = kb[0]          # half the key blocks identical: one huge tie class
    qb[: N // 3] = 0.0                        # all-tied rows (every score 0)
    for k in sorted({1, max(1, N // 7), N // 2, N - 1, N}):
        ref = oracle_mod.select_plain(qb, kb, k, 1.0, force_diagonal=fd)
        got = P.select_topk_plain(torch.tensor(qb, dtype=torch.float32).cuda()[None],
                                  torch.tensor(kb, dtype=torch.float32).cuda()[None], k, 1.0,
                                  force_diagonal=fd).cpu().numpy()[0]
        assert np.array_equal(got, ref), (N, k, fd, np.where((got != ref).any(1))[0][:5])


# ------------------------------------------------------------ fused forward --
SHAPES = [
    ("gaussian", 2, 1024, 128, 0.75),
    ("clustered", 2, 1024, 64, 0.75),
    ("gaussian", 1, 1000, 128, 0.5),      # ragged: 15 full blocks + 40 rows
    ("clustered", 2, 2048, 128, 0.875),
    ("clustered", 1, 4096, 64, 0.75),     # BASELINE configs[0] head dim
    ("gaussian", 1, 320, 128, 0.0),       # full coverage
    ("clustered", 1, 8256, 128, 0.875),   # odd N (129 blocks)
]


@pytest.mark.parametrize("variant", ["hybrid", "zeroth", "sparse_only", "global_centroid"])
@pytest.mark.parametrize("kind,H,L,d,r", SHAPES)
def test_fused_matches_oracle(P, oracle_mod, variant, kind, H, L, d, r):
    O = oracle_mod
    q, k, v = O.gen(kind, 0, H, L, d)
    V = {"hybrid": P.PisaVariant.Hybrid, "zeroth": P.PisaVariant.Zeroth,
         "sparse_only": P.PisaVariant.SparseOnly, "global_centroid": P.PisaVariant.GlobalCentroid}
    out, ex = run_fwd(P, q, k, v, sparsity=r, variant=V[variant])
    scale = d ** -0.5
    for h in range(H):
        st = O.block_stats(k[h], v[h])
        ref_sel = O.select_plain(O.query_means(q[h]), st[0], ex["selected"].shape[-1], scale)
        assert np.array_equal(ex["selected"][h], ref_sel)
        ref, m, ell, et = O.pisa_attention(q[h], k[h], v[h], ex["selected"][h], st, scale, variant)
        check_close(out[h], ref)
        # diagnostics (PisaOutput.denom / ell_tail): shift-invariant products
        den_gpu = ex["ell"][h].astype(np.float64) * np.exp(ex["row_max"][h].astype(np.float64))
        np.testing.assert_allclose(den_gpu, ell * np.exp(m), rtol=2e-2)
        if variant != "sparse_only" and r > 0:
            et_gpu = ex["ell_tail"][h].astype(np.float64) * np.exp(ex["row_max"][h].astype(np.float64))
            np.testing.assert_allclose(et_gpu, et * np.exp(m), rtol=3e-2)


@pytest.mark.parametrize("L,d,r", [(1, 128, 0.5), (17, 64, 0.5), (64, 128, 0.0), (65, 128, 0.5),
                                   (127, 64, 0.5), (130, 128, 0.6), (200, 64, 0.99)])
def test_tiny_and_ragged_lengths(P, oracle_mod, L, d, r):
    """Degenerate shapes: one block (N = 1), a last block of 1 row (L = 65),
    N = 2..4, k = 1 (r = 0.99), all variants' code paths through Hybrid."""
    O = oracle_mod
    q, k, v = O.gen("gaussian", 7, 2, L, d)
    out, ex = run_fwd(P, q, k, v, sparsity=r)
    scale = d ** -0.5
    for h in range(2):
        st = O.block_stats(k[h], v[h])
        ref_sel = O.select_plain(O.query_means(q[h]), st[0], ex["selected"].shape[-1], scale)
        assert np.array_equal(ex["selected"][h], ref_sel)
        ref = O.pisa_attention(q[h], k[h], v[h], ex["selected"][h], st, scale, "hybrid")[0]
        assert np.isfinite(out[h]).all()
        assert float(np.abs(out[h] - ref).max()) <= ATOL


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*_h*_l*.npz"))),
                         ids=lambda p: os.path.basename(p)[:-4])
def test_fused_matches_reference_golden(P, path):
    """Against the reference's own pisa_multihead outputs (fixtures made from the
    unmodified library): plan bit-exact, outputs within the bf16 tolerance."""
    f = np.load(path)
    fd = bool(f["force_diagonal"])
    for variant, pv in (("hybrid", P.PisaVariant.Hybrid), ("zeroth", P.PisaVariant.Zeroth),
                        ("sparse_only", P.PisaVariant.SparseOnly),
                        ("global_centroid", P.PisaVariant.GlobalCentroid)):
        out, ex = run_fwd(P, f["q"], f["k"], f["v"], sparsity=float(f["r"]), variant=pv,
                          force_diagonal=fd)
        assert np.array_equal(ex["selected"], f["selected"]), variant
        check_close(out, f[f"out_{variant}"].astype(np.float64))


def test_strided_bshd_layout_and_batch(P, oracle_mod):
    """DiT layout [B][L][H][d] through strides, batch 2, against the [H][L][d] run."""
    import torch
    O = oracle_mod
    B, H, L, d = 2, 3, 1088, 128
    q, k, v = O.gen("clustered", 5, B * H, L, d)
    to = lambda x: torch.from_numpy(x).to(torch.bfloat16).cuda().view(B, H, L, d)
    qh, kh, vh = to(q), to(k), to(v)
    ref = P.fwd(qh, kh, vh, sparsity=0.75, out_dtype=torch.float32)
    qs, ks, vs = (x.transpose(1, 2).contiguous() for x in (qh, kh, vh))  # [B][L][H][d]
    out = P.fwd(qs, ks, vs, layout="blhd", sparsity=0.75, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(out.transpose(1, 2), ref)


def test_constant_key_blocks_exact(P, oracle_mod):
    # test_engine.cpp:68-99 on the GPU path: constant key blocks -> tail exact
    O = oracle_mod
    L, d = 1024, 128
    q, k, v = O.gen("gaussian", 0, 1, L, d)
    rng = np.random.default_rng(100)
    for j in range(L // 64):
        k[0, j * 64:(j + 1) * 64] = O.round_bf16(rng.standard_normal(d).astype(np.float32))
    dense = O.dense(q[0], k[0], v[0], d ** -0.5)
    for variant in (P.PisaVariant.Zeroth, P.PisaVariant.Hybrid):
        out, _ = run_fwd(P, q, k, v, sparsity=0.75, variant=variant)
        check_close(out[0], dense, atol=1e-2, cos=0.9999)


def test_literal_phase3(P, oracle_mod):
    O = oracle_mod
    q, k, v = O.gen("clustered", 4, 1, 1024, 128)
    z, _ = run_fwd(P, q, k, v, sparsity=0.75, variant=P.PisaVariant.Zeroth)
    dflt, _ = run_fwd(P, q, k, v, sparsity=0.75, variant=P.PisaVariant.Hybrid)
    lit, _ = run_fwd(P, q, k, v, sparsity=0.75, variant=P.PisaVariant.Hybrid, literal_phase3=True)
    np.testing.assert_allclose(dflt - z, 64.0 * (lit - z), rtol=0, atol=5e-3)


def test_bitwise_deterministic_and_identical_heads(P, oracle_mod):
    # test_engine.cpp:211-257: identical heads -> identical outputs; run-to-run bits
    O = oracle_mod
    q, k, v = O.gen("clustered", 0, 1, 2048, 128)
    q2, k2, v2 = (np.concatenate([x, x]) for x in (q, k, v))
    a, ea = run_fwd(P, q2, k2, v2, sparsity=0.5)
    b, eb = run_fwd(P, q2, k2, v2, sparsity=0.5)
    assert np.array_equal(a, b) and np.array_equal(ea["selected"], eb["selected"])
    assert np.array_equal(a[0], a[1])


def test_numerical_overflow_reported(P):
    # test_engine.cpp:296-308: huge V overflows the accumulator -> NumericalOverflow
    import torch
    q = torch.randn((1, 1, 256, 64), device="cuda").bfloat16()
    k = torch.randn((1, 1, 256, 64), device="cuda").bfloat16()
    v = torch.full((1, 1, 256, 64), 3.0e38, device="cuda").bfloat16()
    with pytest.raises(P.NumericalOverflow):
        P.fwd(q, k, v, topk=1, check_finite=True, out_dtype=torch.float32)


def test_numerical_overflow_through_multihead_and_host_path(P):
    """check_output_finite (engine.hpp:83-93, :368) on the reference-facing
    entries: pisa_multihead raises NumericalOverflow; the host-buffer forward
    ORs the device flag over all staged chunks and reports it after its final
    synchronisation; with the check off the call returns the non-finite output."""
    import torch
    H, L, d = 3, 320, 64
    q, k = (torch.randn((1, H, L, d), device="cuda").bfloat16() for _ in range(2))
    v = torch.randn((1, H, L, d), device="cuda").bfloat16()
    v[0, 1] = 3.0e38  # one head of three overflows
    with pytest.raises(P.NumericalOverflow):
        P.pisa_multihead(P.TensorBundle(q[0], k[0], v[0]), 0.75, P.RouterOptions(), P.PisaVariant.Hybrid,
                         P.AttentionConfig(), True)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    ho = torch.empty((1, H, L, d), dtype=torch.bfloat16).pin_memory()
    with pytest.raises(P.NumericalOverflow):
        P.fwd_host(hq, hk, hv, ho, sparsity=0.75, check_finite=True)
    P.fwd_host(hq, hk, hv, ho, sparsity=0.75)  # unchecked: returns
    assert not torch.isfinite(ho[0, 1].float()).all() and torch.isfinite(ho[0, 0].float()).all()
    v[0, 1] = 1.0
    hv = v.cpu().pin_memory()
    P.fwd_host(hq, hk, hv, ho, sparsity=0.75, check_finite=True)  # the flag was reset
    assert torch.isfinite(ho.float()).all()


def test_output_and_engine_input_validation(P, oracle_mod):
    """fwd() checks O (shape, device, dtype, 16-byte rows) and pisa_streaming /
    pisa_reference check the plan and statistics against the inputs
    (check_engine_inputs, engine.hpp:61-80) instead of reading past buffers."""
    import torch
    O = oracle_mod
    q, k, v = (dev_bf16(x) for x in O.gen("gaussian", 1, 1, 512, 128))
    with pytest.raises(P.InvalidDimension):
        P.fwd(q, k, v, torch.empty((1, 1, 448, 128), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(P.Unsupported):
        P.fwd(q, k, v, torch.empty_like(q, dtype=torch.float16))
    wide = torch.zeros((1, 1, 512, 132), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(P.InvalidDimension):  # row stride 132 bf16 = 264 B: not 16-byte rows
        P.fwd(q, k, v, wide[..., :128])
    wide = torch.zeros((1, 1, 512, 136), dtype=torch.bfloat16, device="cuda")
    P.fwd(q, k, v, wide[..., :128], sparsity=0.75)  # 272 B rows: fine, padding untouched
    torch.cuda.synchronize()
    assert not wide[..., 128:].any() and torch.equal(wide[..., :128], P.fwd(q, k, v, sparsity=0.75))
    st = P.compute_prepare(q[0], k[0], v[0])
    sel = P.select_topk_plain(st.q_bar, st.k_bar, 2, 128 ** -0.5)
    out, _ = P.pisa_streaming(q[0], k[0], v[0], sel, st)
    with pytest.raises(P.InvalidDimension):  # plan for fewer query blocks
        P.pisa_streaming(q[0], k[0], v[0], sel[:, :, :7], st)
    with pytest.raises(P.InvalidDimension):  # statistics of another length
        P.pisa_streaming(q[0], k[0], v[0], sel,
                         P.BlockStatistics(7, 64, 128, st.k_bar[:, :, :7], st.v_hat[:, :, :7], st.h_bar))
    with pytest.raises(P.InvalidDimension):  # block size mismatch
        P.pisa_reference(q[0], k[0], v[0], sel, P.BlockStatistics(8, 32, 128, st.k_bar, st.v_hat, st.h_bar),
                         P.PisaVariant.Zeroth)


def test_literal_phase3_only_on_the_streaming_path(P, oracle_mod):
    """literal_phase3 divides the Phase-3 weight by B on the streaming path only
    (engine.hpp:345-346); pisa_reference and GlobalCentroid ignore it
    (engine.hpp:194-209), and pisa_multihead(use_streaming=False) with it."""
    import torch
    O = oracle_mod
    q, k, v = (dev_bf16(x, False) for x in O.gen("clustered", 4, 1, 1024, 128))
    st = P.compute_prepare(q, k, v)
    sel = P.select_topk_plain(st.q_bar, st.k_bar, 4, 128 ** -0.5)
    lit_cfg = P.AttentionConfig(literal_phase3=True)
    f32 = dict(out_dtype=torch.float32)
    a, _ = P.pisa_reference(q, k, v, sel, st, P.PisaVariant.Hybrid, lit_cfg, **f32)
    b, _ = P.pisa_reference(q, k, v, sel, st, P.PisaVariant.Hybrid, **f32)
    c, _ = P.pisa_streaming(q, k, v, sel, st, lit_cfg, **f32)
    assert torch.equal(a, b) and not torch.equal(b, c)
    g0, _ = P.pisa_reference(q, k, v, sel, st, P.PisaVariant.GlobalCentroid, lit_cfg, **f32)
    g3, _ = P.pisa_reference(q, k, v, sel, st, P.PisaVariant.GlobalCentroid, **f32)
    g1 = P.fwd(q[None], k[None], v[None], topk=4, variant=P.PisaVariant.GlobalCentroid, literal_phase3=True,
               **f32)
    g2 = P.fwd(q[None], k[None], v[None], topk=4, variant=P.PisaVariant.GlobalCentroid, **f32)
    assert torch.equal(g1, g2) and torch.equal(g0, g3)
    bundle = P.TensorBundle(q, k, v)
    r_ref = P.pisa_multihead(bundle, 0.75, P.RouterOptions(), P.PisaVariant.Hybrid, lit_cfg, False, **f32)
    r_dflt = P.pisa_multihead(bundle, 0.75, P.RouterOptions(), P.PisaVariant.Hybrid, P.AttentionConfig(), True,
                              **f32)
    r_lit = P.pisa_multihead(bundle, 0.75, P.RouterOptions(), P.PisaVariant.Hybrid, lit_cfg, True, **f32)
    assert torch.equal(r_ref.heads[0].output, r_dflt.heads[0].output)
    assert not torch.equal(r_lit.heads[0].output, r_dflt.heads[0].output)


def test_concurrent_streams_do_not_share_workspace(P):
    """Forwards of different shapes enqueued back to back on two streams of one
    context (no synchronisation in between) equal the same forwards run alone:
    each stream has its own workspace."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    xa = [torch.randn((1, 4, 4096, 128), generator=g, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    xb = [torch.randn((1, 2, 2000, 64), generator=g, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    ref_a = P.fwd(*xa, sparsity=0.875)
    ref_b = P.fwd(*xb, sparsity=0.5)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            oa = P.fwd(*xa, sparsity=0.875)
        with torch.cuda.stream(s2):
            ob = P.fwd(*xb, sparsity=0.5)
        outs.append((oa, ob))
    torch.cuda.synchronize()
    for oa, ob in outs:
        assert torch.equal(oa, ref_a) and torch.equal(ob, ref_b)


def test_attention_with_given_plan_and_validation(P, oracle_mod):
    """pisa_streaming / pisa_reference with the REFERENCE plan and fp32 stats,
    and SelectionPlan::validate semantics for a bad plan (router.hpp:50-70)."""
    import torch
    O = oracle_mod
    q, k, v = O.gen("clustered", 3, 1, 1024, 128)
    st = O.block_stats(k[0], v[0])
    sel = O.select_plain(O.query_means(q[0]), st[0], 4, 128 ** -0.5)
    stats = P.BlockStatistics(16, 64, 128, torch.tensor(st[0], dtype=torch.float32).cuda()[None, None],
                              torch.tensor(st[1], dtype=torch.float32).cuda()[None, None],
                              torch.tensor(st[2], dtype=torch.float32).cuda()[None, None])
    out, ex = P.pisa_streaming(dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False),
                               torch.tensor(sel).cuda()[None, None], stats,
                               out_dtype=torch.float32)
    ref, *_ = O.pisa_attention(q[0], k[0], v[0], sel, st, 128 ** -0.5, "hybrid")
    check_close(out[0, 0].cpu().numpy(), ref)
    bad = sel.copy()
    bad[3] = bad[3][::-1]
    with pytest.raises(P.InvalidSparsity):
        P.pisa_streaming(dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False),
                         torch.tensor(bad.copy()).cuda()[None, None], stats)


@pytest.mark.parametrize("B,H,L", [(1, 5, 2048), (2, 23, 512), (1, 40, 320)])
def test_host_path_equals_device_path(P, B, H, L):
    """pisa_b200_fwd_host (staged chunks: a remainder, full chunks, a 2 / 1
    tail from 33 (b, h) units up) equals the device-resident forward."""
    import torch
    d = 128
    x = [torch.randn((B, H, L, d), device="cuda").bfloat16() for _ in range(3)]
    dev_out = P.fwd(*x, sparsity=0.875)
    hx = [t.cpu().pin_memory() for t in x]
    ho = torch.empty((B, H, L, d), dtype=torch.bfloat16).pin_memory()
    P.fwd_host(*hx, ho, sparsity=0.875)
    torch.cuda.synchronize()
    assert torch.equal(ho, dev_out.cpu())


def test_multihead_api_mirror(P, oracle_mod):
    """pisa_multihead(bundle, r, RouterOptions, variant, cfg, use_streaming) result
    structure and values (engine.hpp:392-470)."""
    import torch
    O = oracle_mod
    q, k, v = O.gen("clustered", 2, 2, 1024, 128)
    b = P.TensorBundle(dev_bf16(q, False), dev_bf16(k, False), dev_bf16(v, False))
    res = P.pisa_multihead(b, 0.75, P.RouterOptions(), P.PisaVariant.Hybrid, P.AttentionConfig(),
                           True, out_dtype=torch.float32)
    assert res.k == 4 and res.num_blocks == 16 and res.sparsity_realized == pytest.approx(0.75)
    assert len(res.heads) == 2 and len(res.plans) == 2
    ref = O.multihead(q, k, v, r=0.75)
    for h in range(2):
        assert np.array_equal(res.plans[h].selected.cpu().numpy(), ref["selected"][h])
        check_close(res.heads[h].output.cpu().numpy(), ref["out"][h])
        np.testing.assert_allclose(res.heads[h].tail_mass.cpu().numpy(),
                                   64 * ref["ell_tail"][h] * np.exp(ref["row_max"][h]), rtol=3e-2)
    with pytest.raises(P.BlockDivisibility):
        P.pisa_multihead(P.TensorBundle(*(t[:, :1000] for t in (b.q, b.k, b.v))), 0.75,
                         ragged=False)
    with pytest.raises(P.Unsupported):  # row-level routing stays off the GPU path
        P.pisa_multihead(b, 0.75, P.RouterOptions(row_level=True))


# ------------------------------------------------------- full-size shapes ---
@pytest.mark.parametrize("name,L,r", [("wan2.1-14b", 75600, 0.875), ("wan2.1-1.3b", 32760, 0.875),
                                      ("hunyuan", 118800, 0.9)])
def test_full_size_head_parity(P, oracle_mod, name, L, r):
    """One head at a BASELINE shape (ragged L): plan exact on every query block,
    outputs vs the oracle on a spread of query blocks, and determinism."""
    import torch
    O = oracle_mod
    d = 128
    q, k, v = O.gen("gaussian", 0, 1, L, d)
    out, ex = run_fwd(P, q, k, v, sparsity=r)
    N = (L + 63) // 64
    scale = d ** -0.5
    st = O.block_stats(k[0], v[0])
    oqb = O.query_means(q[0])
    nbad, non_tie = _near_tie_swaps(O, oqb, st[0], ex["selected"][0], ex["selected"].shape[-1], scale)
    assert not non_tie and nbad <= max(1, N // 500), (nbad, non_tie)
    blocks = sorted(set([0, 1, N // 3, N // 2, N - 2, N - 1]))
    for i in blocks:
        ref, *_ = O.pisa_attention(q[0], k[0], v[0], ex["selected"][0], st, scale, "hybrid",
                                   qb0=i, qb1=i + 1)
        rows = slice(i * 64, min(L, (i + 1) * 64))
        check_close(out[0][rows], ref[rows])
    out2, _ = run_fwd(P, q, k, v, sparsity=r)
    assert np.array_equal(out, out2)
    assert np.isfinite(out).all()
    torch.cuda.empty_cache()


def test_cpp_shim_drop_in(P, oracle_mod, tmp_path):
    """A reference-style C++ caller (tests/cpp/shim_demo.cpp) compiled against
    include/pisa_b200.hpp and linked to the C ABI library: pisa_multihead on one
    and on two "devices", the step functions (compute_block_stats ->
    compute_global_stats -> query_block_means -> select_topk_plain ->
    pisa_streaming / pisa_reference), NumericalOverflow, the error classes and
    the reference generators -- all checked here against the oracle / the
    reference's own values."""
    import subprocess
    O = oracle_mod
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "shim_demo"
    subprocess.run(["g++", "-std=c++17", "-O2", "-pthread", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "shim_demo.cpp"),
                    "-L", os.path.join(root, "paper_2602_01077_b200", "lib"), "-lpisa_b200",
                    "-Wl,-rpath," + os.path.join(root, "paper_2602_01077_b200", "lib"),
                    "-o", str(exe)], check=True)
    H, L, d, r = 2, 1000, 128, 0.75
    q, k, v = O.gen("clustered", 9, H, L, d)
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        for x in (q, k, v):
            f.write(np.ascontiguousarray(x, np.float32).tobytes())
    res = subprocess.run([str(exe), str(inp), str(tmp_path), str(H), str(L), str(d), str(r)],
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    for check in ("multidevice ok", "BlockDivisibility ok", "steps ok", "covariance ok",
                  "InvalidDimension ok", "NumericalOverflow ok", "gen ok"):
        assert check in res.stdout, (check, res.stdout)
    out = np.fromfile(tmp_path / "multihead_out.bin", np.float32).reshape(H, L, d)
    N = 16
    kk = int(res.stdout.split()[0])
    plan = np.fromfile(tmp_path / "multihead_plan.bin", np.int32).reshape(H, N, kk)
    ref = O.multihead(q, k, v, r=r)
    assert np.array_equal(plan, ref["selected"])
    for h in range(H):
        check_close(out[h], ref["out"][h])
    # step functions on head 0 floored to 960 rows vs the oracle's steps
    Lf, Nf = 960, 15
    kf = O.sparsity_to_k(r, Nf)[0]
    kb, vh, hb, kg = O.block_stats(k[0, :Lf], v[0, :Lf])
    qb = O.query_means(q[0, :Lf])
    stats = np.fromfile(tmp_path / "steps_stats.bin", np.float64)
    g_kb, g_vh, g_qb = (stats[i * Nf * d:(i + 1) * Nf * d].reshape(Nf, d) for i in range(3))
    g_hb = stats[3 * Nf * d:].reshape(d, d)
    np.testing.assert_allclose(g_kb, kb, rtol=0, atol=1e-6)
    np.testing.assert_allclose(g_vh, vh, rtol=0, atol=1e-5)
    np.testing.assert_allclose(g_qb, qb, rtol=0, atol=1e-6)
    assert np.abs(g_hb - hb).max() <= 1e-4 * max(1.0, np.abs(hb).max())
    splan = np.fromfile(tmp_path / "steps_plan.bin", np.int32).reshape(Nf, kf)
    assert np.array_equal(splan, O.select_plain(qb, kb, kf, d ** -0.5))
    sout = np.fromfile(tmp_path / "steps_out.bin", np.float32).reshape(Lf, d)
    ref_s = O.pisa_attention(q[0, :Lf], k[0, :Lf], v[0, :Lf], splan, (kb, vh, hb, kg), d ** -0.5,
                             "hybrid")[0]
    check_close(sout, ref_s)
    # the reference's generator values (gen_gaussian<float>(42, 2, 64, 8, 1.0))
    gen = np.fromfile(tmp_path / "gen.bin", np.float32).reshape(3, 2, 64, 8)
    gq, gk, gv = O.gen("gaussian", 42, 2, 64, 8, bf16=False)
    assert np.array_equal(gen[0], gq) and np.array_equal(gen[1], gk) and np.array_equal(gen[2], gv)


# ----------------------------------- (head x query-block range) sharding (§8e) --
def test_qrange_pieces_reassemble(P, oracle_mod):
    """Eight simulated ranks over 3 heads (ragged L = 1000, N = 16): each runs
    pisa_b200_fwd_qrange on its (head, query-block range) pieces; the assembled
    output equals the full call's to rounding (pieces may pair query blocks
    differently, which moves the online softmax's lazy-rescale points), rows
    outside a range are untouched."""
    import torch

    from paper_2602_01077_b200.sharding import fwd_pieces, unit_qblock_pieces
    q, k, v = (dev_bf16(x) for x in oracle_mod.gen("clustered", 21, 3, 1000, 128))
    kw = dict(sparsity=0.75)
    full = P.fwd(q, k, v, **kw)
    out = torch.full_like(full, float("nan"))
    for r in range(8):
        fwd_pieces(q, k, v, out, unit_qblock_pieces(1, 3, 16, 8, r), **kw)
    torch.cuda.synchronize()
    assert not torch.isnan(out).any()
    assert (out.float() - full.float()).abs().max().item() <= 4e-3
    # a single range: rows outside it are untouched, rows inside equal the full call
    part = torch.zeros_like(full)
    P.fwd(q, k, v, part, q_blocks=(5, 11), **kw)
    torch.cuda.synchronize()
    assert (part[:, :, 5 * 64:11 * 64].float() - full[:, :, 5 * 64:11 * 64].float()).abs().max().item() <= 4e-3
    assert not part[:, :, :5 * 64].any() and not part[:, :, 11 * 64:].any()
    # the ragged last block alone, and a lone first block
    for rng in ((15, 16), (0, 1)):
        part.zero_()
        P.fwd(q, k, v, part, q_blocks=rng, **kw)
        torch.cuda.synchronize()
        sl = slice(rng[0] * 64, rng[1] * 64)
        assert (part[:, :, sl].float() - full[:, :, sl].float()).abs().max().item() <= 4e-3
    # odd-length ranges: the last block's would-be partner lies outside the
    # range and must not be written (also with f32 output and diagnostics)
    for rng in ((0, 1), (4, 7), (9, 12)):
        part = torch.zeros_like(full)
        P.fwd(q, k, v, part, q_blocks=rng, **kw)
        part32 = torch.zeros(full.shape, dtype=torch.float32, device=full.device)
        P.fwd(q, k, v, part32, q_blocks=rng, out_dtype=torch.float32, **kw)
        torch.cuda.synchronize()
        sl = slice(rng[0] * 64, rng[1] * 64)
        for o in (part, part32):
            assert (o[:, :, sl].float() - full[:, :, sl].float()).abs().max().item() <= 4e-3
            assert not o[:, :, :rng[0] * 64].any() and not o[:, :, rng[1] * 64:].any(), rng
    for bad in ((3, 3), (-1, 4), (0, 17), (12, 5)):
        with pytest.raises(P.InvalidDimension):
            P.fwd(q, k, v, part, q_blocks=bad, **kw)


def test_torchrun_world2_same_gpu(tmp_path):
    """The multi-rank path end to end under torchrun (world 2, both ranks on
    GPU 0, gloo): head sharding + all_gather reproduces the single-rank output
    bit for bit (a head's result does not depend on the other heads in the
    launch); (head x query-block) pieces + the pieces gather agree to rounding."""
    import json
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "dist.json"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "tests", "dist_fwd_worker.py"), str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.loads(out.read_text())
    assert res["world"] == 2 and res["heads_bit_equal"], res
    assert res["pieces_max_abs_diff"] <= 4e-3, res


def test_pairing_modes_agree_and_fewer_tiles(P, oracle_mod):
    """Overlap-aware query-block pairing only regroups work: the plan is bitwise
    identical with it forced on or off, the outputs agree to rounding (a block's
    key blocks are grouped into super-tiles differently, so the online softmax's
    lazy-rescale points move), and on multi-cluster routing where alike blocks
    are far apart it executes fewer union tiles."""
    import torch
    q, k, v = (dev_bf16(x) for x in oracle_mod.gen("clustered", 31, 2, 4096, 128))
    # shuffle query blocks so that blocks routing alike are not neighbours
    perm = torch.randperm(64, generator=torch.Generator().manual_seed(3))
    q = q.view(1, 2, 64, 64, 128)[:, :, perm].reshape(1, 2, 4096, 128).contiguous()
    ctx = P.Context.get(0)
    outs, tiles = [], []
    try:
        for mode in (0, 2):
            ctx.set_pairing(mode)
            ctx.set_profiling(True)
            ctx.fused_tiles()
            o, ex = P.fwd(q, k, v, sparsity=0.875, return_plan=True)
            torch.cuda.synchronize()
            tiles.append(ctx.fused_tiles())
            ctx.set_profiling(False)
            outs.append((o, ex["selected"]))
    finally:
        ctx.set_pairing(1)
        ctx.set_profiling(False)
    assert torch.equal(outs[0][1], outs[1][1])
    assert (outs[0][0].float() - outs[1][0].float()).abs().max().item() <= 4e-3
    assert tiles[1] < tiles[0], tiles
    with pytest.raises(P.InvalidDimension):
        ctx.set_pairing(3)


@pytest.mark.parametrize("kind", ["gaussian", "clustered"])
def test_pairing_full_search(P, oracle_mod, kind, monkeypatch):
    """K2c over the whole query-block range (default: overlap matrix on tcgen05
    kind::i8, nearest-first ties) against the +-48 window
    (PISA_B200_PAIR_FULL=0): the same plan, outputs equal to rounding, and on
    independent (gaussian) routing fewer union tiles."""
    import torch
    q, k, v = (dev_bf16(x) for x in oracle_mod.gen(kind, 5, 2, 64000, 128))
    ctx = P.Context.get(0)
    res = {}
    try:
        ctx.set_pairing(2)
        for full in ("1", "0"):
            monkeypatch.setenv("PISA_B200_PAIR_FULL", full)
            ctx.set_profiling(True)
            ctx.fused_tiles()
            o, ex = P.fwd(q, k, v, sparsity=0.875, return_plan=True)
            torch.cuda.synchronize()
            res[full] = (o, ex["selected"], ctx.fused_tiles())
            ctx.set_profiling(False)
    finally:
        ctx.set_pairing(1)
        ctx.set_profiling(False)
    assert torch.equal(res["1"][1], res["0"][1])
    assert (res["1"][0].float() - res["0"][0].float()).abs().max().item() <= 4e-3
    if kind == "gaussian":
        assert res["1"][2] < res["0"][2], (res["1"][2], res["0"][2])


@pytest.mark.parametrize("q_blocks,N", [((1, 130), 131), ((3, 300), 300), ((0, 257), 257)])
def test_pairing_full_search_ranges(P, oracle_mod, q_blocks, N):
    """The full-range pairing search on query-block ranges with an odd first
    block or an odd N (the overlap matrix's row stores lose 4-byte alignment):
    forced on, the range's output equals the unpaired range's to rounding and the
    rest of O is untouched."""
    import torch
    L = N * 64 - 17
    q, k, v = (dev_bf16(x) for x in oracle_mod.gen("gaussian", 8, 1, L, 128))
    ctx = P.Context.get(0)
    outs = []
    try:
        for mode in (2, 0):
            ctx.set_pairing(mode)
            out = torch.zeros_like(q)
            P.fwd(q, k, v, out, sparsity=0.75, ctx=ctx, q_blocks=q_blocks)
            torch.cuda.synchronize()
            outs.append(out)
    finally:
        ctx.set_pairing(1)
    r0, r1 = q_blocks[0] * 64, min(L, q_blocks[1] * 64)
    assert (outs[0][..., :r0, :] == 0).all() and (outs[0][..., r1:, :] == 0).all()
    assert (outs[0].float() - outs[1].float()).abs().max().item() <= 4e-3


@pytest.mark.parametrize("L,d", [(1024, 128), (1000, 64)])
def test_dense_online_matches_reference(P, oracle_mod, L, d):
    """dense_online (attention.hpp:186-193), the baseline PISA is timed against,
    vs the reference's own dense_online through the oracle library."""
    import torch
    q, k, v = oracle_mod.gen("gaussian", 9, 1, L, d)
    o = P.dense_online(*(torch.from_numpy(x[0]).to(torch.bfloat16).cuda() for x in (q, k, v)))
    ref = oracle_mod.dense(*(torch.from_numpy(x[0]).to(torch.bfloat16).float().numpy() for x in (q, k, v)),
                           d ** -0.5)
    check_close(o.float().cpu().numpy(), ref)


def _random_configs(n, seed=2602):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        out.append(dict(kind=str(rng.choice(["gaussian", "clustered"])), H=int(rng.integers(1, 4)),
                        L=int(rng.integers(65, 5000)), d=int(rng.choice([64, 128])),
                        r=float(rng.choice([0.5, 0.75, 0.875, 0.95])),
                        variant=str(rng.choice(["hybrid", "zeroth", "sparse_only", "global_centroid"])),
                        router=str(rng.choice(["plain", "covariance"])), pairing=int(rng.choice([0, 2])),
                        layout=str(rng.choice(["bhld", "blhd"])), seed=int(rng.integers(0, 1 << 16))))
    return out


@pytest.mark.parametrize("cfg", _random_configs(32), ids=lambda c: "-".join(str(v) for v in c.values()))
def test_randomized_shapes_match_oracle(P, oracle_mod, cfg):
    """Seeded random shapes (ragged L, d 64 / 128), variants, routers, layouts
    and pairing modes: the fused output equals the oracle's attention on the
    GPU's own plan (max abs <= 2e-2, cosine >= 0.999)."""
    import torch
    O = oracle_mod
    V = {"hybrid": P.PisaVariant.Hybrid, "zeroth": P.PisaVariant.Zeroth,
         "sparse_only": P.PisaVariant.SparseOnly, "global_centroid": P.PisaVariant.GlobalCentroid}
    q, k, v = O.gen(cfg["kind"], cfg["seed"], cfg["H"], cfg["L"], cfg["d"])
    to = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda().unsqueeze(0)
    qd, kd, vd = to(q), to(k), to(v)
    if cfg["layout"] == "blhd":
        qd, kd, vd = (t.transpose(1, 2).contiguous() for t in (qd, kd, vd))
    router = P.RouterStrategy.CovarianceAware if cfg["router"] == "covariance" else P.RouterStrategy.Plain
    ctx = P.Context.get(0)
    ctx.set_pairing(cfg["pairing"])
    try:
        out, ex = P.fwd(qd, kd, vd, layout=cfg["layout"], out_dtype=torch.float32, return_plan=True,
                        sparsity=cfg["r"], variant=V[cfg["variant"]], router=router)
        torch.cuda.synchronize()
    finally:
        ctx.set_pairing(1)
    if cfg["layout"] == "blhd":
        out = out.transpose(1, 2)
    out = out[0].cpu().numpy()
    sel = ex["selected"][0].cpu().numpy()
    scale = cfg["d"] ** -0.5
    for h in range(cfg["H"]):
        st = O.block_stats(k[h], v[h])
        ref = O.pisa_attention(q[h], k[h], v[h], sel[h], st, scale, cfg["variant"])[0]
        check_close(out[h], ref)


@pytest.mark.parametrize("router", ["plain", "covariance"])
def test_fwd_cuda_graph_capture_replays_bit_identical(P, router):
    """P.fwd is stream-ordered with no host syncs (profiling and check_finite
    off), so a CUDA graph captures the whole forward; the replay recomputes
    from the current inputs and matches the eager call bit for bit."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(77)
    q, k, v = (torch.randn((1, 3, 2000, 128), generator=g, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    kw = dict(sparsity=0.75, router=P.RouterStrategy.CovarianceAware if router == "covariance"
              else P.RouterStrategy.Plain)
    P.fwd(q, k, v, out, **kw)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        P.fwd(q, k, v, out, **kw)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        P.fwd(q, k, v, out, **kw)
    q.copy_(torch.randn(q.shape, generator=g, device="cuda", dtype=torch.bfloat16))  # new inputs, same buffers
    ref = P.fwd(q, k, v, **kw)
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_block_norms_full_length_head_against_fp64_svd(P):
    """K1c at BASELINE scale: one Wan2.1-14B-length head (1182 blocks, ragged
    last block). Lanczos must be converged on every block, including slow-gap
    ones (20 steps leave some 0.8% off): M_j within 2e-6 of sigma_max(H_j -
    H_bar) from an fp64 SVD."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(31)
    L, d = 75600, 128
    q, k, v = (torch.randn((1, 1, L, d), generator=g, device="cuda").bfloat16() for _ in range(3))
    m = P.block_norms(q, k, v)[0, 0].double()
    kf, vf = k[0, 0].double(), v[0, 0].double()
    N = -(-L // 64)
    H = torch.stack([(kf[j * 64:(j + 1) * 64] - kf[j * 64:(j + 1) * 64].mean(0)).T @ vf[j * 64:(j + 1) * 64]
                     for j in range(N)])
    exact = torch.linalg.matrix_norm(H - H.mean(0), ord=2)
    rel = ((m - exact).abs() / exact).max().item()
    assert rel < 2e-6, rel
