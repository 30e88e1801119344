"""DiT integration surface (paper_2602_01077_b200/dit.py): the paper's warmup
policy and presets, dispatch, layouts and MMDiT
joint text+image attention. CPU tests cover the policy; GPU tests the paths."""
import numpy as np
import pytest


def test_presets_follow_the_paper():
    import paper_2602_01077_b200 as P
    # video: 1 dense layer + 15 / 10 dense steps; image: 4 dense layers, covariance router
    assert P.PRESETS["wan2.1-1.3b"].policy == P.WarmupPolicy(1, 15)
    assert P.PRESETS["wan2.1-14b"].policy == P.WarmupPolicy(1, 10)
    assert P.PRESETS["hunyuanvideo-13b"].policy == P.WarmupPolicy(1, 10)
    for img in ("sd3.5-medium", "sd3.5-turbo", "flux.1-schnell", "flux.1-dev"):
        assert P.PRESETS[img].policy == P.WarmupPolicy(4, 0)
        assert P.PRESETS[img].router == P.RouterStrategy.CovarianceAware
    assert all(p.density == 0.125 for p in P.PRESETS.values())


@pytest.mark.parametrize("layer,step,dense", [(0, 50, True), (1, 9, True), (1, 10, False),
                                              (5, 30, False), (None, 3, True), (2, None, False)])
def test_warmup_policy(layer, step, dense):
    import paper_2602_01077_b200 as P
    assert P.WarmupPolicy(1, 10).is_dense(layer, step) == dense
    assert not P.WarmupPolicy().is_dense(0, 0)


def test_bad_arguments():
    import paper_2602_01077_b200 as P
    with pytest.raises(P.InvalidSparsity):
        P.PisaAttention(density=0.0)
    with pytest.raises(P.InvalidDimension):
        P.PisaAttention(layout="lbhd")
    with pytest.raises(KeyError):
        P.PisaAttention.from_preset("sd1.5")


@pytest.mark.gpu
def test_dispatch_and_layout(oracle_mod):
    """Warmup calls equal dense SDPA; PISA calls in [B, L, H, d] equal the
    [B, H, L, d] fused forward and the oracle."""
    import torch

    import paper_2602_01077_b200 as P
    O = oracle_mod
    B, H, L, d = 1, 2, 1000, 128  # ragged L
    q, k, v = O.gen("clustered", 11, H, L, d)
    to = lambda x: torch.from_numpy(x).to(torch.bfloat16).cuda().unsqueeze(0).transpose(1, 2).contiguous()
    qd, kd, vd = to(q), to(k), to(v)  # [B, L, H, d]
    attn = P.PisaAttention.from_preset("wan2.1-14b", density=0.25)
    o_dense = attn(qd, kd, vd, layer=0, step=20)
    ref_dense = torch.nn.functional.scaled_dot_product_attention(
        *(t.transpose(1, 2) for t in (qd, kd, vd))).transpose(1, 2)
    assert torch.equal(o_dense, ref_dense)
    o = attn(qd, kd, vd, layer=3, step=20)
    assert attn.calls == {"dense": 1, "pisa": 1}
    o_bhld = P.fwd(*(t.transpose(1, 2).contiguous() for t in (qd, kd, vd)), sparsity=0.75)
    assert torch.equal(o.transpose(1, 2).contiguous(), o_bhld)
    og = o[0].transpose(0, 1).float().cpu().numpy()
    kk = O.sparsity_to_k(0.75, 16)[0]
    for h in range(H):
        st = O.block_stats(k[h], v[h])
        sel = O.select_plain(O.query_means(q[h]), st[0], kk, d ** -0.5)
        ref = O.pisa_attention(q[h], k[h], v[h], sel, st, d ** -0.5, "hybrid")[0]
        assert np.abs(og[h] - ref).max() <= 2e-2


@pytest.mark.gpu
def test_joint_text_image_attention():
    """MMDiT joint attention over [text; image]: equals PISA on the concatenated
    sequence, split back into text and image outputs (FLUX.1 shape, 333 text
    tokens so the joint length is ragged)."""
    import torch

    import paper_2602_01077_b200 as P
    g = torch.Generator(device="cuda").manual_seed(0)
    B, H, d, n_txt, n_img = 1, 4, 128, 333, 4096
    mk = lambda n: torch.randn((B, n, H, d), generator=g, device="cuda", dtype=torch.bfloat16)
    txt = (mk(n_txt), mk(n_txt), mk(n_txt))
    img = (mk(n_img), mk(n_img), mk(n_img))
    attn = P.PisaAttention.from_preset("flux.1-dev")
    o_t, o_i = attn.joint(txt, img, layer=10, step=0)
    assert o_t.shape == (B, n_txt, H, d) and o_i.shape == (B, n_img, H, d)
    q, k, v = (torch.cat([a, b], 1) for a, b in zip(txt, img))
    o = P.fwd(q, k, v, layout="blhd", sparsity=0.875, router=P.RouterStrategy.CovarianceAware)
    assert torch.equal(torch.cat([o_t, o_i], 1), o)
    # warmup layer (layer < 4): dense
    o_t2, o_i2 = attn.joint(txt, img, layer=0, step=0)
    dense = P.dit.dense_attention(q, k, v)
    assert torch.equal(torch.cat([o_t2, o_i2], 1), dense)
