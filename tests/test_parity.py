"""Parity at the BASELINE configurations against the reference itself
(oracle/parity.py; the full sweep with ~64 sampled query blocks per head on
every head is tools/parity.py -> PARITY_r02.json).

Every head's routing plan is compared with the unmodified reference's
select_topk_plain (floored lengths) or the ragged restatement (published
ragged lengths); index sets must be identical apart from near-tie swaps (fp64
gap to the k-th score <= 1e-6 |s_k|, counted and reported). Outputs are
compared on sampled query blocks of a few heads: max-abs <= 2e-2, cosine >=
0.999 (north_star)."""
import json

import pytest

from oracle import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2602_01077_b200 as P
    return P


def _check(res):
    print(json.dumps({k: res[k] for k in ("kind", "L", "density", "rows_differing", "near_tie_swaps",
                                          "non_tie_rows", "max_abs", "min_cos")}))
    assert not res["non_tie_rows"], res["non_tie_rows"]
    assert res["max_abs"] <= parity.ATOL and res["min_cos"] >= parity.COS, (res["max_abs"], res["min_cos"])


@pytest.mark.parametrize("kind", ["gaussian", "clustered"])
@pytest.mark.parametrize("name", ["smoke", "flux"])
def test_image_and_smoke_configs_exact(P, oracle_mod, name, kind):
    """smoke (H=2, L=4096, d=64, 25 %) and FLUX (H=24, L=4608, d=128, 12.5 %):
    every head, every query block's plan and output against the reference."""
    H, L, d, dens = parity.CONFIGS[name]
    _check(parity.run_case(P, kind, H, L, d, dens, nsample=10 ** 6))


@pytest.mark.parametrize("kind", ["gaussian", "clustered"])
@pytest.mark.parametrize("ragged", [False, True], ids=["floored-vs-reference", "ragged-vs-oracle"])
@pytest.mark.parametrize("name", ["wan13b", "wan14b", "hunyuan"])
def test_video_configs_all_heads(P, oracle_mod, name, ragged, kind):
    """Wan2.1-1.3B / Wan2.1-14B / HunyuanVideo: all heads' plans; outputs of two
    heads on 16 query blocks (the first and the last included)."""
    H, L, d, dens = parity.CONFIGS[name]
    Lx = L if ragged else L - L % 64
    _check(parity.run_case(P, kind, H, Lx, d, dens, out_heads=[0, H - 1], nsample=16))


@pytest.mark.parametrize("density", [0.1, 0.25, 0.5])
def test_hunyuan_density_sweep(P, oracle_mod, density):
    """BASELINE configs[4]: the density sweep (10-50 %) at the floored Hunyuan
    length against the reference."""
    H, L, d, _ = parity.CONFIGS["hunyuan"]
    _check(parity.run_case(P, "gaussian", H, L - L % 64, d, density, out_heads=[0], nsample=16))
