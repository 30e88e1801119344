"""PQKV I/O (io.hpp) and the GPU-path CLI harness (tools/pisa_cli.cpp parity):
files byte-compatible with the reference writer/reader, the reference's error
classes and exit codes, flop_model, and the run / sweep / bench commands."""
import json
import os
import struct

import numpy as np
import pytest


@pytest.fixture()
def bundle():
    rng = np.random.default_rng(0)
    return tuple(rng.standard_normal((2, 128, 16)).astype(np.float32) for _ in range(3))


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_pqkv_byte_identical_to_reference_writer(oracle_mod, ref_available, tmp_path, bundle, dtype):
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    from paper_2602_01077_b200 import pqkv
    a, b = str(tmp_path / "ours.pqkv"), str(tmp_path / "ref.pqkv")
    n1 = pqkv.write_bundle(a, *bundle, dtype=dtype)
    n2 = oracle_mod.ref_pqkv_write(b, *bundle, dtype=dtype)
    assert n1 == n2 == os.path.getsize(a)
    assert open(a, "rb").read() == open(b, "rb").read()
    q, k, v, name = pqkv.read_bundle(b)
    assert name == dtype
    for x, y in zip((q, k, v), bundle):
        np.testing.assert_array_equal(x, y)
    rq, rk, rv, tag = oracle_mod.ref_pqkv_read(a)
    assert tag == (1 if dtype == "f32" else 2)
    np.testing.assert_array_equal(rq, bundle[0])


def test_pqkv_bf16_roundtrip_and_version(oracle_mod, ref_available, tmp_path, bundle):
    import torch

    from paper_2602_01077_b200 import pqkv
    p = str(tmp_path / "b.pqkv")
    pqkv.write_bundle(p, *bundle, dtype="bf16")
    raw = open(p, "rb").read()
    assert raw[:4] == b"PQKV" and struct.unpack("<5I", raw[4:24])[:2] == (2, 3)
    q, k, v, name = pqkv.read_bundle(p)
    assert name == "bf16"
    ref = torch.from_numpy(bundle[1]).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(k, ref)
    if ref_available:  # the reference rejects the bf16 extension cleanly
        with pytest.raises(oracle_mod.OracleError) as e:
            oracle_mod.ref_pqkv_read(p)
        assert e.value.message.startswith("UnsupportedVersion")


def _corrupt(path, fn):
    raw = bytearray(open(path, "rb").read())
    raw = fn(raw)
    open(path, "wb").write(bytes(raw))


@pytest.mark.parametrize("name,fn,cls", [
    ("magic", lambda r: b"PQKX" + r[4:], "BadMagic"),
    ("version", lambda r: r[:4] + struct.pack("<I", 7) + r[8:], "UnsupportedVersion"),
    ("dtype", lambda r: r[:8] + struct.pack("<I", 9) + r[12:], "UnsupportedDtype"),
    ("header", lambda r: r[:10], "MalformedFile"),
    ("truncated", lambda r: r[:-4], "MalformedFile"),
    ("trailing", lambda r: r + b"\0\0\0\0", "MalformedFile"),
    ("nan", lambda r: r[:24 + 4 * (2 * 2048 + 17)] + struct.pack("<f", float("nan")) + r[24 + 4 * (2 * 2048 + 18):],
     "NonFiniteValue"),
])
def test_pqkv_errors_match_reference(oracle_mod, ref_available, tmp_path, bundle, name, fn, cls):
    import paper_2602_01077_b200 as P
    from paper_2602_01077_b200 import pqkv
    p = str(tmp_path / f"{name}.pqkv")
    pqkv.write_bundle(p, *bundle)
    _corrupt(p, fn)
    with pytest.raises(getattr(P, cls)) as e:
        pqkv.read_bundle(p)
    assert e.value.kind == P.ErrorKind.Io
    if ref_available:
        with pytest.raises(oracle_mod.OracleError) as r:
            oracle_mod.ref_pqkv_read(p)
        assert r.value.message.split(":")[0] == cls
        if name == "nan":  # same offender: K head 0 row 1 col 1 (io.hpp:84-101)
            assert str(e.value).split(":", 1)[1].strip() == r.value.message.split(":", 1)[1].strip()


def test_pqkv_io_error(tmp_path):
    import paper_2602_01077_b200 as P
    from paper_2602_01077_b200 import pqkv
    with pytest.raises(P.IoError):
        pqkv.read_bundle(str(tmp_path / "missing.pqkv"))


@pytest.mark.parametrize("L,d,b,k,variant", [(4096, 64, 64, 16, "hybrid"), (75584, 128, 64, 148, "hybrid"),
                                             (2048, 64, 64, 8, "sparse_only"), (2048, 64, 64, 8, "zeroth"),
                                             (2048, 64, 64, 8, "block_first"),
                                             (2048, 64, 64, 8, "global_centroid")])
def test_flop_model_matches_reference(oracle_mod, ref_available, L, d, b, k, variant):
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    from paper_2602_01077_b200 import cli
    ours = cli.flop_model(L, d, b, k, cli.VARIANTS[variant])
    ref = oracle_mod.ref_flop_model(L, d, b, k, variant)
    for key, val in ref.items():
        assert ours[key] == pytest.approx(val, rel=1e-15), key


def test_cli_exit_codes(tmp_path):
    from paper_2602_01077_b200 import cli, pqkv
    assert cli.main(["run", "--variant", "nope"]) == 2            # parse / validation
    assert cli.main(["gen", "--len", "1000", "--out", str(tmp_path / "x")]) == 2  # BlockDivisibility
    bad = tmp_path / "bad.pqkv"
    bad.write_bytes(b"NOPE" + bytes(20))
    assert cli.main(["run", "--in", str(bad)]) == 3               # BadMagic: Io
    del pqkv


@pytest.mark.gpu
def test_cli_gen_run_sweep_bench(tmp_path, capsys):
    from paper_2602_01077_b200 import cli
    f = str(tmp_path / "x.pqkv")
    assert cli.main(["gen", "--kind", "clustered", "--heads", "2", "--len", "2048", "--dim", "128",
                     "--out", f]) == 0
    g = json.loads(capsys.readouterr().out)
    assert g["bytes"] == os.path.getsize(f) == 24 + 3 * 2 * 2048 * 128 * 4
    assert cli.main(["run", "--in", f, "--sparsity", "0.75", "--deterministic"]) == 0
    r = json.loads(capsys.readouterr().out)
    assert r["seq_len"] == 2048 and r["num_heads"] == 2 and r["sparsity_realized"] == 0.75
    assert r["l1_rel"] < 0.1 and r["wall_ms"] == 0.0
    assert r["flops_ratio"] == pytest.approx(cli.flop_model(2048, 128, 64, 8, cli.VARIANTS["hybrid"])["pisa_ratio"])
    # full coverage (r = 0) is dense attention up to bf16 rounding
    assert cli.main(["run", "--in", f, "--sparsity", "0.0"]) == 0
    assert json.loads(capsys.readouterr().out)["max_abs"] < 2e-2
    assert cli.main(["run", "--in", f, "--strategy", "cov"]) == 0
    capsys.readouterr()
    assert cli.main(["sweep", "--lengths", "1024,2048", "--sparsities", "0.5,0.875",
                     "--variants", "hybrid,block_first", "--heads", "2", "--dim", "64"]) == 0
    rows = capsys.readouterr().out.strip().split("\n")
    assert rows[0].startswith("method,strategy,seed,head")
    assert len(rows) == 1 + 2 * 2 * 2 * 2
    assert sum(r.endswith(",ok") for r in rows[1:]) == 8
    assert sum(r.endswith(",Unsupported") for r in rows[1:]) == 8  # BlockFirst is off the GPU path
    assert cli.main(["bench", "--len", "8192", "--heads", "4", "--dim", "128", "--reps", "3",
                     "--sparsity", "0.875"]) == 0
    b = json.loads(capsys.readouterr().out)
    assert b["hybrid_ms"] > 0 and b["speedup"] > 0


def test_verify_unknown_check_exit_code():
    """cmd_verify (pisa_cli.cpp:668-693): an unknown --only is exit code 2."""
    from paper_2602_01077_b200 import cli
    assert cli.main(["verify", "--only", "no_such_check"]) == 2


@pytest.mark.gpu
def test_verify_all_checks_pass(capsys):
    """The reference's invariant suite on the GPU path (cmd_verify): oracle
    equivalence vs fp64 piecewise attention, full coverage == dense, constant-key
    exactness, Theorem 1 and Jensen bounds on the GPU plans, streaming ==
    reference, router properties."""
    from paper_2602_01077_b200 import cli
    rc = cli.main(["verify", "--seeds", "2"])
    out = capsys.readouterr().out
    assert rc == 0, out
    for name in cli.VERIFY_CHECKS:
        assert f"pass  {name}" in out
