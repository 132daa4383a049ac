"""CPU tests: the oracle restatement is pinned against the reference itself
(oracle/_ref) and against the committed golden vectors (tests/golden/)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _golden_layouts():
    with open(os.path.join(GOLD, "layouts.json")) as fh:
        return json.load(fh)["layouts"]


@pytest.mark.parametrize("g", _golden_layouts(), ids=lambda g: f"f{g['f']}s{g['s']}B{g['B']}sink{int(g['sink'])}")
def test_restatement_matches_golden_layout_bytes(g):
    rp, ci = O.blockify(g["f"], g["s"], g["B"], "radial", g["sink"])
    data = O.serialize(g["f"], g["s"], g["B"], "radial", g["sink"], rp, ci)
    assert len(data) == g["bytes"]
    assert hashlib.sha256(data).hexdigest() == g["sha256"]


def test_survey_hashes_are_the_golden_ones():
    # SURVEY.md 8c table, measured with the reference blockify
    survey = {
        (8, 256, 64, True): "bdbef9352e6de30d1be8f82c0d6cce8dfbbcd09a2fae0343f17eb5a89ca4bce1",
        (8, 256, 64, False): "506c0f359a4e6dd8a6bc43eeed6ee7b250b50a0f18bcccb8c20df56c63734dbb",
        (33, 3600, 128, True): "f3d663bff274b40450f994bd2f8e0bffd200fff5771001195e651361ad6aec6c",
        (33, 3600, 128, False): "667e253a1dba37b055f7f712bddb81f1490f4b4435ccc075d61db1afac80bae5",
        (21, 3600, 128, True): "21741ca790e8f774ac70fb49e2eb5f8a9911b1f4a57b5d51c538f1598f17ad38",
        (21, 3600, 128, False): "02ecdb2724966428969b3457698835aea95953b83f15eea9a04c5cc30cdfac24",
        (28, 1590, 128, True): "0eb4614e1c8a2784dbf048f399c25028c575cafb37e4b0e7382e5aa14d53826e",
        (28, 1590, 128, False): "db06e8e2c7d1702634569d46688b06851239e4cf9cc168130ee01381d45a8012",
        (132, 3600, 128, True): "d0f5843eef87b417ab6867c912c70307d270415412f182b1fdc4b366a0ef6295",
        (132, 3600, 128, False): "5ccb9d10345398cc39c1b35dbeeed1700f3ee847935c0554e2c4d5d33ad7b596",
    }
    gold = {(g["f"], g["s"], g["B"], g["sink"]): g["sha256"] for g in _golden_layouts()}
    for key, h in survey.items():
        assert gold[key] == h


@need_ref
def test_restatement_matches_reference_all_kinds_small_shapes():
    rng = np.random.default_rng(5)
    kinds = [("radial", 0, 0), ("dense", 0, 0), ("sta", 2, 2), ("temporal", 0, 1),
             ("spatial", 1, 0), ("harmonic", 0, 0), ("power", 0, 0)]
    shapes = [(8, 4, 4), (8, 4, 3), (5, 7, 4), (12, 5, 8), (9, 3, 2), (6, 6, 16), (16, 4, 8)]
    shapes += [tuple(int(x) for x in (1 + rng.integers(12), 1 + rng.integers(12), 1 + rng.integers(9)))
               for _ in range(40)]
    for f, s, B in shapes:
        for kind, tw, sw in kinds:
            for sink in (True, False):
                rp, ci = O.blockify(f, s, B, kind, sink, tw, sw)
                mine = O.serialize(f, s, B, kind, sink, rp, ci)
                assert mine == O.ref_serialize(f, s, B, kind, sink, tw, sw), (f, s, B, kind, sink)


@need_ref
def test_radial_keep_exhaustive_vs_reference():
    # test_grid_mask.cpp:110-129
    lib_c, lib_r = O.c(), O.ref()
    for f in range(1, 10):
        for s in range(1, 10):
            for sink in (0, 1):
                for i in range(f):
                    for j in range(f):
                        for k in range(s):
                            for l in range(s):
                                assert lib_c.ro_radial_keep(i, j, k, l, s, sink) == \
                                    lib_r.ref_radial_keep(f, s, i, j, k, l, sink)


def test_pixel_kats_f256_s64_b64():
    # test_blocksparse.cpp:229-243
    rp, ci = O.blockify(256, 64, 64, "radial", True)
    R = len(rp) - 1
    kept = np.zeros((R, R), bool)
    for I in range(R):
        kept[I, ci[rp[I]:rp[I + 1]]] = True
    assert kept[:, 0].all() and np.diag(kept).all()
    assert not kept[1, 130] and kept[1, 129]
    assert kept.sum() == rp[-1]


def test_blockify_strictly_increasing_and_b1_token_mask():
    rp, ci = O.blockify(6, 5, 1, "radial", True)
    lib = O.c()
    n = 30
    for u in range(n):
        row = set(ci[rp[u]:rp[u + 1]].tolist())
        for v in range(n):
            assert (v in row) == bool(lib.ro_radial_keep(u // 5, v // 5, u % 5, v % 5, 5, 1))
    for f, s, B in [(33, 3600, 128), (8, 256, 64)]:
        rp, ci = O.blockify(f, s, B)
        for I in range(len(rp) - 1):
            seg = ci[rp[I]:rp[I + 1]].astype(np.int64)
            assert (np.diff(seg) > 0).all()


@need_ref
def test_random_instance_matches_reference():
    q, k, v = O.random_instance(8 * 256, 64, 42)
    q2, k2, v2 = O.ref_random_instance(8, 256, 64, 42)
    assert np.array_equal(q, q2) and np.array_equal(k, k2) and np.array_equal(v, v2)


def test_random_instance_matches_golden():
    g = np.load(os.path.join(GOLD, "attention_small.npz"))
    q, k, v = O.random_instance(2048, 64, 42)
    assert np.array_equal(q[:4], g["tiny_seed42_q_head"])
    assert np.array_equal(k[:4], g["tiny_seed42_k_head"])
    assert np.array_equal(v[-4:], g["tiny_seed42_v_tail"])


def test_attention_rows_match_golden_reference_outputs():
    g = np.load(os.path.join(GOLD, "attention_small.npz"))
    rp, ci = O.blockify(6, 6, 4, "radial", True)
    out = O.attention_rows(g["f6s6_q"], g["f6s6_k"], g["f6s6_v"], 4, rp, ci, np.arange(36))
    assert np.abs(out - g["f6s6_out"]).max() < 1e-12
    dense = O.attention_rows(g["f8s8_q"], g["f8s8_k"], g["f8s8_v"], 8, None, None, np.arange(64))
    assert np.abs(dense - g["f8s8_dense"]).max() < 1e-12


@need_ref
def test_attention_rows_match_reference_tiny_config():
    f, s, d, B = 8, 256, 64, 64
    q, k, v = O.ref_random_instance(f, s, d, 42)
    rp, ci = O.blockify(f, s, B)
    ref = O.ref_masked_attention(f, s, q, k, v, B, rp, ci)
    rows = np.arange(0, f * s, 7)
    mine = O.attention_rows(q, k, v, B, rp, ci, rows)
    assert np.abs(mine - ref[rows]).max() < 1e-12


def test_empty_row_raises_row_0():
    # test_attention.cpp:143-154
    q, k, v = O.random_instance(4, 4, 1)
    rp = np.zeros(3, np.uint64)
    with pytest.raises(RuntimeError, match="row 0"):
        O.attention_rows(q, k, v, 2, rp, np.zeros(0, np.uint32), np.arange(4))


def test_bwd_oracle_matches_torch_autograd_and_finite_differences():
    torch = pytest.importorskip("torch")
    f, s, B, d = 4, 6, 4, 8
    n = f * s
    rp, ci = O.blockify(f, s, B)
    rng = np.random.default_rng(0)
    q, k, v, do = (rng.standard_normal((n, d)).astype(np.float32) for _ in range(4))
    dq, dk, dv = O.attention_bwd(q, k, v, do, B, rp, ci)
    R = len(rp) - 1
    mask = np.zeros((n, n), bool)
    for I in range(R):
        for J in ci[rp[I]:rp[I + 1]]:
            mask[I * B:(I + 1) * B, J * B:(J + 1) * B] = True
    tq, tk, tv = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (q, k, v))
    sc = (tq @ tk.T) / np.sqrt(d)
    sc = sc.masked_fill(~torch.tensor(mask), float("-inf"))
    o = torch.softmax(sc, -1) @ tv
    o.backward(torch.tensor(do, dtype=torch.float64))
    assert np.abs(dq - tq.grad.numpy()).max() < 1e-10
    assert np.abs(dk - tk.grad.numpy()).max() < 1e-10
    assert np.abs(dv - tv.grad.numpy()).max() < 1e-10
    # forward output of the oracle equals torch's masked softmax
    fwd = O.attention_rows(q, k, v, B, rp, ci, np.arange(n))
    assert np.abs(fwd - o.detach().numpy()).max() < 1e-12


@need_ref
@pytest.mark.parametrize("kind,sink,tw,sw", [("power", False, 0, 0), ("power", True, 0, 0), ("radial", True, 0, 0),
                                             ("sta", True, 1, 9), ("harmonic", False, 0, 0)])
def test_token_attention_rows_match_reference_every_kind(kind, sink, tw, sw):
    """The token-exact restatement (attention.hpp:184-225 over for_each_kept_interval,
    mask.hpp:238-272, power included) equals the reference's own masked_attention(inst,
    PatternSpec) on fp32-exact inputs."""
    f, s, d = 6, 37, 16
    q, k, v = (x.astype(np.float32).astype(np.float64) for x in O.random_instance(f * s, d, 9))
    ref = O.ref_masked_attention_pattern(f, s, q, k, v, kind, sink, tw, sw)
    mine = O.token_attention_rows(q, k, v, f, s, np.arange(f * s), kind, sink, tw, sw)
    assert np.abs(mine - ref).max() < 1e-12


def test_vectorised_radial_token_rule_matches_oracle():
    """tests._util.radial_token_keep (used by the GPU full-coverage token-exact test) equals the
    oracle's radial_keep, which test_radial_keep_exhaustive_vs_reference pins to the reference;
    random (i, j, k, l) including far frames where 2^e > s (the diagonal case)."""
    import torch
    from tests._util import radial_token_keep
    lib = O.c()
    rng = np.random.default_rng(11)
    for s, f in ((3600, 33), (5, 600), (1, 300), (7, 9)):
        i, j = rng.integers(0, f, 4000), rng.integers(0, f, 4000)
        k, l = rng.integers(0, s, 4000), rng.integers(0, s, 4000)
        for sink in (True, False):
            got = radial_token_keep(torch.from_numpy(i * s + k), torch.from_numpy(j * s + l), s, sink).numpy()
            want = [bool(lib.ro_radial_keep(int(a), int(b), int(c), int(e), s, int(sink))) for a, b, c, e in zip(i, j, k, l)]
            assert got.tolist() == want, (s, f, sink)
