"""GPU parity: K1 (on-device blockify) is bit-exact with the reference layout bytes."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU test on a box without CUDA"
    import paper_2506_19852_b200 as P
    return P


def _golden():
    with open(os.path.join(GOLD, "layouts.json")) as fh:
        return json.load(fh)["layouts"]


@pytest.mark.parametrize("g", _golden(), ids=lambda g: f"f{g['f']}s{g['s']}B{g['B']}sink{int(g['sink'])}")
def test_device_blockify_matches_golden_sha256(P, g):
    lay = P.device_layout(P.GridShape(g["f"], g["s"]), P.PatternSpec.radial(g["sink"]), g["B"],
                          cache=False)
    host = lay.host()
    data = P.serialize(host)
    assert len(data) == g["bytes"]
    assert hashlib.sha256(data).hexdigest() == g["sha256"]
    assert lay.kept_blocks() == g["nnz"] and lay.grid_rows == g["R"]


def test_device_blockify_exhaustive_small_shapes(P):
    # f, s in [1,16], B in [1,20], sink on/off (the survey's verification sweep)
    bad = []
    for f in range(1, 17):
        for s in range(1, 17):
            for B in range(1, 21):
                for sink in (True, False):
                    host = P.blockify(P.GridShape(f, s), P.PatternSpec.radial(sink), B)
                    rp, ci = O.blockify(f, s, B, "radial", sink)
                    if not (np.array_equal(host.row_ptr, rp) and np.array_equal(host.col_idx, ci)):
                        bad.append((f, s, B, sink))
    assert not bad, bad[:10]


def test_device_blockify_all_kinds(P):
    specs = [(P.PatternSpec.dense(), "dense", 0, 0), (P.PatternSpec.sta(2, 2), "sta", 2, 2),
             (P.PatternSpec.temporal(1, True), "temporal", 0, 1),
             (P.PatternSpec.spatial(1), "spatial", 1, 0),
             (P.PatternSpec.harmonic(True), "harmonic", 0, 0), (P.PatternSpec.power(), "power", 0, 0),
             (P.PatternSpec.power(True), "power", 0, 0)]
    shapes = [(8, 4, 4), (8, 4, 3), (5, 7, 4), (12, 5, 8), (9, 3, 2), (6, 6, 16), (16, 4, 8),
              (33, 60, 16), (7, 100, 64)]
    for f, s, B in shapes:
        for spec, kind, tw, sw in specs:
            host = P.blockify(P.GridShape(f, s), spec, B)
            rp, ci = O.blockify(f, s, B, kind, spec.sink, tw, sw)
            assert np.array_equal(host.row_ptr, rp) and np.array_equal(host.col_idx, ci), (f, s, B, kind)


def test_csc_is_the_transpose(P):
    for f, s, B in [(33, 3600, 128), (8, 256, 64), (5, 7, 4)]:
        for sink in (True, False):
            lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(sink), B, cache=False)
            host = lay.host()
            cp, ri = lay.csc()
            R = host.grid_rows
            rows = np.repeat(np.arange(R), np.diff(host.row_ptr).astype(np.int64))
            order = np.lexsort((rows, host.col_idx))
            want_ri = rows[order].astype(np.uint32)
            want_cp = np.concatenate([[0], np.cumsum(np.bincount(host.col_idx, minlength=R))])
            assert np.array_equal(cp, want_cp.astype(np.uint64))
            assert np.array_equal(ri, want_ri)


def test_layout_from_host_csr_roundtrip_and_validation(P):
    host = P.blockify(P.GridShape(8, 256), P.PatternSpec.radial(), 64)
    dev = P.layout_from_host(host)
    assert dev.host() == host
    bad = P.BlockLayout(host.shape, 64, host.grid_rows, host.row_ptr.copy(), host.col_idx.copy())
    bad.col_idx[1] = bad.col_idx[0]
    with pytest.raises(ValueError, match="strictly increasing"):
        P.layout_from_host(bad)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("f,s", [(33, 3600), (28, 1590)])
def test_device_blockify_all_kinds_paper_scale_vs_reference(P, f, s):
    """K1 for every pattern kind at the BASELINE shapes, byte-identical with the reference's
    own blockify + serialize (oracle/_ref, the unmodified reference headers)."""
    B = 128
    specs = [(P.PatternSpec.dense(), "dense", 0, 0), (P.PatternSpec.sta(2, 600), "sta", 2, 600),
             (P.PatternSpec.temporal(300, True), "temporal", 0, 300), (P.PatternSpec.spatial(2), "spatial", 2, 0),
             (P.PatternSpec.harmonic(True), "harmonic", 0, 0), (P.PatternSpec.power(True), "power", 0, 0),
             (P.PatternSpec.radial(False), "radial", 0, 0)]
    for spec, kind, tw, sw in specs:
        mine = P.serialize(P.blockify(P.GridShape(f, s), spec, B))
        assert mine == O.ref_serialize(f, s, B, kind, spec.sink, tw, sw), (f, s, kind)
