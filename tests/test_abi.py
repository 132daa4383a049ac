"""CPU tests: the C-ABI library loads and exports every symbol include/radial_cuda.h
declares; host-side logic (serialization, accounting) matches the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "radial_cuda.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(radial_cuda_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_2506_19852_b200 as P
    lib = ctypes.CDLL(P.library_path())
    syms = _declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.radial_cuda_abi_version() == 2


def test_library_is_sm100a():
    import subprocess
    import paper_2506_19852_b200 as P
    out = subprocess.run(["cuobjdump", "--list-elf", P.library_path()], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_serialize_roundtrip_and_matches_oracle_bytes():
    import oracle as O
    import paper_2506_19852_b200 as P
    rng = np.random.default_rng(23)
    for _ in range(30):
        f, s, B = (int(x) for x in (1 + rng.integers(12), 1 + rng.integers(12), 1 + rng.integers(9)))
        sink = bool(rng.integers(2))
        rp, ci = O.blockify(f, s, B, "radial", sink)
        lay = P.BlockLayout(P.GridShape(f, s), B, len(rp) - 1, rp, ci, 0, sink)
        data = P.serialize(lay)
        assert data == O.serialize(f, s, B, "radial", sink, rp, ci)
        assert P.deserialize(data) == lay


def test_parse_errors_are_structured():
    # test_blocksparse.cpp:172-217
    import oracle as O
    import paper_2506_19852_b200 as P
    rp, ci = O.blockify(4, 4, 4)
    good = P.serialize(P.BlockLayout(P.GridShape(4, 4), 4, 4, rp, ci))
    cases = [(b"X" + good[1:], "magic"), (good[:4] + b"\x7f" + good[5:], "version"),
             (good[:-1], "col_idx"), (good + b"\0", "trailer"),
             (good[:18] + bytes([9]) + good[19:], "kind")]
    for data, fieldname in cases:
        with pytest.raises(P.ParseError, match=fieldname):
            P.deserialize(data)
    with pytest.raises(P.ParseError):
        P.deserialize(good[:10])
    with pytest.raises(P.ParseError) as ei:
        P.deserialize(b"RAMK")
    assert ei.value.field == "version"


def test_attention_flops_and_sparsity_match_reference_convention():
    import oracle as O
    import paper_2506_19852_b200 as P
    rp, ci = O.blockify(33, 3600, 128)
    lay = P.BlockLayout(P.GridShape(33, 3600), 128, len(rp) - 1, rp, ci)
    rep = P.attention_flops(lay, 128, 24)
    assert rep.sparse_flops == pytest.approx(7.8399e13, rel=1e-4)
    assert rep.dense_flops == pytest.approx(1.73426e14, rel=1e-4)
    assert P.sparsity(lay) == pytest.approx(0.5488, abs=1e-4)
    if O.ref_available():
        d, sp, red, spars = (ctypes.c_double() for _ in range(4))
        assert O.ref().ref_attention_flops(33, 3600, 128, 1, 128, 24, ctypes.byref(d),
                                           ctypes.byref(sp), ctypes.byref(red),
                                           ctypes.byref(spars)) == 0
        assert rep.sparse_flops == sp.value and rep.dense_flops == d.value
        assert P.sparsity(lay) == spars.value
    with pytest.raises(ValueError):
        P.attention_flops(lay, 0, 1)


def test_grid_shape_and_pattern_validation():
    import paper_2506_19852_b200 as P
    with pytest.raises(ValueError):
        P.GridShape(0, 4)
    with pytest.raises(ValueError):
        P.GridShape(1 << 20, 1 << 13)
    with pytest.raises(ValueError, match="temporal_window"):
        P.PatternSpec(P.PatternKind.sta, False, None, 2).validate()


def test_scatter_forward_argument_validation():
    """radial_cuda_attn_fwd_scatter rejects bad destination lists before touching the GPU."""
    import paper_2506_19852_b200 as P
    lib = P._lib
    VP = ctypes.c_void_p
    fake = VP(0x1000)
    dst = (VP * 9)(*([0x2000] * 9))
    lib.radial_cuda_last_error.restype = ctypes.c_char_p

    def call(n_dst, head_base, heads_full, heads=2, ptrs=dst):
        return lib.radial_cuda_attn_fwd_scatter(fake, fake, fake, ptrs, n_dst, head_base, heads_full, None,
                                               heads, 4096, 128, ctypes.c_float(0.0), None, None)
    assert call(0, 0, 2) == 1 and b"destination" in lib.radial_cuda_last_error()
    assert call(9, 0, 2) == 1
    assert call(2, 7, 8) == 1 and b"heads_full" in lib.radial_cuda_last_error()
    nulls = (VP * 2)(0x2000, 0)
    assert call(2, 0, 2, ptrs=nulls) == 1 and b"null destination" in lib.radial_cuda_last_error()
    assert call(1, 0, 2) == 1 and b"null layout" in lib.radial_cuda_last_error()


@pytest.mark.parametrize("kind,tw,sw,msg", [(2, None, 0, "spatial pattern requires temporal_window"),
                                            (3, 0, None, "temporal pattern requires spatial_window"),
                                            (4, 1, None, "sta pattern requires spatial_window"),
                                            (4, None, 3, "sta pattern requires temporal_window")])
def test_mask_build_rejects_missing_windows(kind, tw, sw, msg):
    """PatternSpec::validate (grid.hpp:118-139) through the C-ABI: RADIAL_WINDOW_NONE marks an
    absent window; a kind that reads it fails with the reference's message (no CUDA call)."""
    import paper_2506_19852_b200 as P
    h = ctypes.c_void_p()
    none = P.WINDOW_NONE
    rc = P._lib.radial_cuda_mask_build(4, 16, 4, kind, 0, none if tw is None else tw, none if sw is None else sw,
                                       None, ctypes.byref(h))
    assert rc == P.ERR_INVALID
    assert P._lib.radial_cuda_last_error().decode() == msg
    assert not h.value


def test_missing_cuda_library_fails_loudly(tmp_path):
    """No CPU fallback: importing the package without its CUDA library raises ImportError
    (a fresh interpreter, pointed at a path that does not exist)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RADIAL_CUDA_LIB=str(tmp_path / "missing" / "libradial_cuda.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2506_19852_b200"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "ImportError" in r.stderr or "OSError" in r.stderr, r.stderr[-2000:]
