"""Both GPU CLIs -- the native one (tools/radial_cli.cpp -> paper_2506_19852_b200/lib/radial_cli,
C++ over the drop-in headers) and the Python mirror (paper_2506_19852_b200/cli.py) -- keep the
reference CLI's flags, JSON keys and exit codes (reference tools/radial_cli.cpp, tests/test_cli.cpp)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NATIVE = os.path.join(ROOT, "paper_2506_19852_b200", "lib", "radial_cli")


@pytest.fixture(params=["native", "python"])
def _cli(request):
    if request.param == "native":
        if not os.path.exists(NATIVE):
            subprocess.run(["make", "-C", ROOT, "cli"], check=True, capture_output=True)
        prefix = [NATIVE]
    else:
        prefix = [sys.executable, "-m", "paper_2506_19852_b200.cli"]

    def run(*args):
        r = subprocess.run([*prefix, *args], capture_output=True, text=True, cwd=ROOT, timeout=600)
        return r.returncode, r.stdout, r.stderr
    return run


def test_stats_from_ramk_file_matches_reference_keys(tmp_path, _cli):
    rp, ci = O.blockify(33, 3600, 128)
    path = tmp_path / "h33.ramk"
    path.write_bytes(O.serialize(33, 3600, 128, "radial", True, rp, ci))
    rc, out, err = _cli("stats", "--in", str(path), "--head-dim", "128", "--heads", "24")
    assert rc == 0, err
    j = json.loads(out)
    assert set(j) == {"f", "s", "B", "kept_blocks", "sparsity", "dense_flops", "sparse_flops", "reduction"}
    assert j["kept_blocks"] == 389411 and j["sparse_flops"] == pytest.approx(7.8399e13, rel=1e-4)


def test_usage_and_input_errors_exit_2(tmp_path, _cli):
    assert _cli("stats", "--pattern", "nope", "--frames", "2", "--tokens", "2")[0] == 2
    assert _cli("stats")[0] == 2  # no shape
    assert _cli("frobnicate")[0] == 2
    bad = tmp_path / "bad.ramk"
    bad.write_bytes(b"RAMX")
    rc, _, err = _cli("stats", "--in", str(bad))
    assert rc == 2 and "magic" in err


@pytest.mark.gpu
def test_stats_presets_match_reference_acceptance_values(_cli):
    # acceptance_main.cpp:182-212: hunyuan-509 reduction ~4.46x (formula), sparsities 59.6/68.0/77.6%
    rc, out, _ = _cli("stats", "--preset", "hunyuan-509", "--head-dim", "128")
    assert rc == 0
    assert json.loads(out)["reduction"] == pytest.approx(4.46, abs=0.01)
    got = [json.loads(_cli("stats", "--preset", p)[1])["sparsity"] for p in ("wan-161", "hunyuan-253", "hunyuan-509")]
    assert got == pytest.approx([0.596, 0.680, 0.776], abs=0.001)


@pytest.mark.gpu
def test_mask_writes_reference_bytes_and_pgm(tmp_path, _cli):
    out, pgm = tmp_path / "m.ramk", tmp_path / "m.pgm"
    rc, so, err = _cli("mask", "--frames", "256", "--tokens", "64", "--block", "64", "--out", str(out), "--pgm", str(pgm))
    assert rc == 0, err
    rp, ci = O.blockify(256, 64, 64)
    assert out.read_bytes() == O.serialize(256, 64, 64, "radial", True, rp, ci)
    img = pgm.read_bytes()
    px = np.frombuffer(img[len(b"P5\n256 256\n255\n"):], np.uint8).reshape(256, 256)
    assert px[1, 130] == 255 and px[1, 129] == 0 and (px[:, 0] == 0).all()
    assert json.loads(so)["kept_blocks"] == int(rp[-1])


@pytest.mark.gpu
def test_bench_emits_reference_keys(_cli):
    rc, out, err = _cli("bench", "--frames", "16", "--tokens", "256", "--head-dim", "64", "--block", "64")
    assert rc == 0, err
    j = json.loads(out)
    assert set(j) == {"dense_seconds", "masked_seconds", "speedup", "flops_reduction"}
    assert j["dense_seconds"] > 0 and j["masked_seconds"] > 0
