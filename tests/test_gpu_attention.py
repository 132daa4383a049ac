"""GPU parity: K2 sparse forward and K4 dense forward against the fp64 oracle (and the
reference itself where it is cheap), per (head, query block)."""
import os

import numpy as np
import pytest

import oracle as O
from tests._util import (assert_within, bf16_bits, bits_to_f32, block_errors, instance_bf16,
                         to_torch_bf16)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU test on a box without CUDA"
    import paper_2506_19852_b200 as P
    return P


def _run_sparse(P, f, s, B, d, H, sink=True, q_scale=1.0, seed0=42):
    import torch
    q, k, v = instance_bf16(f, s, d, H, seed0, q_scale)
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(sink), B)
    o, lse = P.masked_attention(to_torch_bf16(q), to_torch_bf16(k), to_torch_bf16(v), lay,
                                return_lse=True)
    torch.cuda.synchronize()
    return q, k, v, lay.host(), o.float().cpu().numpy(), lse.cpu().numpy()


def test_debug_tile_mma_building_blocks(P):
    """S = Q K^T (SS, K-major) and O = P V (TS, MN-major V) on one 128x128x128 tile."""
    import ctypes
    import torch
    lib = ctypes.CDLL(P.debug_library_path())
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, p = (torch.randn(128, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    s_out = torch.empty(128, 128, device="cuda")
    o_out = torch.empty(128, 128, device="cuda")
    rc = lib.radial_cuda_debug_tile(ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(k.data_ptr()),
                                    ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(p.data_ptr()),
                                    ctypes.c_void_p(s_out.data_ptr()), ctypes.c_void_p(o_out.data_ptr()),
                                    ctypes.c_void_p(0))
    assert rc == 0
    torch.cuda.synchronize()
    s_ref = q.float() @ k.float().T
    o_ref = p.float() @ v.float()
    es = (s_out - s_ref).abs().max().item()
    eo = (o_out - o_ref).abs().max().item()
    assert es < 1e-2 * s_ref.abs().max().item(), f"S mismatch {es}"
    assert eo < 1e-2 * o_ref.abs().max().item(), f"O mismatch {eo}"


def test_tiny_config_vs_oracle_all_rows(P):
    # BASELINE configs[0]: 8 frames x 256 tokens, 2 heads, head_dim 64, block 64
    f, s, B, d, H = 8, 256, 64, 64, 2
    q, k, v, host, o, lse = _run_sparse(P, f, s, B, d, H)
    n = f * s
    rows = np.arange(n)
    for h in range(H):
        want, wl = O.attention_rows(q[h], k[h], v[h], B, host.row_ptr, host.col_idx, rows,
                                    want_lse=True)
        assert_within(block_errors(o[h], want, rows, B), f"tiny head {h}")
        assert np.abs(lse[h] - wl).max() < 2e-2


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_tiny_config_vs_reference_library(P):
    """The reference's own masked_attention on the same bf16-rounded inputs."""
    f, s, B, d = 8, 256, 64, 64
    q, k, v, host, o, _ = _run_sparse(P, f, s, B, d, 1)
    ref = O.ref_masked_attention(f, s, q[0].astype(np.float64), k[0].astype(np.float64),
                                 v[0].astype(np.float64), B, host.row_ptr, host.col_idx)
    assert_within(block_errors(o[0], ref, np.arange(f * s), B), "tiny vs reference")


@pytest.mark.parametrize("f,s,B,d", [(5, 300, 128, 128), (3, 1000, 128, 128), (7, 200, 64, 128),
                                     (4, 333, 128, 64), (2, 64, 64, 64), (1, 100, 128, 128),
                                     (9, 130, 64, 64), (12, 257, 128, 128)])
@pytest.mark.parametrize("sink", [True, False])
def test_ragged_shapes_vs_oracle(P, f, s, B, d, sink):
    H = 2
    q, k, v, host, o, lse = _run_sparse(P, f, s, B, d, H, sink=sink, seed0=7)
    rows = np.arange(f * s)
    for h in range(H):
        want, wl = O.attention_rows(q[h], k[h], v[h], B, host.row_ptr, host.col_idx, rows,
                                    want_lse=True)
        assert_within(block_errors(o[h], want, rows, B), f"f{f}s{s}B{B}d{d} head {h}")
        assert np.abs(lse[h] - wl).max() < 2e-2


def test_random_shape_fuzz_vs_oracle(P):
    """40 random grids (frames 1-20, tokens per frame 1-700, block 64/128, head_dim 64/128,
    sink on/off, 1-3 heads): every query block of every head against the fp64 oracle --
    exercises short KV lists (fewer steps than the K/V ring), tails inside a tile, and
    chunks whose second tile is past the grid."""
    rng = np.random.default_rng(2025)
    for case in range(40):
        f = int(rng.integers(1, 21))
        s = int(rng.integers(1, 701))
        if f * s < 2:
            continue
        B = int(rng.choice([64, 128]))
        d = int(rng.choice([64, 128]))
        sink = bool(rng.integers(0, 2))
        H = int(rng.integers(1, 4))
        q, k, v, host, o, lse = _run_sparse(P, f, s, B, d, H, sink=sink, seed0=100 + case)
        rows = np.arange(f * s)
        for h in range(H):
            want, wl = O.attention_rows(q[h], k[h], v[h], B, host.row_ptr, host.col_idx, rows, want_lse=True)
            assert_within(block_errors(o[h], want, rows, B), f"case {case}: f{f}s{s}B{B}d{d}sink{sink} head {h}")
            assert np.abs(lse[h] - wl).max() < 2e-2, f"case {case} lse"


@pytest.mark.parametrize("B,d", [(128, 128), (64, 64)])
def test_peaked_logits_q_times_8(P, B, d):
    f, s, H = 6, 400, 2
    q, k, v, host, o, _ = _run_sparse(P, f, s, B, d, H, q_scale=8.0, seed0=3)
    rows = np.arange(f * s)
    for h in range(H):
        want = O.attention_rows(q[h], k[h], v[h], B, host.row_ptr, host.col_idx, rows)
        assert_within(block_errors(o[h], want, rows, B), f"peaked head {h}")


@pytest.mark.parametrize("n,d,B", [(1500, 128, 128), (2048, 64, 64), (700, 128, 64)])
def test_dense_kernel_vs_oracle(P, n, d, B):
    import torch
    H = 2
    q, k, v = instance_bf16(1, n, d, H, 11)
    o = P.dense_attention(to_torch_bf16(q), to_torch_bf16(k), to_torch_bf16(v), block_size=B)
    torch.cuda.synchronize()
    o = o.float().cpu().numpy()
    rows = np.arange(n)
    for h in range(H):
        want = O.attention_rows(q[h], k[h], v[h], B, None, None, rows)
        assert_within(block_errors(o[h], want, rows, B), f"dense n{n} head {h}")


def test_dense_pattern_layout_equals_dense_kernel(P):
    """masked_attention over the dense PatternSpec == the dense comparator (acceptance crit. 5)."""
    import torch
    f, s, d, H = 4, 300, 128, 2
    q, k, v = (to_torch_bf16(x) for x in instance_bf16(f, s, d, H, 5))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.dense(), 128)
    a = P.masked_attention(q, k, v, lay)
    b = P.dense_attention(q, k, v, block_size=128)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_host_buffer_api_matches_device_path(P):
    import torch
    f, s, B, d, H = 8, 256, 64, 64, 2
    q, k, v = instance_bf16(f, s, d, H, 42)
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    dev = P.masked_attention(to_torch_bf16(q), to_torch_bf16(k), to_torch_bf16(v), lay)
    torch.cuda.synchronize()
    host = P.masked_attention_host(bf16_bits(q), bf16_bits(k), bf16_bits(v), lay)
    assert np.array_equal(host, dev.view(torch.int16).cpu().numpy().view(np.uint16))


def test_errors_follow_reference_semantics(P):
    import torch
    q = torch.zeros(1, 16, 64, device="cuda", dtype=torch.bfloat16)
    # fully masked rows: attention.hpp:255-258 ("row 0"), test_attention.cpp:143-154
    empty = P.BlockLayout(P.GridShape(1, 16), 64, 1, np.zeros(2, np.uint64), np.zeros(0, np.uint32))
    with pytest.raises(RuntimeError, match="row 0"):
        P.masked_attention(q, q, q, empty)
    lay = P.device_layout(P.GridShape(2, 8), P.PatternSpec.radial(), 64)
    with pytest.raises(ValueError, match="shape mismatch"):
        P.masked_attention(torch.zeros(1, 32, 64, device="cuda", dtype=torch.bfloat16),
                           torch.zeros(1, 32, 64, device="cuda", dtype=torch.bfloat16),
                           torch.zeros(1, 32, 64, device="cuda", dtype=torch.bfloat16), lay)
    q32 = torch.zeros(1, 16, 32, device="cuda", dtype=torch.bfloat16)
    lay16 = P.device_layout(P.GridShape(1, 16), P.PatternSpec.radial(), 64)
    with pytest.raises(ValueError, match="head_dim"):
        P.masked_attention(q32, q32, q32, lay16)
    lay_b4 = P.device_layout(P.GridShape(1, 16), P.PatternSpec.radial(), 4)
    with pytest.raises(ValueError, match="block_size"):
        P.masked_attention(q, q, q, lay_b4)


def test_paper_scale_hunyuan33_sampled_blocks(P):
    """BASELINE configs[1] at full size: every head computed on the GPU; a sample of
    (head, query block) pairs -- first, tail, sink-adjacent and random -- checked
    against the fp64 oracle on the same bf16 inputs (rows are independent)."""
    import torch
    f, s, B, d, H = 33, 3600, 128, 128, 24
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(1234)
    q = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o = P.masked_attention(q, k, v, lay)
    torch.cuda.synchronize()
    host = lay.host()
    R = host.grid_rows
    rng = np.random.default_rng(0)
    for h in (0, 23):
        blocks = sorted({0, 1, 28, R // 2, R - 2, R - 1} | set(rng.integers(0, R, 4).tolist()))
        rows = np.concatenate([np.arange(I * B, min(n, (I + 1) * B)) for I in blocks])
        qh, kh, vh = (x[h].float().cpu().numpy() for x in (q, k, v))
        want = O.attention_rows(qh, kh, vh, B, host.row_ptr, host.col_idx, rows)
        got = o[h].float().cpu().numpy()[rows]
        assert_within(block_errors(got, want, rows, B), f"H33 head {h}")


def test_scatter_epilogue_writes_every_destination(P):
    """masked_attention_scatter (fused C1 reassembly): O rows of these heads land in every
    destination buffer at head_base + h, bit-identical to masked_attention, and nothing
    else in the buffers is touched (two local buffers stand in for two ranks' memory)."""
    import torch
    f, s, B, d, H, Hfull, base = 5, 300, 128, 128, 3, 8, 4
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o_ref, lse_ref = P.masked_attention(q, k, v, lay, return_lse=True)
    sentinel = torch.tensor(7.25, dtype=torch.bfloat16)
    bufs = [torch.full((Hfull, n, d), 7.25, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    lse = torch.empty(H, n, device="cuda")
    P.masked_attention_scatter(q, k, v, lay, [b.data_ptr() for b in bufs], base, Hfull, lse=lse)
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b[base:base + H], o_ref)
        assert bool((b[:base] == sentinel).all()) and bool((b[base + H:] == sentinel).all())
    assert torch.equal(lse, lse_ref)


def test_host_multi_device_entry_matches_single_call(P):
    """radial_cuda_attn_fwd_host_multi (one host thread per listed device, heads split
    evenly, mask built per device) equals the single-device forward; device 0 listed twice
    stands in for two GPUs (two threads, two pipelines, one device)."""
    import ctypes
    import torch
    f, s, B, d, H = 6, 500, 128, 128, 5
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(8)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o_ref, lse_ref = P.masked_attention(q, k, v, lay, return_lse=True)
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    for devs in ([0], [0, 0]):
        ho = torch.empty_like(hq).pin_memory()
        hl = torch.empty(H, n, dtype=torch.float32).pin_memory()
        arr = (ctypes.c_int * len(devs))(*devs)
        rc = P._lib.radial_cuda_attn_fwd_host_multi(hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr(),
                                                   hl.data_ptr(), H, n, d, 0.0, f, s, B, 0, 1, 0, 0, arr, len(devs))
        assert rc == 0, P._lib.radial_cuda_last_error()
        assert torch.equal(ho, o_ref.cpu()), devs
        assert torch.equal(hl, lse_ref.cpu()), devs


def test_fused_reassembly_through_symmetric_memory():
    """The multi-rank plumbing of the fused reassembly (torch symmetric memory rendezvous,
    peer pointers, barrier) under torchrun with the ranks this box has (1 here): every
    rank's full-O buffer equals the single-GPU forward of all heads."""
    import subprocess
    import sys
    import torch
    # RADIAL_TEST_RANKS pins the rank count (e.g. 8 on an 8-GPU node): fewer visible GPUs
    # is a failure, not a silent single-rank run
    want = os.environ.get("RADIAL_TEST_RANKS")
    nproc = int(want) if want else max(1, min(torch.cuda.device_count(), 8))
    assert torch.cuda.device_count() >= nproc, f"{nproc} ranks requested, {torch.cuda.device_count()} GPUs visible"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", "29561",
           os.path.join(ROOT, "scripts", "fused_gather_check.py"), "--expect-ranks", str(nproc)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert '"identical": true' in r.stdout
    assert f'"ranks": {nproc}' in r.stdout


@pytest.mark.parametrize("f,s,H", [(21, 3600, 40), (28, 1590, 24), (132, 3600, 24)],
                         ids=["wan21", "mochi28", "hunyuan132"])
def test_paper_scale_other_configs_sampled_blocks(P, f, s, H):
    """BASELINE configs[2..4] at full size (W21 40 heads, M28, the 475k-token H132): every
    head on the GPU, a sample of (head, query block) pairs against the fp64 oracle; the
    H132 lse is checked too (the backward consumes it)."""
    import torch
    B, d = 128, 128
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(99)
    q = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    torch.cuda.synchronize()
    host = lay.host()
    R = host.grid_rows
    rng = np.random.default_rng(f)
    for h in (0, H - 1):
        blocks = sorted({0, R // 3, R - 1} | set(rng.integers(0, R, 2).tolist()))
        rows = np.concatenate([np.arange(I * B, min(n, (I + 1) * B)) for I in blocks])
        qh, kh, vh = (x[h].float().cpu().numpy() for x in (q, k, v))
        want, want_lse = O.attention_rows(qh, kh, vh, B, host.row_ptr, host.col_idx, rows, want_lse=True)
        got = o[h].float().cpu().numpy()[rows]
        assert_within(block_errors(got, want, rows, B), f"f{f} s{s} head {h}")
        np.testing.assert_allclose(lse[h].cpu().numpy()[rows], want_lse, rtol=0, atol=2e-3)
    del q, k, v, o, lse
    torch.cuda.empty_cache()


def test_paper_scale_dense_comparator_sampled_rows(P):
    """K4 at the M28 shape (44,520 tokens, every key): sampled query blocks of two heads
    against the fp64 dense oracle (the reference's dense_attention, attention.hpp:141-163)."""
    import torch
    f, s, B, d, H = 28, 1590, 128, 128, 4
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    o = P.dense_attention(q, k, v, block_size=B)
    torch.cuda.synchronize()
    R = (n + B - 1) // B
    for h in (0, H - 1):
        blocks = [0, R // 2, R - 1]
        rows = np.concatenate([np.arange(I * B, min(n, (I + 1) * B)) for I in blocks])
        qh, kh, vh = (x[h].float().cpu().numpy() for x in (q, k, v))
        want = O.attention_rows(qh, kh, vh, B, None, None, rows)
        got = o[h].float().cpu().numpy()[rows]
        assert_within(block_errors(got, want, rows, B), f"dense M28 head {h}")


@pytest.mark.parametrize("f,s,B,d,kind,sink,tw,sw", [
    (8, 256, 64, 64, "radial", True, 0, 0), (6, 300, 128, 128, "radial", False, 0, 0),
    (33, 150, 128, 128, "radial", True, 0, 0), (5, 333, 64, 128, "sta", True, 1, 40),
    (7, 200, 128, 64, "harmonic", False, 0, 0), (9, 100, 128, 128, "temporal", True, 0, 17),
    (7, 90, 128, 64, "power", True, 0, 0), (12, 50, 64, 128, "power", False, 0, 0)])
def test_token_exact_forward_vs_oracle(P, f, s, B, d, kind, sink, tw, sw):
    """masked_attention(inst, PatternSpec) (attention.hpp:184-225) on the GPU: exact token mask."""
    import torch
    H = 2
    q, k, v = instance_bf16(f, s, d, H, 21)
    mk = {"radial": lambda: P.PatternSpec.radial(sink), "sta": lambda: P.PatternSpec.sta(tw, sw, sink),
          "harmonic": lambda: P.PatternSpec.harmonic(sink), "temporal": lambda: P.PatternSpec.temporal(sw, sink),
          "power": lambda: P.PatternSpec.power(sink)}
    o, lse = P.masked_attention_pattern(to_torch_bf16(q), to_torch_bf16(k), to_torch_bf16(v), P.GridShape(f, s),
                                        mk[kind](), block_size=B, return_lse=True)
    torch.cuda.synchronize()
    o = o.float().cpu().numpy()
    rows = np.arange(f * s)
    for h in range(H):
        want, wl = O.token_attention_rows(q[h], k[h], v[h], f, s, rows, kind, sink, tw, sw, want_lse=True)
        assert_within(block_errors(o[h], want, rows, B), f"token {kind} head {h}")
        assert np.abs(lse[h].cpu().numpy() - wl).max() < 2e-2 if hasattr(lse, "cpu") else True


def test_token_exact_random_fuzz_vs_oracle(P):
    """28 random token-exact cases over every kind (radial, dense, spatial, temporal, sta,
    harmonic, power) with random windows, sink, block and head_dim."""
    import torch
    rng = np.random.default_rng(4242)
    kinds = ["radial", "dense", "spatial", "temporal", "sta", "harmonic", "power"]
    for case in range(28):
        kind = kinds[case % len(kinds)]
        f = int(rng.integers(1, 14))
        s = int(rng.integers(2, 401))
        B = int(rng.choice([64, 128]))
        d = int(rng.choice([64, 128]))
        sink = bool(rng.integers(0, 2))
        tw = int(rng.integers(0, 4))
        sw = int(rng.integers(0, s))
        spec = {"radial": lambda: P.PatternSpec.radial(sink), "dense": lambda: P.PatternSpec.dense(),
                "spatial": lambda: P.PatternSpec.spatial(tw, sink),
                "temporal": lambda: P.PatternSpec.temporal(sw, sink),
                "sta": lambda: P.PatternSpec.sta(tw, sw, sink),
                "harmonic": lambda: P.PatternSpec.harmonic(sink),
                "power": lambda: P.PatternSpec.power(sink)}[kind]()
        q, k, v = instance_bf16(f, s, d, 1, 500 + case)
        try:
            o = P.masked_attention_pattern(to_torch_bf16(q), to_torch_bf16(k), to_torch_bf16(v), P.GridShape(f, s),
                                           spec, block_size=B)
        except RuntimeError as e:  # a row that keeps no key: the reference throws too
            assert "keeps no keys" in str(e), e
            continue
        torch.cuda.synchronize()
        rows = np.arange(f * s)
        want = O.token_attention_rows(q[0], k[0], v[0], f, s, rows,
                                      "dense" if kind == "dense" else kind,
                                      True if kind == "dense" else sink, tw, sw)
        assert_within(block_errors(o[0].float().cpu().numpy(), want, rows, B),
                      f"case {case}: {kind} f{f}s{s}B{B}d{d}sink{sink}tw{tw}sw{sw}")


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("kind,sink", [("radial", True), ("power", True), ("power", False)])
def test_token_exact_forward_vs_reference_library(P, kind, sink):
    import torch
    f, s, d = 8, 256, 64
    q, k, v = instance_bf16(f, s, d, 1, 42)
    spec = P.PatternSpec.radial(sink) if kind == "radial" else P.PatternSpec.power(sink)
    o = P.masked_attention_pattern(to_torch_bf16(q), to_torch_bf16(k), to_torch_bf16(v), P.GridShape(f, s),
                                   spec, block_size=64)
    torch.cuda.synchronize()
    ref = O.ref_masked_attention_pattern(f, s, q[0].astype(np.float64), k[0].astype(np.float64),
                                         v[0].astype(np.float64), kind, sink)
    assert_within(block_errors(o[0].float().cpu().numpy(), ref, np.arange(f * s), 64), "token vs reference")
