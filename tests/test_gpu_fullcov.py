"""GPU parity with FULL coverage at paper scale: every (head, query block) pair of the
H33 and H132 forwards (and the peaked Q x 8 variant at H33) against an fp32 blockwise
restatement of the reference rule, computed on the GPU from the CSR itself.

The rule checked is radial::masked_attention(inst, layout) (reference
attention.hpp:229-270): query row u attends every key of every kept block of its block
row (clipped to n), softmax over exactly those keys.  The restatement gathers each
query block's kept K/V blocks by index from the CSR (``row_ptr`` / ``col_idx``, the
bytes the K1 tests pin to the reference), so a single miswired work-list entry in any
chunk shows up in that block's error -- SURVEY 7 shows such an error is invisible to a
global metric, hence the per-(head, block) gate (max-abs <= 2e-2, rel-L2 <= 1e-2).

The restatement itself is pinned against the fp64 oracle on sampled blocks in the same
test, so the chain is kernel == fp32 restatement == fp64 oracle == reference.
"""
import numpy as np
import pytest

import oracle as O
from tests._util import MAX_ABS, REL_L2, assert_within, block_errors, radial_token_keep

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU test on a box without CUDA"
    import paper_2506_19852_b200 as P
    return P


def _padded_lists(row_ptr, col_idx, R, device):
    """[R, Lmax] int64 block indices per query block, padded with R (an all-zero block)."""
    import torch
    rp = torch.from_numpy(row_ptr.astype(np.int64)).to(device)
    ci = torch.from_numpy(col_idx.astype(np.int64)).to(device)
    lens = rp[1:] - rp[:-1]
    Lmax = int(lens.max().item())
    rows = torch.repeat_interleave(torch.arange(R, device=device), lens)
    pos = torch.arange(ci.numel(), device=device) - rp[rows]
    idx = torch.full((R, Lmax), R, dtype=torch.int64, device=device)
    idx[rows, pos] = ci
    return idx, lens


def fp32_blockwise(q, k, v, idx, lens, B, n, scale, blocks=None, rows_per_batch=None, token_keep=None):
    """fp32 restatement of attention.hpp:238-268 for one head, query blocks `blocks` (all by
    default): O [len(blocks) * B, d] (rows >= n are zero) and lse [len(blocks) * B].
    q/k/v: bf16 [n, d] on the GPU; idx: padded kept-block lists (pad = R)."""
    import torch
    R = idx.shape[0]
    d = q.shape[1]
    pad = R * B + B - n  # one extra all-zero block at index R for the padding entries
    qf = torch.nn.functional.pad(q.float(), (0, 0, 0, pad)).view(R + 1, B, d)
    kf = torch.nn.functional.pad(k.float(), (0, 0, 0, pad)).view(R + 1, B, d)
    vf = torch.nn.functional.pad(v.float(), (0, 0, 0, pad)).view(R + 1, B, d)
    blocks = torch.arange(R, device=q.device) if blocks is None else blocks
    outs, lses = [], []
    Lmax = idx.shape[1]
    nb = rows_per_batch or max(1, int(2 ** 29 // (Lmax * B * B * 4)))  # S of a batch <= 512 MB
    ar = torch.arange(B, device=q.device)
    for b0 in range(0, blocks.numel(), nb):
        bl = blocks[b0:b0 + nb]
        L = int(lens[bl].max().item())
        ib = idx[bl, :L]                                             # [nb, L]
        kg = kf[ib].reshape(bl.numel(), L * B, d)                    # [nb, L*B, d]
        vg = vf[ib].reshape(bl.numel(), L * B, d)
        key = (ib[:, :, None] * B + ar).reshape(bl.numel(), 1, L * B)
        ok = (ib[:, :, None] < R).expand(-1, -1, B).reshape(bl.numel(), 1, L * B) & (key < n)
        s = torch.bmm(qf[bl], kg.transpose(1, 2)) * scale           # [nb, B, L*B]
        if token_keep is not None:
            qrow = (bl[:, None] * B + ar).reshape(bl.numel(), B, 1)
            ok = ok & token_keep(qrow, key)
        s = s.masked_fill(~ok, float("-inf"))
        m = s.amax(dim=2, keepdim=True)
        p = torch.exp(s - m)
        l = p.sum(dim=2, keepdim=True)
        outs.append((torch.bmm(p, vg) / l).reshape(-1, d))
        lses.append((m + torch.log(l)).reshape(-1))
    return torch.cat(outs), torch.cat(lses)


def _per_block_errors(got, want, B, ulp_slack=False):
    """Per query block (max_abs, rel_l2) on the GPU; got/want [nb * B, d] fp32.  With
    ulp_slack the absolute error of each element is first reduced by the bf16 half-ulp of the
    reference value (2^-8 |want|): the rounding any bf16 output of that value must carry."""
    import torch
    diff = (got - want).view(-1, B, got.shape[1])
    w = want.view(-1, B, got.shape[1])
    ad = diff.abs()
    if ulp_slack:
        ad = (ad - w.abs() * 2.0 ** -8).clamp_min(0.0)
    mx = ad.amax(dim=(1, 2))
    rel = torch.linalg.vector_norm(diff, dim=(1, 2)) / torch.linalg.vector_norm(w, dim=(1, 2)).clamp_min(1e-30)
    return mx, rel


def _full_coverage(P, f, s, H, q_scale=1.0, seed=4321, pin_heads=(0,), B=128, d=128):
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    n = f * s
    scale = 1.0 / np.sqrt(d)
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.randn(H, n, d, device="cuda", generator=g) * q_scale).to(torch.bfloat16)
    k = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    torch.cuda.synchronize()
    host = lay.host()
    R = host.grid_rows
    idx, lens = _padded_lists(host.row_ptr, host.col_idx, R, q.device)
    worst_abs = worst_rel = worst_lse = 0.0
    checked = 0
    for h in range(H):
        want, want_lse = fp32_blockwise(q[h], k[h], v[h], idx, lens, B, n, scale)
        got = torch.nn.functional.pad(o[h].float(), (0, 0, 0, R * B - n))
        valid = torch.arange(R * B, device=q.device) < n
        want = want * valid[:, None]
        # peaked softmax (Q x 8): rows are nearly one-hot, so O is a single V row with |O| up to
        # ~6 over 365M outputs, where the bf16 output rounding alone reaches 0.016: the max-abs
        # gate is taken after removing that intrinsic half-ulp (rel-L2 is unchanged)
        mx, rel = _per_block_errors(got, want, B, ulp_slack=q_scale != 1.0)
        worst_abs = max(worst_abs, float(mx.max()))
        worst_rel = max(worst_rel, float(rel.max()))
        worst_lse = max(worst_lse, float((lse[h] - want_lse[:n]).abs().max()))
        checked += R
        assert float(mx.max()) <= MAX_ABS and float(rel.max()) <= REL_L2, (
            f"f{f} head {h}: block {int(rel.argmax())} rel-L2 {float(rel.max()):.3e}, "
            f"block {int(mx.argmax())} max-abs {float(mx.max()):.3e}")
        if h in pin_heads:
            # pin the restatement to the fp64 oracle (and so to the reference) on sampled blocks
            rng = np.random.default_rng(h)
            blocks = sorted({0, R // 2, R - 1} | set(rng.integers(0, R, 3).tolist()))
            rows = np.concatenate([np.arange(I * B, min(n, (I + 1) * B)) for I in blocks])
            qh, kh, vh = (x[h].float().cpu().numpy() for x in (q, k, v))
            ref = O.attention_rows(qh, kh, vh, B, host.row_ptr, host.col_idx, rows)
            mine = want[torch.from_numpy(rows).to(q.device)].cpu().numpy()
            assert np.abs(mine - ref).max() < 1e-4, "fp32 restatement disagrees with the fp64 oracle"
            if q_scale == 1.0:
                assert_within(block_errors(o[h].float().cpu().numpy()[rows], ref, rows, B), f"f{f} head {h} vs fp64")
    assert checked == H * R
    assert worst_lse <= 2e-3, worst_lse
    del q, k, v, o, lse
    torch.cuda.empty_cache()
    return worst_abs, worst_rel


def test_full_coverage_hunyuan33(P):
    """BASELINE configs[1]: all 24 x 929 (head, query block) pairs."""
    wa, wr = _full_coverage(P, 33, 3600, 24)
    print(f"H33 full coverage: worst per-block max-abs {wa:.3e}, rel-L2 {wr:.3e}")


def test_full_coverage_hunyuan33_peaked(P):
    """The peaked variant (Q x 8: 'always also run') at H33, every pair."""
    wa, wr = _full_coverage(P, 33, 3600, 24, q_scale=8.0, seed=77)
    print(f"H33 Qx8 full coverage: worst per-block max-abs {wa:.3e}, rel-L2 {wr:.3e}")


def test_full_coverage_hunyuan132(P):
    """BASELINE configs[4] (475k tokens): all 24 x 3,713 (head, query block) pairs."""
    wa, wr = _full_coverage(P, 132, 3600, 24, seed=132)
    print(f"H132 full coverage: worst per-block max-abs {wa:.3e}, rel-L2 {wr:.3e}")


@pytest.mark.parametrize("f,s,H", [(21, 3600, 40), (28, 1590, 24)], ids=["wan21", "mochi28"])
def test_full_coverage_other_configs(P, f, s, H):
    """BASELINE configs[2] and [3]: every (head, query block) pair of the forward."""
    wa, wr = _full_coverage(P, f, s, H, seed=f * 100 + H)
    print(f"f{f} s{s} full coverage: worst per-block max-abs {wa:.3e}, rel-L2 {wr:.3e}")


@pytest.mark.parametrize("B,d", [(64, 128), (64, 64), (128, 64)])
def test_full_coverage_other_tile_shapes_mochi28(P, B, d):
    """The other K2 instantiations (block 64 and / or head_dim 64) at the M28 shape, every
    (head, query block) pair."""
    wa, wr = _full_coverage(P, 28, 1590, 24, seed=B * 1000 + d, B=B, d=d)
    print(f"M28 B{B} d{d} full coverage: worst per-block max-abs {wa:.3e}, rel-L2 {wr:.3e}")


def test_dense_comparator_hunyuan33_sampled(P):
    """K4 at the headline H33 shape (118,800 keys per row) on sampled query blocks of every
    head, against the fp32 dense restatement (dense_attention, attention.hpp:141-163)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    f, s, H, B, d = 33, 3600, 24, 128, 128
    n = f * s
    R = (n + B - 1) // B
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    o = P.dense_attention(q, k, v, block_size=B)
    torch.cuda.synchronize()
    full = torch.arange(R, device="cuda").expand(R, R).contiguous()
    lens = torch.full((R,), R, device="cuda")
    rng = np.random.default_rng(1)
    for h in range(H):
        blocks = torch.tensor(sorted({0, R - 1} | set(rng.integers(0, R, 2).tolist())), device="cuda")
        want, _ = fp32_blockwise(q[h], k[h], v[h], full, lens, B, n, 1.0 / np.sqrt(d), blocks, rows_per_batch=2)
        got = torch.nn.functional.pad(o[h].float(), (0, 0, 0, R * B - n)).view(R, B, d)[blocks].reshape(-1, d)
        rows_ok = ((blocks[:, None] * B + torch.arange(B, device="cuda")) < n).reshape(-1, 1)
        mx, rel = _per_block_errors(got * rows_ok, want * rows_ok, B)
        assert float(mx.max()) <= MAX_ABS and float(rel.max()) <= REL_L2, (h, float(mx.max()), float(rel.max()))


# ------------------------------------------------------------------------------ backward
def fp32_blockwise_bwd(q, k, v, do, idx, lens, B, n, scale):
    """fp32 restatement of the K3 gradients for one head over the kept blocks (no reference
    exists): P = exp(S - lse), dV = P^T dO, dP = dO V^T, D = rowsum(dO o O),
    dS = P o (dP - D), dQ = scale dS K, dK = scale dS^T Q.  q/k/v/do bf16 [n, d] on the GPU;
    returns fp32 dq, dk, dv [R * B, d] (rows >= n are zero)."""
    import torch
    R = idx.shape[0]
    d = q.shape[1]
    o, lse = fp32_blockwise(q, k, v, idx, lens, B, n, scale)
    pad = R * B + B - n
    qf = torch.nn.functional.pad(q.float(), (0, 0, 0, pad)).view(R + 1, B, d)
    kf = torch.nn.functional.pad(k.float(), (0, 0, 0, pad)).view(R + 1, B, d)
    vf = torch.nn.functional.pad(v.float(), (0, 0, 0, pad)).view(R + 1, B, d)
    dof = torch.nn.functional.pad(do.float(), (0, 0, 0, pad)).view(R + 1, B, d)
    lsef = torch.nn.functional.pad(lse, (0, B)).view(R + 1, B)
    valid = (torch.arange((R + 1) * B, device=q.device) < n).view(R + 1, B)
    dvec = (dof[:R] * o.view(R, B, d)).sum(-1) * valid[:R]
    dq = torch.zeros(R, B, d, device=q.device)
    dk = torch.zeros(R + 1, B, d, device=q.device)
    dv = torch.zeros(R + 1, B, d, device=q.device)
    Lmax = idx.shape[1]
    nb = max(1, int(2 ** 28 // (Lmax * B * B * 4)))
    ar = torch.arange(B, device=q.device)
    for b0 in range(0, R, nb):
        bl = torch.arange(b0, min(R, b0 + nb), device=q.device)
        L = int(lens[bl].max().item())
        ib = idx[bl, :L]                                              # [nb, L]
        kg = kf[ib].reshape(bl.numel(), L * B, d)
        vg = vf[ib].reshape(bl.numel(), L * B, d)
        key = (ib[:, :, None] * B + ar).reshape(bl.numel(), 1, L * B)
        ok = (ib[:, :, None] < R).expand(-1, -1, B).reshape(bl.numel(), 1, L * B) & (key < n) & valid[bl][:, :, None]
        s = torch.bmm(qf[bl], kg.transpose(1, 2)) * scale
        p = torch.exp(s - lsef[bl][:, :, None]).masked_fill(~ok, 0.0)      # [nb, B, L*B]
        dp = torch.bmm(dof[bl], vg.transpose(1, 2))
        ds = p * (dp - dvec[bl][:, :, None])
        dq[bl] = torch.bmm(ds, kg) * scale
        # per kept (I, J): dK_J += dS_IJ^T Q_I, dV_J += P_IJ^T dO_I
        ds4 = ds.view(bl.numel(), B, L, B)
        p4 = p.view(bl.numel(), B, L, B)
        dkc = torch.einsum("nilj,nid->nljd", ds4, qf[bl]) * scale        # [nb, L, B, d]
        dvc = torch.einsum("nilj,nid->nljd", p4, dof[bl])
        dk.index_add_(0, ib.reshape(-1), dkc.reshape(-1, B, d))
        dv.index_add_(0, ib.reshape(-1), dvc.reshape(-1, B, d))
    return dq.reshape(-1, d), dk[:R].reshape(-1, d), dv[:R].reshape(-1, d)


def test_backward_restatement_matches_fp64_oracle(P):
    """The fp32 backward restatement equals the fp64 oracle (oracle.attention_bwd) on a small
    ragged shape, so the full-coverage comparison below is anchored to it."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    f, s, d, B = 6, 300, 128, 128
    n = f * s
    rng = np.random.default_rng(9)
    q, k, v, do = (O.bf16_round(rng.standard_normal((n, d)).astype(np.float32)) for _ in range(4))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    host = lay.host()
    R = host.grid_rows
    idx, lens = _padded_lists(host.row_ptr, host.col_idx, R, "cuda")
    t = lambda x: torch.from_numpy(x).cuda().to(torch.bfloat16)
    got = fp32_blockwise_bwd(t(q), t(k), t(v), t(do), idx, lens, B, n, 1.0 / np.sqrt(d))
    want = O.attention_bwd(q, k, v, do, B, host.row_ptr, host.col_idx)
    for g, w in zip(got, want):
        assert np.abs(g[:n].cpu().numpy() - w).max() < 1e-4


def _full_coverage_bwd(P, f, s, H, seed):
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    B, d = 128, 128
    n = f * s
    scale = 1.0 / np.sqrt(d)
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v, do = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    dq, dk, dv = P.masked_attention_backward(q, k, v, o, lse, do, lay)
    torch.cuda.synchronize()
    host = lay.host()
    R = host.grid_rows
    idx, lens = _padded_lists(host.row_ptr, host.col_idx, R, q.device)
    worst = {"dQ": 0.0, "dK": 0.0, "dV": 0.0}
    for h in range(H):
        wants = fp32_blockwise_bwd(q[h], k[h], v[h], do[h], idx, lens, B, n, scale)
        for name, got, want in zip(("dQ", "dK", "dV"), (dq[h], dk[h], dv[h]), wants):
            gotp = torch.nn.functional.pad(got.float(), (0, 0, 0, R * B - n))
            _, rel = _per_block_errors(gotp, want, B)
            glob = float(torch.linalg.vector_norm(gotp - want) / torch.linalg.vector_norm(want))
            worst[name] = max(worst[name], float(rel.max()))
            assert float(rel.max()) <= 1e-2 and glob <= 6e-3, (
                f"f{f} head {h} {name}: block {int(rel.argmax())} rel-L2 {float(rel.max()):.3e}, global {glob:.3e}")
    del q, k, v, do, o, lse, dq, dk, dv
    torch.cuda.empty_cache()
    return worst


def test_backward_full_coverage_mochi28(P):
    """BASELINE configs[3] (the fwd + bwd LoRA path): dQ of every (head, query block) and dK / dV
    of every (head, KV block), 24 x 348 each, against the fp32 restatement."""
    w = _full_coverage_bwd(P, 28, 1590, 24, seed=28)
    print("M28 backward full coverage, worst per-block rel-L2:", {k: f"{v:.3e}" for k, v in w.items()})


def test_backward_full_coverage_hunyuan33(P):
    """The headline shape: every (head, block) of dQ, dK, dV at H33 (24 x 929 each)."""
    w = _full_coverage_bwd(P, 33, 3600, 24, seed=33)
    print("H33 backward full coverage, worst per-block rel-L2:", {k: f"{v:.3e}" for k, v in w.items()})


# ------------------------------------------------------------------------------ token-exact
def test_token_exact_full_coverage_hunyuan33(P):
    """masked_attention(inst, PatternSpec) (attention.hpp:184-225) at the
    headline shape: every (head, query block) against the fp32 restatement over the radial block
    layout with the reference token rule applied inside each block; the restatement is pinned to
    the fp64 token oracle on sampled rows."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    f, s, H, B, d = 33, 3600, 24, 128, 128
    n = f * s
    scale = 1.0 / np.sqrt(d)
    g = torch.Generator(device="cuda").manual_seed(8)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    o = P.masked_attention_pattern(q, k, v, P.GridShape(f, s), P.PatternSpec.radial(), block_size=B)
    torch.cuda.synchronize()
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    host = lay.host()
    R = host.grid_rows
    idx, lens = _padded_lists(host.row_ptr, host.col_idx, R, q.device)
    keep = lambda rows, keys: radial_token_keep(rows, keys, s, sink=True)
    worst_abs = worst_rel = 0.0
    for h in range(H):
        want, _ = fp32_blockwise(q[h], k[h], v[h], idx, lens, B, n, scale, token_keep=keep,
                                 rows_per_batch=4)
        got = torch.nn.functional.pad(o[h].float(), (0, 0, 0, R * B - n))
        valid = torch.arange(R * B, device=q.device) < n
        want = want * valid[:, None]
        mx, rel = _per_block_errors(got, want, B)
        worst_abs, worst_rel = max(worst_abs, float(mx.max())), max(worst_rel, float(rel.max()))
        assert float(mx.max()) <= MAX_ABS and float(rel.max()) <= REL_L2, (
            f"head {h}: block {int(rel.argmax())} rel-L2 {float(rel.max()):.3e}, max-abs {float(mx.max()):.3e}")
        if h == 0:
            rng = np.random.default_rng(3)
            rows = np.sort(rng.choice(n, 300, replace=False))
            qh, kh, vh = (x[h].float().cpu().numpy() for x in (q, k, v))
            ref = O.token_attention_rows(qh, kh, vh, f, s, rows)
            mine = want[torch.from_numpy(rows).to(q.device)].cpu().numpy()
            assert np.abs(mine - ref).max() < 1e-4, "fp32 token restatement disagrees with the fp64 oracle"
    print(f"H33 token-exact full coverage: worst per-block max-abs {worst_abs:.3e}, rel-L2 {worst_rel:.3e}")
