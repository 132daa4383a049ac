"""Shared helpers for the GPU parity tests (compare the CUDA path with the oracle)."""
import numpy as np

import oracle as O

# north-star tolerance for bf16 I/O vs the fp64 oracle on the same rounded inputs,
# evaluated per (head, query block) and maximised
MAX_ABS = 2e-2
REL_L2 = 1e-2


def bf16_bits(x_f32: np.ndarray) -> np.ndarray:
    """float32 values that are exactly bf16 -> uint16 bit patterns."""
    return (np.ascontiguousarray(x_f32, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def instance_bf16(f, s, d, heads, seed0=42, q_scale=1.0):
    """random_instance(GridShape(f,s), d, seed0+h) per head (attention.hpp:89-104), rounded
    to bf16 (RNE); returns float32 arrays [H, n, d] holding exactly-bf16 values."""
    n = f * s
    qs, ks, vs = [], [], []
    for h in range(heads):
        q, k, v = O.random_instance(n, d, seed0 + h)
        qs.append(O.bf16_round(q * q_scale))
        ks.append(O.bf16_round(k))
        vs.append(O.bf16_round(v))
    return np.stack(qs), np.stack(ks), np.stack(vs)


def to_torch_bf16(x_f32: np.ndarray, device="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x_f32)).to(device=device, dtype=torch.bfloat16)


def block_errors(got: np.ndarray, want: np.ndarray, rows: np.ndarray, B: int):
    """Per query block (max_abs, rel_l2) over the given rows; got/want [len(rows), d]."""
    out = {}
    blocks = rows // B
    for I in np.unique(blocks):
        sel = blocks == I
        g, w = got[sel].astype(np.float64), want[sel]
        diff = g - w
        mx = float(np.abs(diff).max())
        rel = float(np.linalg.norm(diff) / max(np.linalg.norm(w), 1e-30))
        out[int(I)] = (mx, rel)
    return out


def assert_within(errs: dict, what: str):
    worst_abs = max(v[0] for v in errs.values())
    worst_rel = max(v[1] for v in errs.values())
    assert worst_abs <= MAX_ABS and worst_rel <= REL_L2, (
        f"{what}: worst per-block max-abs {worst_abs:.3e} (<= {MAX_ABS}), "
        f"rel-L2 {worst_rel:.3e} (<= {REL_L2})")
    return worst_abs, worst_rel


def bf16_pipeline_bwd(q, k, v, do, B, row_ptr, col_idx):
    """The backward's bf16 noise floor: exact fp64 math except at the points where K3 rounds
    (O stored as bf16 by the forward and used for D = rowsum(dO*O); P and dS rounded to bf16 as
    MMA operands; P from an fp32 exponent).  Dense n x n restatement, small shapes only."""
    n, d = q.shape
    sc = 1.0 / np.sqrt(d)
    mask = np.zeros((n, n), bool)
    for I in range(len(row_ptr) - 1):
        for J in col_idx[row_ptr[I]:row_ptr[I + 1]]:
            mask[I * B:(I + 1) * B, int(J) * B:(int(J) + 1) * B] = True
    q64, k64, v64, do64 = (x.astype(np.float64) for x in (q, k, v, do))
    S = np.where(mask, (q64 @ k64.T) * sc, -np.inf)
    e = np.exp(S - S.max(1, keepdims=True))
    p = e / e.sum(1, keepdims=True)
    o_b = O.bf16_round((p @ v64).astype(np.float32)).astype(np.float64)
    p32 = p.astype(np.float32).astype(np.float64)
    ds = p32 * (do64 @ v64.T - (do64 * o_b).sum(1, keepdims=True))
    p_b = O.bf16_round(p32.astype(np.float32)).astype(np.float64)
    ds_b = O.bf16_round(ds.astype(np.float32)).astype(np.float64)
    return (ds_b @ k64) * sc, (ds_b.T @ q64) * sc, p_b.T @ do64


def radial_token_keep(rows, keys, s, sink=True):
    """The reference token rule for the radial kind (mask.hpp:105-154 kept_span with
    k_lo = k_hi = k, plus the sink of mask.hpp:120), vectorised: bool of broadcast(rows, keys)
    global token indices."""
    import torch
    i, k = rows // s, rows % s
    j, l = keys // s, keys % s
    d = (i - j).abs()
    e = torch.where(d <= 1, torch.zeros_like(d), torch.floor(torch.log2(d.clamp_min(1).double())).long())
    # floor(log2 d) from a double: correct a rounding to either side
    e = e - ((1 << e) > d).long() * (d > 1).long()
    e = e + ((1 << (e + 1)) <= d).long() * (d > 1).long()
    pw = 1 << e
    band = pw <= s
    sigma = (s >> e.clamp_max(62)) - 1
    keep = band & ((k - l).abs() <= sigma)
    period = (pw + s - 1) // s
    keep = keep | (~band & (l == k) & (d % period == 0))
    if sink:
        keep = keep | (j == 0)
    return keep
