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
