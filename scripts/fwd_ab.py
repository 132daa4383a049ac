"""Forward timing at a BASELINE config for the kernel this process selects
(default: one-CTA K2; RADIAL_FWD_PAIR=1: the CTA-pair kernel), sparse and dense, plus a
checksum of O so two runs can be compared.

    python scripts/fwd_ab.py [--config hunyuan33] ; RADIAL_FWD_PAIR=1 python scripts/fwd_ab.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402


def timeit(fn, it):
    import torch
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hunyuan33", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--no-dense", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = CONFIGS[a.config]
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    torch.cuda.synchronize()
    fl = 4.0 * lay.kept_blocks() * B * B * d * H
    ts = timeit(lambda: P.masked_attention(q, k, v, lay, out=o, lse=lse, return_lse=True), a.iters)
    rec = {"config": a.config, "pair": os.environ.get("RADIAL_FWD_PAIR", "0") == "1",
           "sparse_ms": ts, "sparse_tflops": fl / ts / 1e9,
           "o_sum": float(o.float().sum()), "o_abs": float(o.float().abs().sum()), "lse_sum": float(lse.sum())}
    if not a.no_dense:
        od = P.dense_attention(q, k, v, block_size=B)
        td = timeit(lambda: P.dense_attention(q, k, v, block_size=B, out=od), max(2, a.iters // 2))
        rec.update(dense_ms=td, dense_tflops=4.0 * n * n * d * H / td / 1e9, speedup=td / ts,
                   od_sum=float(od.float().sum()))
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
