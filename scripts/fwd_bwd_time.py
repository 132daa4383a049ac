"""Forward and backward time at a BASELINE config for the library this process loads
(RADIAL_CUDA_LIB selects a variant build), for same-box A/B runs of work-order and kernel
variants.

    python scripts/fwd_bwd_time.py --config hunyuan132 ; RADIAL_CUDA_LIB=variants/x/libradial_cuda.so python ...
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
    ap.add_argument("--fwd-iters", type=int, default=10)
    ap.add_argument("--bwd-iters", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = CONFIGS[a.config]
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    fl = 4.0 * lay.kept_blocks() * B * B * d * H
    tf = timeit(lambda: P.masked_attention(q, k, v, lay, out=o, lse=lse, return_lse=True), a.fwd_iters)
    tb = timeit(lambda: P.masked_attention_backward(q, k, v, o, lse, do, lay), a.bwd_iters)
    print(json.dumps({"config": a.config, "lib": os.environ.get("RADIAL_CUDA_LIB", "in-tree"),
                      "fwd_ms": tf, "fwd_tflops": fl / tf / 1e9, "bwd_ms": tb, "bwd_tflops": 2.5 * fl / tb / 1e9}))


if __name__ == "__main__":
    main()
