"""One sparse and one dense forward at a BASELINE config, for ncu (launch list / full capture).

    ncu --set full -k regex:radial_attn_fwd -c 1 python scripts/profile_step.py --config hunyuan33
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hunyuan33", choices=sorted(CONFIGS))
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--token", action="store_true", help="token-exact forward (masked_attention_pattern)")
    ap.add_argument("--iters", type=int, default=1)
    a = ap.parse_args()
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = CONFIGS[a.config]
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    for _ in range(a.iters):
        if a.token:
            P.masked_attention_pattern(q, k, v, P.GridShape(f, s), P.PatternSpec.radial(), block_size=B)
            continue
        P.masked_attention(q, k, v, lay, return_lse=True)
        if a.dense:
            P.dense_attention(q, k, v, block_size=B, return_lse=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
