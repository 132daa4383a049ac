"""One forward + backward at a BASELINE config, for ncu (launch list / full capture)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mochi28", choices=sorted(CONFIGS))
    a = ap.parse_args()
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = CONFIGS[a.config]
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    P.masked_attention_backward(q, k, v, o, lse, do, lay)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
