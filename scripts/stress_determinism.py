"""Race detector by determinism: the forward and backward kernels have no atomics and a
fixed reduction order, so repeated calls on the same inputs must be bit-identical.  Runs
N forward+backward passes at a BASELINE shape (and the token-exact forward) and compares
every output with the first pass.  Prints one JSON line; exit 1 on any mismatch."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hunyuan33", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = CONFIGS[a.config]
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(31)
    q, k, v, do = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    shape, pat = P.GridShape(f, s), P.PatternSpec.radial()
    lay = P.device_layout(shape, pat, B)
    ref = None
    mism = {}
    for it in range(a.iters):
        o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
        outs = {"o": o, "lse": lse, "o_token": P.masked_attention_pattern(q, k, v, shape, pat, block_size=B)}
        if B == 128:
            dq, dk, dv = P.masked_attention_backward(q, k, v, o, lse, do, lay)
            outs.update(dq=dq, dk=dk, dv=dv)
        torch.cuda.synchronize()
        if ref is None:
            ref = {kk: t.clone() for kk, t in outs.items()}
            continue
        for kk, t in outs.items():
            if not torch.equal(t, ref[kk]):
                mism[kk] = mism.get(kk, 0) + 1
    print(json.dumps({"config": a.config, "iters": a.iters, "tensors": sorted(ref), "mismatches": mism}))
    sys.exit(1 if mism else 0)


if __name__ == "__main__":
    main()
