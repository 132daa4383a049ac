"""Token-exact forward (masked_attention(inst, PatternSpec)) vs the block-layout forward at
H33: the cost of the per-row keep mask inside K2."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timeit(fn, it=10):
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
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = 33, 3600, 24, 128, 128
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    shape, pat = P.GridShape(f, s), P.PatternSpec.radial()
    lay = P.device_layout(shape, pat, B)
    tb = timeit(lambda: P.masked_attention(q, k, v, lay))
    tt = timeit(lambda: P.masked_attention_pattern(q, k, v, shape, pat, block_size=B))
    fl = 4.0 * lay.kept_blocks() * B * B * d * H
    print(f"block layout: {tb:.2f} ms ({fl / tb / 1e9:.0f} TF/s)   token-exact: {tt:.2f} ms "
          f"({fl / tt / 1e9:.0f} TF/s over the same blocks)  ratio {tt / tb:.3f}")


if __name__ == "__main__":
    main()
