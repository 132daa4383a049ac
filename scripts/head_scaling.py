"""Per-rank forward time at the head shares of N = 1, 2, 4, 8 GPUs (24 / N heads of H33),
timed on one GPU: strong-scaling efficiency of the head-parallel split without NCCL."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = 33, 3600, 24, 128, 128
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    base = None
    for N in (1, 2, 4, 8):
        h = H // N
        qs, ks, vs = q[:h].contiguous(), k[:h].contiguous(), v[:h].contiguous()
        for _ in range(3):
            P.masked_attention(qs, ks, vs, lay)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        it = 10
        for _ in range(it):
            P.masked_attention(qs, ks, vs, lay)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        base = base or ms
        print(f"N={N} heads/rank={h:2d}: {ms:8.3f} ms  efficiency vs N=1: {base / (N * ms):.3f}")


if __name__ == "__main__":
    main()
