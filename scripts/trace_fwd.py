"""Per-step event timeline of the forward kernel (needs a -DRADIAL_TRACE build):
    RADIAL_CUDA_LIB=variants/trace/libradial_cuda.so python scripts/trace_fwd.py"""
import ctypes
import os
import sys

import numpy as np

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
    CT, ST, EV = 4, 64, 24
    buf = torch.zeros(CT * ST * EV, dtype=torch.int64, device="cuda")
    lib = ctypes.CDLL(P.library_path())
    for _ in range(3):
        P.masked_attention(q, k, v, lay)
    assert lib.radial_cuda_debug_trace(ctypes.c_void_p(buf.data_ptr())) == 0
    P.masked_attention(q, k, v, lay)
    torch.cuda.synchronize()
    t = buf.view(CT, ST, EV).cpu().numpy().astype(np.int64)
    names = ["A.wait", "A.S", "A.P0", "A.P1", "B.wait", "B.S", "B.P0", "B.P1",
             "M.PA0", "M.PA1", "M.PB0", "M.PB1", "M.SA", "M.SB", "A.ld", "A.max", "M.kfull", "M.vfull", "L.K", "L.V", "M.vw0", "M.kw0"]
    for c in range(CT):
        base = t[c, 1, 1]
        print(f"CTA {c}: times relative to step-1 A.S (clk)")
        for j in range(8, 16):
            print(j, " ".join(f"{nm}={int(t[c, j, e] - base) if t[c, j, e] else -1:>7}" for e, nm in enumerate(names)))
        js = np.arange(10, 60)
        def d(a, b, jo=0):
            x = t[c, js + jo, b] - t[c, js, a]
            ok = (t[c, js + jo, b] > 0) & (t[c, js, a] > 0)
            return float(np.median(x[ok])) if ok.any() else float("nan")
        print(" period A (A.S j->j+1):", d(1, 1, 1), " period B:", d(5, 5, 1))
        print(" softmax A: S->P0", d(1, 2), " S->P1", d(1, 3), "| B: S->P0", d(5, 6), " S->P1", d(5, 7))
        print(" S issue->seen A", d(12, 1), " B", d(13, 5))
        print(" P arrive->MMA sees A0", d(2, 8), " A1", d(3, 9), " B0", d(6, 10), " B1", d(7, 11))
        print(" A.P1 -> next A.S (PV_A + S_A + latency):", d(3, 1, 1), " B:", d(7, 5, 1))
        print(" A wait-start -> S seen (idle):", d(0, 1))
        print(" MMA: SB issued -> kfull(j+1) seen", d(13, 16, 1), " -> vfull seen", d(13, 17, 1), " K(j) load issue - S_B(j-2) seen", d(5, 18, 2), " V load issue", d(5, 19, 2))
        print(" K(j) issue -> MMA kfull(j) seen", d(18, 16), " V(j) issue -> vfull seen (step j+1)", d(19, 17, 1))
        print(" A: S seen -> ld done", d(1, 14), " ld -> max", d(14, 15), " max -> P0", d(15, 2))


if __name__ == "__main__":
    main()
