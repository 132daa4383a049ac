"""Per-block event timeline of the dQ kernel (needs a -DRADIAL_TRACE build):
    RADIAL_CUDA_LIB=vtrace/tr_bwd/libradial_cuda.so python scripts/trace_dq.py"""
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
    q, k, v, do = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    lib = ctypes.CDLL(P.library_path())
    buf = torch.zeros(4 * 64 * 16, dtype=torch.int64, device="cuda")
    dq = torch.empty_like(q)
    P.masked_attention_backward(q, k, v, o, lse, do, lay)
    assert lib.radial_cuda_debug_btrace(ctypes.c_void_p(buf.data_ptr())) == 0
    # the dK/dV kernel runs second and overwrites the buffer: time a dQ-only call
    os.environ["RADIAL_BWD_DQ_ONLY"] = "1"
    P.masked_attention_backward(q, k, v, o, lse, do, lay)
    torch.cuda.synchronize()
    t = buf.view(4, 64, 16).cpu().numpy().astype(np.int64)
    names = {1: "M.S", 2: "M.dP", 3: "M.dsseen", 5: "W0.s", 6: "W0.ds"}
    for c in range(4):
        base = t[c, 1, 1]
        print(f"CTA {c}")
        for j in range(8, 13):
            print(j, " ".join(f"{nm}={int(t[c, j, e] - base):>7}" for e, nm in names.items()))
        js = np.arange(4, 40)

        def d_(a, b, jo=0):
            x = t[c, js + jo, b] - t[c, js, a]
            ok = (t[c, js + jo, b] > 0) & (t[c, js, a] > 0)
            return float(np.median(x[ok])) if ok.any() else float("nan")
        print(" period (S issue):", d_(1, 1, 1), " W0 s->ds:", d_(5, 6), " ds->MMA sees (next block):", d_(6, 3, 1))
        print(" S issue -> W0 s seen:", d_(1, 5), " S->dP issued:", d_(1, 2), " dP -> dsseen(j+1):", d_(2, 3, 1))


if __name__ == "__main__":
    main()
