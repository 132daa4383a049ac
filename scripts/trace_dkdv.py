"""Per-block event timeline of the dK/dV kernel (needs a -DRADIAL_TRACE build):
    RADIAL_CUDA_LIB=vtrace/tr_bwd/libradial_cuda.so python scripts/trace_dkdv.py"""
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
    P.masked_attention_backward(q, k, v, o, lse, do, lay)
    assert lib.radial_cuda_debug_btrace(ctypes.c_void_p(buf.data_ptr())) == 0
    P.masked_attention_backward(q, k, v, o, lse, do, lay)
    torch.cuda.synchronize()
    t = buf.view(4, 64, 16).cpu().numpy().astype(np.int64)
    names = ["M.S", "M.dK", "M.dP", "M.pseen", "M.dV", "W0.s", "-", "W0.p", "W0.dp", "W0.ds", "W1.p", "W1.ds"]
    for c in range(4):
        base = t[c, 1, 0]
        print(f"CTA {c}")
        for j in range(8, 14):
            print(j, " ".join(f"{nm}={int(t[c, j, e] - base) if t[c, j, e] else -1:>7}" for e, nm in enumerate(names) if nm != "-"))
        js = np.arange(4, 40)

        def d_(a, b, jo=0):
            x = t[c, js + jo, b] - t[c, js, a]
            ok = (t[c, js + jo, b] > 0) & (t[c, js, a] > 0)
            return float(np.median(x[ok])) if ok.any() else float("nan")
        print(" period (S issue):", d_(0, 0, 1), " W0 s->p:", d_(5, 7), " W1 s->p:", d_(5, 10), " p->MMA sees:", d_(10, 3))
        print(" M.S issue -> W0 s seen:", d_(0, 5), " dP issue -> W0 dp seen:", d_(2, 8), " W0 dp->ds:", d_(8, 9))
        print(" pseen -> dV issued:", d_(3, 4), " dV issued -> next S issued:", d_(4, 0, 1), " next S->dK issued", d_(0, 1, 1))


if __name__ == "__main__":
    main()
