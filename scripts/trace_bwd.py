"""Per-block event timeline of the dQ backward kernel (needs a -DRADIAL_TRACE build)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_19852_b200 as P
    f, s, H, d, B = 28, 1590, 24, 128, 128
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
    buf = torch.zeros(4 * 64 * 16, dtype=torch.int64, device="cuda")
    lib = ctypes.CDLL(P.library_path())
    P.masked_attention_backward(q, k, v, o, lse, do, lay)
    assert lib.radial_cuda_debug_btrace(ctypes.c_void_p(buf.data_ptr())) == 0
    P.masked_attention_backward(q, k, v, o, lse, do, lay)
    torch.cuda.synchronize()
    t = buf.view(4, 64, 16).cpu().numpy().astype(np.int64)
    names = {0: "M.kfull", 1: "M.S0", 2: "M.S1", 3: "M.ds0", 4: "M.ds1", 5: "W0.s", 6: "W0.ds", 7: "W1.s", 8: "W1.ds"}
    for c in range(2):
        base = t[c, 1, 0]
        print(f"CTA {c} (dkdv kernel overwrote nothing: dq only)")
        for j in range(6, 12):
            print(j, " ".join(f"{nm}={int(t[c, j, e] - base) if t[c, j, e] else -1:>7}" for e, nm in names.items()))
        js = np.arange(4, 40)

        def d_(a, b, jo=0):
            x = t[c, js + jo, b] - t[c, js, a]
            ok = (t[c, js + jo, b] > 0) & (t[c, js, a] > 0)
            return float(np.median(x[ok])) if ok.any() else float("nan")
        print(" period (kfull j->j+1):", d_(0, 0, 1))
        print(" WG0 s->ds:", d_(5, 6), " WG1 s->ds:", d_(7, 8))
        print(" S0 commit -> W0 sees:", d_(1, 5), " S1 commit -> W1 sees:", d_(2, 7))
        print(" W0 ds -> MMA sees:", d_(6, 3), " W1 ds -> MMA sees:", d_(8, 4))
        print(" kfull -> S0 commit:", d_(0, 1), " S0 commit -> S1 commit:", d_(1, 2))


if __name__ == "__main__":
    main()
