"""Last-P-part arrival of tile 0's warp on sub-partition Q relative to warp 4 (sub-partition 0),
from a -DRADIAL_TRACE -DRADIAL_TRACE_WARPQ=Q build (event 23 vs event 3)."""
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
    js = np.arange(8, 60)
    dlt = (t[:, js, 23] - t[:, js, 3]).ravel()
    ok = (t[:, js, 23] > 0).ravel() & (t[:, js, 3] > 0).ravel()
    print(f"Q={sys.argv[1] if len(sys.argv) > 1 else '?'}: P1 arrival minus warp 4's: median {np.median(dlt[ok]):.0f} clk, "
          f"p90 {np.percentile(dlt[ok], 90):.0f}")


if __name__ == "__main__":
    main()
