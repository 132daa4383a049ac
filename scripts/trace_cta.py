"""Per-CTA fixed cost of the forward (needs a -DRADIAL_TRACE build):
    RADIAL_CUDA_LIB=vtr/tre/libradial_cuda.so python scripts/trace_cta.py
start -> first S seen, tile-0 softmax done -> final O ready, final O -> CTA end, steady period."""
import ctypes, os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
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
for _ in range(3): P.masked_attention(q, k, v, lay)
assert lib.radial_cuda_debug_trace(ctypes.c_void_p(buf.data_ptr())) == 0
P.masked_attention(q, k, v, lay)
torch.cuda.synchronize()
t = buf.view(CT, ST, EV).cpu().numpy().astype(np.int64)
for c in range(CT):
    st, en, smd, ofin = t[c,0,22], t[c,1,22], t[c,2,22], t[c,3,22]
    firstS = t[c,0,1]  # A.S at step 0
    # period from steps 10..60
    per = np.median(np.diff(t[c,10:60,1]))
    print(f"CTA {c}: total {en-st} clk; start->first S {firstS-st}; softmax done->O final {ofin-smd}; O final->end {en-ofin}; period {per}")
