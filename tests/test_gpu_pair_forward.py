"""GPU parity of the opt-in CTA-pair forward (csrc/attn_fwd2.cu, RADIAL_FWD_PAIR=1): the same
per-(head, query block) gate against the fp64 oracle as the product kernel, for the sparse
layout (ragged tails, odd block counts, sink on / off) and the dense comparator.  The switch is
read once per process, so each case runs in a subprocess."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SNIPPET = r'''
import json, sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import oracle as O
import paper_2506_19852_b200 as P
from tests._util import block_errors, instance_bf16, to_torch_bf16
f, s, H, sink, dense = {f}, {s}, {H}, {sink}, {dense}
B = d = 128
n = f * s
q, k, v = instance_bf16(f, s, d, H, 7)
tq, tk, tv = (to_torch_bf16(x) for x in (q, k, v))
lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.dense() if dense else P.PatternSpec.radial(sink), B)
o = (P.dense_attention(tq, tk, tv, block_size=B) if dense else P.masked_attention(tq, tk, tv, lay))
torch.cuda.synchronize()
h = lay.host()
rows = np.arange(n)
worst_abs = worst_rel = 0.0
for hh in range(H):
    want = O.attention_rows(q[hh], k[hh], v[hh], B, h.row_ptr, h.col_idx, rows)
    for a, r in block_errors(o[hh].float().cpu().numpy(), want, rows, B).values():
        worst_abs, worst_rel = max(worst_abs, a), max(worst_rel, r)
print(json.dumps({{"abs": worst_abs, "rel": worst_rel}}))
'''


@pytest.mark.parametrize("f,s,H,sink,dense", [(8, 1000, 2, True, False), (5, 777, 3, False, False),
                                              (3, 1100, 2, True, True)])
def test_pair_forward_vs_oracle(f, s, H, sink, dense):
    code = _SNIPPET.format(root=ROOT, f=f, s=s, H=H, sink=sink, dense=dense)
    env = dict(os.environ, RADIAL_FWD_PAIR="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["abs"] <= 2e-2 and got["rel"] <= 1e-2, got
