"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): K1 mask builds (radial, spatial, power; tiny and ragged shapes),
K2 forward (block layout, token-exact, scatter epilogue), K4 dense, K3 backward, and the
host-buffer pipeline.  Run as

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py

Prints one line per case; exits non-zero on a Python-side failure.  Outputs are also
checked against the fp64 oracle so a silently corrupted run is caught even where the tool
has no coverage (tcgen05 / TMA traffic is invisible to racecheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import oracle as O
    import paper_2506_19852_b200 as P

    torch.cuda.set_device(0)
    cases = [(8, 256, 64, 64, 2), (5, 300, 128, 128, 2), (3, 77, 128, 64, 1)]  # f, s, B, d, H
    for kind in (P.PatternSpec.radial(True), P.PatternSpec.spatial(1), P.PatternSpec.power(True),
                 P.PatternSpec.sta(1, 40)):
        for f, s, B, _, _ in cases:
            lay = P.device_layout(P.GridShape(f, s), kind, B, cache=False)
            rp, ci = O.blockify(f, s, B, kind=P.PatternKind.names[kind.kind], sink=kind.sink,
                                tw=kind.temporal_window or 0, sw=kind.spatial_window or 0)
            h = lay.host()
            assert np.array_equal(h.row_ptr, rp) and np.array_equal(h.col_idx, ci), (f, s, B, kind)
    print("mask builds ok", flush=True)
    g = torch.Generator(device="cuda").manual_seed(0)
    for f, s, B, d, H in cases:
        n = f * s
        q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
        lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(True), B)
        o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
        ot = P.masked_attention_pattern(q, k, v, P.GridShape(f, s), P.PatternSpec.radial(True), block_size=B)
        od = P.dense_attention(q, k, v, block_size=B)
        torch.cuda.synchronize()
        host = lay.host()
        rows = np.arange(n)
        for hh in range(H):
            want = O.attention_rows(q[hh].float().cpu().numpy(), k[hh].float().cpu().numpy(),
                                    v[hh].float().cpu().numpy(), B, host.row_ptr, host.col_idx, rows)
            err = np.abs(o[hh].float().cpu().numpy() - want).max()
            assert err < 2e-2, (f, s, B, d, err)
        assert torch.isfinite(ot.float()).all() and torch.isfinite(od.float()).all()
        bufs = [torch.zeros(H + 1, n, d, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
        P.masked_attention_scatter(q, k, v, lay, [b.data_ptr() for b in bufs], 1, H + 1)
        torch.cuda.synchronize()
        assert torch.equal(bufs[0][1:], o) and torch.equal(bufs[1][1:], o)
        if B == 128:
            do = torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16)
            dq, dk, dv = P.masked_attention_backward(q, k, v, o, lse, do, lay)
            torch.cuda.synchronize()
            assert all(torch.isfinite(x.float()).all() for x in (dq, dk, dv))
        hq, hk, hv = (x.cpu().view(torch.int16).numpy().view(np.uint16) for x in (q, k, v))
        oh = P.masked_attention_host(hq, hk, hv, lay)
        assert np.array_equal(oh, o.cpu().view(torch.int16).numpy().view(np.uint16))
        print(f"attention f{f} s{s} B{B} d{d} H{H} ok", flush=True)
    print("SANITIZE_CASES_OK")


if __name__ == "__main__":
    main()
