"""External comparator: FlashAttention-4 (the CuTe-DSL sm100 kernels vendored in vllm 0.22,
`vllm.vllm_flash_attn.cute`) against our K2 / K4 on the same box, same clock, same inputs.

Legs (H33 by default, bf16, d 128):
  ours_sparse   K2 over the radial block layout (kept-block FLOPs)
  ours_dense    K4, the dense comparator
  fa4_dense     FA4 forward, no mask
  fa4_union     FA4 block-sparse forward. FA4's sparse Q block is q_stage x tile_m = 256 rows, so
                each 256-row pair of our 128-row layout rows runs the UNION of the two rows'
                KV lists for both 128-row tiles: a superset of the radial mask (more FLOPs, and
                not the same output). Reported on its executed FLOPs and on the kept-block FLOPs.
  (--bwd) ours_bwd and fa4_dense_bwd (fwd+bwd minus fwd).

Library code, measurement only: nothing here is on the product path.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {"hunyuan33": (33, 3600, 24), "wan21": (21, 3600, 40), "mochi28": (28, 1590, 24)}


def timed(fn, it, warm=3):
    import torch
    for _ in range(warm):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hunyuan33", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--bwd", action="store_true")
    a = ap.parse_args()

    import numpy as np
    import torch
    import paper_2506_19852_b200 as P
    from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd, flash_attn_func
    from vllm.vllm_flash_attn.cute.block_sparsity import BlockSparseTensorsTorch

    f, s, H = CONFIGS[a.config]
    d, B = 128, 128
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    host = lay.host()
    kept = host.kept_blocks()
    R = host.grid_rows
    blk = 4.0 * B * B * d * H
    fl_kept = kept * blk
    fl_dense = 4.0 * n * n * d * H
    res = {"config": a.config, "n": n, "heads": H, "kept_blocks": kept}

    # FA4 wants (batch, seqlen, heads, d); a permuted view of our [H][n][d] keeps stride(-1)=1,
    # so both kernels read the same bytes.
    fq, fk, fv = (t.permute(1, 0, 2).unsqueeze(0) for t in (q, k, v))

    ms = timed(lambda: P.masked_attention(q, k, v, lay), a.iters)
    res["ours_sparse"] = {"ms": ms, "tflops": fl_kept / ms / 1e9}
    ms = timed(lambda: P.dense_attention(q, k, v), max(3, a.iters // 2))
    res["ours_dense"] = {"ms": ms, "tflops": fl_dense / ms / 1e9}

    try:
        out, _ = _flash_attn_fwd(fq, fk, fv)
        ref = P.dense_attention(q, k, v)
        res["fa4_dense_vs_ours_dense_maxabs"] = float((out[0].permute(1, 0, 2) - ref).abs().max())
        ms = timed(lambda: _flash_attn_fwd(fq, fk, fv), max(3, a.iters // 2))
        res["fa4_dense"] = {"ms": ms, "tflops": fl_dense / ms / 1e9}
    except Exception as e:  # noqa: BLE001 - report, keep the other legs
        res["fa4_dense"] = {"error": f"{type(e).__name__}: {e}"[:400]}

    try:
        rp = host.row_ptr.astype(np.int64)
        ci = host.col_idx.astype(np.int64)
        M = (R + 1) // 2
        rows = []
        for p in range(M):
            a0 = ci[rp[2 * p]:rp[2 * p + 1]]
            a1 = ci[rp[2 * p + 1]:rp[2 * p + 2]] if 2 * p + 1 < R else a0[:0]
            rows.append(np.union1d(a0, a1))
        mx = max(len(r) for r in rows)
        cnt = np.array([len(r) for r in rows], dtype=np.int32)
        idx = np.zeros((M, mx), dtype=np.int32)
        for p, r in enumerate(rows):
            idx[p, :len(r)] = r
        union_tiles = int(sum(len(r) * (2 if 2 * p + 1 < R else 1) for p, r in enumerate(rows)))
        dev = q.device
        bst = BlockSparseTensorsTorch(
            mask_block_cnt=torch.zeros(1, 1, M, dtype=torch.int32, device=dev),
            mask_block_idx=torch.zeros(1, 1, M, 1, dtype=torch.int32, device=dev),
            full_block_cnt=torch.from_numpy(cnt).to(dev).view(1, 1, M),
            full_block_idx=torch.from_numpy(idx).to(dev).view(1, 1, M, mx),
            block_size=(256, 128))
        _flash_attn_fwd(fq, fk, fv, block_sparse_tensors=bst)
        ms = timed(lambda: _flash_attn_fwd(fq, fk, fv, block_sparse_tensors=bst), a.iters)
        res["fa4_union"] = {"ms": ms, "executed_tiles": union_tiles,
                            "tflops_executed": union_tiles * blk / ms / 1e9,
                            "tflops_kept": fl_kept / ms / 1e9}
    except Exception as e:  # noqa: BLE001
        res["fa4_union"] = {"error": f"{type(e).__name__}: {e}"[:400]}

    if a.bwd:
        do = torch.randn_like(q)
        o, lse = P.masked_attention(q, k, v, lay, return_lse=True)
        ms = timed(lambda: P.masked_attention_backward(q, k, v, o, lse, do, lay), max(3, a.iters // 2))
        res["ours_bwd"] = {"ms": ms, "tflops_2p5": 2.5 * fl_kept / ms / 1e9}
        try:
            xq, xk, xv = (t.detach().clone().requires_grad_(True) for t in (fq, fk, fv))
            fdo = do.permute(1, 0, 2).unsqueeze(0)

            def fb():
                out = flash_attn_func(xq, xk, xv)
                out = out[0] if isinstance(out, tuple) else out
                out.backward(fdo)
            ms_fb = timed(fb, 3)
            ms_f = res["fa4_dense"].get("ms", 0.0)
            res["fa4_dense_bwd"] = {"ms_fwd_bwd": ms_fb, "ms": ms_fb - ms_f,
                                    "tflops_2p5": 2.5 * fl_dense / (ms_fb - ms_f) / 1e9}
        except Exception as e:  # noqa: BLE001
            res["fa4_dense_bwd"] = {"error": f"{type(e).__name__}: {e}"[:400]}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
