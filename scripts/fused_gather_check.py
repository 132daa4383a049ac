"""Fused head-parallel reassembly through torch symmetric memory (run under torchrun,
any number of ranks, NCCL): every rank computes its heads with masked_attention_scatter,
storing O rows into all ranks' full-O buffers; after the barrier each rank's buffer must
equal the single-GPU forward of all heads.  Prints one JSON line from rank 0."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2506_19852_b200 as P
    from paper_2506_19852_b200.heads import HeadParallel
    hp = HeadParallel.from_env("nccl")
    if "--expect-ranks" in sys.argv:
        want = int(sys.argv[sys.argv.index("--expect-ranks") + 1])
        if hp.world != want:
            print(f"fused_gather_check: expected {want} ranks, launched with {hp.world}", file=sys.stderr)
            sys.exit(2)
    if hp.world == 1 and not dist.is_initialized():
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    f, s, d, H, B = 6, 1000, 128, 8, 128
    n = f * s
    g = torch.Generator(device="cuda").manual_seed(21)
    q, k, v = (torch.randn(H, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(), B)
    ref = P.masked_attention(q, k, v, lay)
    full = hp.full_output(H, n, d, force_symmetric=True)
    lo, hi = hp.heads(H)
    P.masked_attention_scatter(q[lo:hi].contiguous(), k[lo:hi].contiguous(), v[lo:hi].contiguous(), lay,
                               full.ptrs, full.head_base, H)
    full.sync()
    torch.cuda.synchronize()
    ok = bool(torch.equal(full.out, ref))
    if hp.rank == 0:
        print(json.dumps({"ranks": hp.world, "destinations": len(full.ptrs), "identical": ok}))
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
