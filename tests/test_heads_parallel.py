"""CPU tests of the head-parallel multi-GPU logic with world_size 2 over
gloo: head partitioning, max-over-ranks timing and the O all-gather (C1)."""
import os
import socket

import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_head_slice_partitions_every_head_exactly_once():
    from paper_2506_19852_b200.heads import head_slice
    for H in (1, 2, 3, 24, 40, 7):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = head_slice(H, world, r)
                assert 0 <= lo <= hi <= H
                assert hi - lo in (H // world, H // world + 1)
                seen.extend(range(lo, hi))
            assert seen == list(range(H))
    with pytest.raises(ValueError):
        head_slice(4, 2, 2)


def _worker(rank, world, port, heads, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2506_19852_b200.heads import HeadParallel
    hp = HeadParallel.from_env("gloo")
    try:
        lo, hi = hp.heads(heads)
        # stand-in per-head result: head index broadcast over [n, d]
        local = torch.arange(lo, hi, dtype=torch.float32)[:, None, None].expand(hi - lo, 5, 3).contiguous()
        full = hp.gather_heads(local, heads)
        hp.barrier()
        mx = hp.max(float(rank + 1) * 1.5)
        q.put((rank, (lo, hi), full.tolist(), mx))
    finally:
        hp.close()


@pytest.mark.parametrize("heads", [24, 5])
def test_two_rank_gloo_head_parallel(heads):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, heads, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    res.sort()
    (r0, s0, full0, m0), (r1, s1, full1, m1) = res
    assert s0[0] == 0 and s0[1] == s1[0] and s1[1] == heads
    want = [[[float(h)] * 3] * 5 for h in range(heads)]
    assert full0 == want and full1 == want
    assert m0 == m1 == 3.0
