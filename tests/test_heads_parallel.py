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


def _bench(args, env_extra=None):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=300)


@pytest.mark.parametrize("n", [2, 3])
def test_bench_spawns_its_own_ranks(n):
    """`bench.py --gpus N` without torchrun re-launches itself with N ranks (the driver's
    command shape) and every rank owns its share of the 24 heads (gloo, no GPU)."""
    import json
    r = _bench(["--gpus", str(n), "--dry-run"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == n
    spans = line["heads_per_rank"]
    assert spans[0][0] == 0 and spans[-1][1] == 24
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert line["max_over_ranks"] == float(n)


def test_bench_rejects_world_size_mismatch():
    r = _bench(["--gpus", "2", "--dry-run"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=1" in r.stderr


def test_bench_refuses_more_gpus_than_visible_without_shared_flag():
    """`--gpus N` on a box with fewer devices fails loudly (exit 2) instead of running all heads
    on one GPU; here (no GPU at all) any N > 0 is more than visible."""
    r = _bench(["--gpus", "2"])
    assert r.returncode == 2
    assert "CUDA device(s) visible" in r.stderr


@pytest.mark.gpu
def test_bench_shared_gpu_runs_the_multi_rank_path():
    """Two ranks on the one GPU of a gpurun box (gloo collectives): the whole N > 1 bench path
    completes and the line is marked as a plumbing test."""
    import json
    r = _bench(["--gpus", "2", "--shared-gpu", "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
                "--no-extra", "--no-bwd", "--no-dense"])
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["heads_per_rank"] == [12, 12]
    assert "shared_gpu_plumbing_test" in line and line["gpu_launches"] >= 4
