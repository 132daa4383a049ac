"""Head-parallel execution across GPUs: the radial mask is static and
shared by all heads and each head's attention is independent (the
reference has one AttentionInstance per head, attention.hpp:51), so heads are split
evenly across ranks with no collective on the attention path.  The only collective is
the optional all-gather that reassembles O [heads, n, d] where a caller needs it.

One process per GPU (torchrun); NCCL on GPUs, gloo for the CPU tests of this logic.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


def head_slice(heads: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) heads owned by `rank`; sizes differ by at most one, covering all heads."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("head_slice: bad world/rank")
    base, rem = divmod(heads, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


@dataclass
class HeadParallel:
    world: int = 1
    rank: int = 0
    local_rank: int = 0
    backend: str = "none"

    @classmethod
    def from_env(cls, backend: str = "nccl") -> "HeadParallel":
        """Reads RANK / WORLD_SIZE / LOCAL_RANK (torchrun) and initialises the process group."""
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if world > 1:
            import torch
            import torch.distributed as dist
            if backend == "nccl":
                torch.cuda.set_device(local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
        return cls(world, rank, local, backend if world > 1 else "none")

    def _device(self):
        import torch
        return torch.device("cuda", self.local_rank) if self.backend == "nccl" else torch.device("cpu")

    def heads(self, total: int) -> tuple[int, int]:
        return head_slice(total, self.world, self.rank)

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, x: float) -> float:
        """Max over ranks (multi-GPU times are reported as the slowest rank's)."""
        if self.world == 1:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self._device())
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather_heads(self, local, total_heads: int, out=None):
        """All-gather per-rank [h_local, n, d] slices into [total_heads, n, d] (C1)."""
        import torch
        if self.world == 1:
            return local
        import torch.distributed as dist
        sizes = [self.heads_of(r, total_heads) for r in range(self.world)]
        if len(set(sizes)) == 1:
            if out is None:
                out = torch.empty((total_heads,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
            dist.all_gather_into_tensor(out, local.contiguous())
            return out
        # uneven split: all-gather equal-size padded slices, then drop the padding
        mx = max(sizes)
        pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        pad[:local.shape[0]].copy_(local)
        parts = [torch.empty_like(pad) for _ in sizes]
        dist.all_gather(parts, pad)
        trimmed = [p[:sz] for p, sz in zip(parts, sizes)]
        return torch.cat(trimmed, 0) if out is None else torch.cat(trimmed, 0, out=out)

    def full_output(self, total_heads: int, n: int, d: int, force_symmetric: bool = False):
        """FusedOutput: a [total_heads, n, d] bf16 buffer on every rank, mapped into every
        other rank's address space (torch symmetric memory over NVLink / NVSwitch), for
        masked_attention_scatter: each rank's kernel epilogue stores its heads' O rows into
        all ranks' buffers, so no all-gather runs after the kernel."""
        return FusedOutput(self, total_heads, n, d, force_symmetric)

    def heads_of(self, rank: int, total: int) -> int:
        lo, hi = head_slice(total, self.world, rank)
        return hi - lo

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


class FusedOutput:
    """Full-O buffer shared across ranks for the fused reassembly (C1 without a collective).

    `ptrs` lists every rank's buffer as a device pointer valid on this rank (peer memory);
    `head_base` is this rank's first head.  After the forward, `sync()` makes all ranks'
    stores visible (symmetric-memory barrier).  World size 1 degenerates to a local buffer."""

    def __init__(self, hp: HeadParallel, total_heads: int, n: int, d: int, force_symmetric: bool = False):
        import torch
        self.hp = hp
        self.head_base, hi = hp.heads(total_heads)
        self.heads_full = total_heads
        dev = torch.device("cuda", torch.cuda.current_device())
        if hp.world > 1 or force_symmetric:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            self.out = symm_mem.empty(total_heads, n, d, dtype=torch.bfloat16, device=dev)
            self._hdl = symm_mem.rendezvous(self.out, dist.group.WORLD)
            self.ptrs = [int(p) for p in self._hdl.buffer_ptrs]
        else:
            self.out = torch.empty(total_heads, n, d, dtype=torch.bfloat16, device=dev)
            self._hdl = None
            self.ptrs = [self.out.data_ptr()]

    def sync(self):
        """All ranks' epilogue stores have landed in every buffer once this returns."""
        if self._hdl is not None:
            self._hdl.barrier()
