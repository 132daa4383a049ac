#!/usr/bin/env python
"""Radial attention forward benchmark (BASELINE.json metric: effective TFLOP/s and
ms/call vs dense) on 1..8 B200s, head-parallel.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself under
torch.distributed.run with N ranks (one per GPU) and fails loudly when the world size
does not match --gpus.

Workload (N=1 line): BASELINE configs[1], HunyuanVideo 720p default length --
33 latent frames x 3600 tokens (n = 118,800), 24 heads, head_dim 128, block 128,
radial mask with attention sink, bf16 Q/K/V [heads][n][128] ~ N(0,1) (synthetic).
A step is one sparse forward over the rank's head slice (heads split evenly across
ranks: strong scaling of the fixed 24-head call, no collective on the data path;
--weak gives every rank all heads instead).  The line also carries the backward (K3)
at the same shape, a Mochi-28 fwd+bwd record (BASELINE configs[3]) and, at N > 1, the
fused / NCCL output reassembly timings.
Effective FLOPs = 4 * kept_blocks * B^2 * d * heads (reference block.hpp:137-148).
Inputs (2.2 GB) are far larger than L2 (126 MB), so no L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (frames, tokens_per_frame, heads, head_dim, block)
    "hunyuan33": (33, 3600, 24, 128, 128),
    "wan21": (21, 3600, 40, 128, 128),
    "mochi28": (28, 1590, 24, 128, 128),
    "hunyuan132": (132, 3600, 24, 128, 128),
    "tiny": (8, 256, 2, 64, 64),
}
METRIC = "radial_attn_fwd_effective_tflops"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return pk["bf16_tflops"], pk.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t.is_alive():
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


_HP = None  # paper_2506_19852_b200.heads.HeadParallel of this process


def dist_setup(backend="nccl"):
    """One process per GPU; NCCL process group when launched by torchrun (N > 1)."""
    global _HP
    import torch
    from paper_2506_19852_b200.heads import HeadParallel
    _HP = HeadParallel.from_env(backend)
    if _HP.world == 1 and backend == "nccl" and torch.cuda.is_available():
        torch.cuda.set_device(0)
    return _HP.world, _HP.rank, _HP.local_rank


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: re-launch this script under
    torch.distributed.run with N ranks on this node (the driver's command shape)."""
    import subprocess
    if not args.dry_run and not args.shared_gpu:
        try:
            import torch
            have = torch.cuda.device_count()
        except Exception:
            have = 0
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def gather_to_rank0(obj):
    """Every rank's small result dict, on rank 0 (None elsewhere)."""
    if _HP is None or _HP.world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * _HP.world if _HP.rank == 0 else None
    dist.gather_object(obj, out, dst=0)
    return out


def barrier(world):
    if _HP is not None:
        _HP.barrier()


def max_over_ranks(x: float, world: int) -> float:
    return _HP.max(x) if _HP is not None else x


def head_slice(H, world, rank):
    from paper_2506_19852_b200.heads import head_slice as hs
    return hs(H, world, rank)


def timed_loop(fn, steps, stream):
    """Per-step CUDA-event times (ms) on the launching stream."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a, b in evs:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own masked_attention (oracle/_ref) on a sample
# ---------------------------------------------------------------------------
def cpu_reference_sample(f, s, d, B, per_thread, steps=1, warmup=0):
    import oracle as O
    cores = os.cpu_count() or 1
    os.environ["RADIAL_THREADS"] = str(cores)
    rp, ci = O.blockify(f, s, B)
    srp, sci, kept, sampled = O.sample_layout(rp, ci, f * s, B, cores, per_thread)
    kind = "reference" if O.ref_available() else "port"
    if kind != "reference":
        raise RuntimeError("oracle/_ref/libradial_ref.so missing: build it here with `make oracle`")
    inst = O.RefInstance(f, s, d, 42)
    flops = 4.0 * kept * B * B * d
    for _ in range(warmup):
        inst.masked_attention(B, srp, sci)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        inst.masked_attention(B, srp, sci)
        times.append(time.perf_counter() - t0)
    sec = statistics.median(times)
    sample = (f"reference radial::masked_attention(inst, layout) (attention.hpp:229), fp64, one head "
              f"of f{f} s{s} d{d} B{B}: {len(sampled)} query blocks ({per_thread} per thread chunk) "
              f"keep their full KV lists, the other {len(rp) - 1 - len(sampled)} rows keep one block; "
              f"{kept} kept blocks executed = {flops:.4g} FLOP per call")
    return {"value": flops / sec / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind,
            "sample": sample, "seconds_per_call": sec,
            "cpu": _cpu_model()}, sec, flops


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, world, rank):
    f, s, H, d, B = CONFIGS[args.config]
    if rank != 0:
        return
    try:
        base, sec, flops = cpu_reference_sample(f, s, d, B, per_thread=1, steps=args.steps,
                                                warmup=args.warmup)
    except Exception as e:  # the oracle always exists in this repo; report instead of crash
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    line = {"metric": METRIC, "value": base["value"], "unit": "TFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (random_instance seed 42)",
            "config": {"workload": f"{args.config}: f{f} x s{s}, {H} heads, head_dim {d}, block {B}, "
                                   "radial+sink; reference path is one head per call (sampled rows)"},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------
def run_ours(args, world, rank, local):
    import torch
    import paper_2506_19852_b200 as P

    f, s, H, d, B = CONFIGS[args.config]
    n = f * s
    h0, h1 = (0, H) if args.weak else head_slice(H, world, rank)
    Hl = h1 - h0
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()

    # mask build (K1), timed separately; the layout is cached for the steps
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(True), B, cache=False)
    t1.record(stream)
    torch.cuda.synchronize()
    mask_ms_first = t0.elapsed_time(t1)
    kept = lay.kept_blocks()
    flops_total = 4.0 * kept * B * B * d * (H * world if args.weak else H)
    flops_local = 4.0 * kept * B * B * d * Hl
    dense_flops_local = 4.0 * n * n * d * Hl

    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    q = torch.randn(Hl, n, d, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
    k = torch.randn(Hl, n, d, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
    v = torch.randn(Hl, n, d, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(Hl, n, device=dev, dtype=torch.float32)

    o_full = None
    fused = None
    if args.gather and world > 1 and not args.gather_nccl:
        # C1 fused into the kernel: O rows stored straight into every rank's full buffer
        fused = _HP.full_output(H, n, d)
    elif args.gather and world > 1:
        o_full = torch.empty(H, n, d, device=dev, dtype=torch.bfloat16)

    def step():
        if fused is not None:
            P.masked_attention_scatter(q, k, v, lay, fused.ptrs, fused.head_base, H, lse=lse, stream=stream)
            fused.sync()
            return
        P.masked_attention(q, k, v, lay, out=o, lse=lse, return_lse=True, stream=stream)
        if o_full is not None:  # C1: reassemble O [H, n, d] on every rank (NCCL all-gather)
            _HP.gather_heads(o, H, out=o_full)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    launches0 = P.kernel_launches()
    with ClockSampler(local) as clk:
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        per = timed_loop(step, args.steps, stream)
        stop.record(stream)
        torch.cuda.synchronize()
    launches = P.kernel_launches() - launches0
    barrier(world)
    total_ms = max_over_ranks(start.elapsed_time(stop), world)
    ms_per_step = total_ms / args.steps
    kernel_ms = max_over_ranks(statistics.mean(per), world)
    value = flops_total / (ms_per_step * 1e-3) / 1e12

    # dense comparator (K4) on the same inputs, same timing discipline
    dense = None
    if not args.no_dense:
        def dstep():
            P.dense_attention(q, k, v, block_size=B, out=o, lse=lse, return_lse=True, stream=stream)
        for _ in range(max(1, args.warmup)):
            dstep()
        torch.cuda.synchronize()
        dsteps = max(2, min(args.steps, 10))
        dper = timed_loop(dstep, dsteps, stream)
        dense_ms = max_over_ranks(statistics.mean(dper), world)
        dense = {"ms_per_step": dense_ms,
                 "dense_tflops": 4.0 * n * n * d * H / (dense_ms * 1e-3) / 1e12,
                 "speedup_sparse_vs_dense": dense_ms / kernel_ms, "steps": dsteps}

    # backward (K3) over the same layout: algorithmic FLOPs = 2.5 x forward (5 GEMMs)
    bwd = None
    if args.no_bwd:
        pass
    elif B != 128:
        # K3 covers the backward configs of BASELINE (block 128); the tiny config (block 64)
        # is forward-only in the reference's own benchmark plan
        bwd = {"unsupported": "backward kernels are built for block_size 128 (BASELINE configs[3], [4])"}
    else:
        bwd = time_backward(P, lay, q, k, v, o, lse, g, flops_total, world, args, stream)

    # BASELINE configs[3]: Mochi 1 480p fwd + bwd (the LoRA tuning path) on the same heads split
    extra = {}
    if not args.no_extra and args.config == "hunyuan33":
        extra["mochi28"] = time_config(P, "mochi28", world, rank, args, stream)

    # N > 1: reassembly of O on every rank -- fused into the epilogue (peer stores) vs NCCL
    gather = None
    if world > 1 and not args.no_gather and not args.weak:
        gather = time_gather(P, lay, q, k, v, lse, H, n, d, world, args, stream)

    # end-to-end through the reference-facing C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(P, lay, q, k, v, Hl, n, d, flops_total, world, args)

    # mask builder time (warm: rebuild without cache)
    mts = []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(True), B, cache=False)
        b.record(stream)
        torch.cuda.synchronize()
        mts.append(a.elapsed_time(b))

    launches_all = gather_to_rank0(launches)
    heads_all = gather_to_rank0(Hl)
    barrier(world)
    _HP.close()  # the other ranks are done: rank 0 alone times the CPU baseline below
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu, _, _ = cpu_reference_sample(f, s, d, B, per_thread=2)
        except Exception as e:
            cpu = {"unavailable": str(e)}
    peak, peak_sus, peak_src = load_peaks()
    achieved = flops_local / (kernel_ms * 1e-3) / 1e12
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tj = json.load(fh)
        if world == 1 or args.weak:  # the capture is of the whole 24-head launch
            traffic = tj.get(args.config)
            traffic_src = tj.get("_source") if traffic is not None else None
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: Q,K,V ~ N(0,1) bf16, torch.Generator seeds 1000+rank",
        "config": {"workload": f"{args.config}: radial attention fwd, f{f} x s{s} (n={n}), {H} heads, "
                               f"head_dim {d}, block {B}, sink on; " +
                               (f"all {H} heads on every rank" if args.weak else f"heads split {heads_all} over ranks"),
                   "frames": f, "tokens_per_frame": s, "heads": H, "head_dim": d, "block": B,
                   "kept_blocks": kept, "block_sparsity": 1 - kept / float(lay.grid_rows ** 2),
                   "parallelism": f"head-parallel x{world}" + ((" + NCCL all-gather(O)" if args.gather_nccl else
                                                                 " + O stored to every rank from the epilogue")
                                                                if args.gather and world > 1 else ""),
                   "heads_per_rank": heads_all,
                   "l2": "inputs (3 x bf16 [H][n][d]) far exceed the 126 MB L2; no flush"},
        "kernel_ms": kernel_ms,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "frac_of_sustained": achieved / peak_sus if peak_sus else None,
                     "peak_source": peak_src, "traffic": traffic,
                     "traffic_source": traffic_src or "no ncu capture for this config",
                     "kernel": "radial_attn_fwd_kernel<128,128>",
                     "flops_per_launch": flops_local},
        "dense": dense,
        "backward": bwd,
        "configs": extra or None,
        "gather": gather,
        "mask_build_ms": {"first": mask_ms_first, "warm_median": statistics.median(mts)},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": int(sum(launches_all)),
        "gpu_launches_per_rank": launches_all,
        "gpu_launches_source": "radial_cuda_kernel_launches() delta over the timed region (this library's kernels)",
        "clocks": clk.summary(),
    }
    if args.shared_gpu and world > 1:
        line["shared_gpu_plumbing_test"] = ("all ranks ran on cuda:0 with gloo collectives: the N > 1 code path "
                                            "end to end, not a multi-GPU measurement")
    print(json.dumps(line))


def time_backward(P, lay, q, k, v, o, lse, g, flops_total, world, args, stream):
    """K3 over the layout: dQ / dK / dV of the forward just timed.  Algorithmic FLOPs = 2.5 x
    forward (S, dP, dV, dK, dQ); executed = what the kernels issue (S and dP recomputed by the
    dQ and the dK/dV kernel: 3.5 x forward)."""
    import torch
    Hl, n, d = q.shape
    dout = torch.randn(Hl, n, d, device=q.device, generator=g, dtype=torch.float32).to(torch.bfloat16)
    P.masked_attention(q, k, v, lay, out=o, lse=lse, return_lse=True, stream=stream)
    ws = torch.empty(P._lib.radial_cuda_attn_bwd_workspace_size(Hl, n, d), dtype=torch.uint8, device=q.device)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)

    def bstep():
        P._check(P._lib.radial_cuda_attn_bwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                                             dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), Hl, n, d,
                                             0.0, lay.handle, ws.data_ptr(), stream.cuda_stream))
    for _ in range(max(1, args.warmup)):
        bstep()
    torch.cuda.synchronize()
    bsteps = max(2, min(args.steps, 10))
    l0 = P.kernel_launches()
    bper = timed_loop(bstep, bsteps, stream)
    nl = P.kernel_launches() - l0
    bwd_ms = max_over_ranks(statistics.mean(bper), world)
    peak, peak_sus, _ = load_peaks()
    eff = 2.5 * flops_total / (bwd_ms * 1e-3) / 1e12
    exe = P.BWD_EXECUTED_FACTOR * flops_total / (bwd_ms * 1e-3) / 1e12
    return {"ms_per_step": bwd_ms, "steps": bsteps,
            "effective_tflops": eff, "executed_tflops": exe,
            "executed_factor": P.BWD_EXECUTED_FACTOR,
            "roofline_frac_effective": eff / peak, "roofline_frac_executed": exe / peak,
            "flops_convention": "effective: 2.5 x forward kept-block FLOPs (S, dP, dV, dK, dQ); executed: "
                                "the GEMMs the kernels issue",
            "launches_per_step": nl / bsteps}


def time_config(P, name, world, rank, args, stream):
    """Forward (+ dense comparator) and backward of another BASELINE config, same heads split."""
    import torch
    f, s, H, d, B = CONFIGS[name]
    n = f * s
    h0, h1 = (0, H) if args.weak else head_slice(H, world, rank)
    Hl = h1 - h0
    Ht = H * world if args.weak else H
    lay = P.device_layout(P.GridShape(f, s), P.PatternSpec.radial(True), B)
    kept = lay.kept_blocks()
    flops = 4.0 * kept * B * B * d * Ht
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev).manual_seed(2000 + rank)
    q, k, v = (torch.randn(Hl, n, d, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
               for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty(Hl, n, device=dev, dtype=torch.float32)

    def fstep():
        P.masked_attention(q, k, v, lay, out=o, lse=lse, return_lse=True, stream=stream)

    def dstep():
        P.dense_attention(q, k, v, block_size=B, out=o, lse=lse, return_lse=True, stream=stream)
    for fn in (fstep, dstep):
        for _ in range(max(1, args.warmup)):
            fn()
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 10))
    fms = max_over_ranks(statistics.mean(timed_loop(fstep, steps, stream)), world)
    dms = max_over_ranks(statistics.mean(timed_loop(dstep, steps, stream)), world)
    peak, _, _ = load_peaks()
    rec = {"workload": f"{name}: f{f} x s{s} (n={n}), {H} heads, head_dim {d}, block {B}, radial+sink",
           "kept_blocks": kept, "fwd_ms": fms, "fwd_tflops": flops / (fms * 1e-3) / 1e12,
           "fwd_roofline_frac": flops / (fms * 1e-3) / 1e12 / peak,
           "dense_ms": dms, "speedup_sparse_vs_dense": dms / fms, "steps": steps}
    if not args.no_bwd:
        b = time_backward(P, lay, q, k, v, o, lse, g, flops, world, args, stream)
        rec["backward"] = b
        rec["fwd_bwd_ms"] = fms + b["ms_per_step"]
        rec["fwd_bwd_effective_tflops"] = 3.5 * flops / ((fms + b["ms_per_step"]) * 1e-3) / 1e12
    return rec


def time_gather(P, lay, q, k, v, lse, H, n, d, world, args, stream):
    """C1 at N > 1: every rank ends the step with the full O [H, n, d].  `fused`: the forward's
    epilogue stores each row into every rank's buffer (peer memory over NVLink) and a
    symmetric-memory barrier closes the step; `nccl`: the plain forward, then an NCCL
    all-gather of O."""
    import torch
    out = {}
    steps = max(2, min(args.steps, 10))
    try:
        fused = _HP.full_output(H, n, d)

        def fstep():
            P.masked_attention_scatter(q, k, v, lay, fused.ptrs, fused.head_base, H, lse=lse, stream=stream)
            fused.sync()
        for _ in range(max(1, args.warmup)):
            fstep()
        torch.cuda.synchronize()
        barrier(world)
        out["fused_ms"] = max_over_ranks(statistics.mean(timed_loop(fstep, steps, stream)), world)
        del fused
    except Exception as e:  # symmetric memory unavailable on this box
        out["fused_error"] = f"{type(e).__name__}: {e}"
    o = torch.empty_like(q)
    o_full = torch.empty(H, n, d, device=q.device, dtype=torch.bfloat16)

    def nstep():
        P.masked_attention(q, k, v, lay, out=o, lse=lse, return_lse=True, stream=stream)
        _HP.gather_heads(o, H, out=o_full)
    for _ in range(max(1, args.warmup)):
        nstep()
    torch.cuda.synchronize()
    barrier(world)
    out["nccl_ms"] = max_over_ranks(statistics.mean(timed_loop(nstep, steps, stream)), world)
    out["steps"] = steps
    out["o_bytes_full"] = H * n * d * 2
    return out


def run_dry(args, world, rank):
    """--dry-run: the launcher and the rank plumbing without a GPU (gloo): each rank reports its
    heads; rank 0 prints the line shape the GPU run would print."""
    f, s, H, d, B = CONFIGS[args.config]
    h0, h1 = (0, H) if args.weak else head_slice(H, world, rank)
    t = max_over_ranks(float(rank + 1), world)
    heads_all = gather_to_rank0([h0, h1])
    _HP.close()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "heads_per_rank": heads_all,
                          "max_over_ranks": t, "scaling": "weak" if args.weak else "strong"}))


def run_e2e(P, lay, q, k, v, Hl, n, d, flops_total, world, args):
    """Same metric through radial_cuda_attn_fwd_host: pinned host Q/K/V in, host O out,
    copies inside the timed region (device-timed with events on the call's stream)."""
    import ctypes
    import torch
    hq = q.cpu().pin_memory()
    hk = k.cpu().pin_memory()
    hv = v.cpu().pin_memory()
    ho = torch.empty_like(hq).pin_memory()
    stream = torch.cuda.current_stream()
    lib = P._lib

    def call():
        P._check(lib.radial_cuda_attn_fwd_host(hq.data_ptr(), hk.data_ptr(), hv.data_ptr(),
                                               ho.data_ptr(), None, Hl, n, d, 0.0, lay.handle,
                                               ctypes.c_void_p(stream.cuda_stream)))

    for _ in range(max(1, min(args.warmup, 3))):
        call()
    steps = max(2, min(args.steps, 10))
    barrier(world)
    per = timed_loop(call, steps, stream)
    ms = max_over_ranks(statistics.mean(per), world)
    tb = Hl * n * d * 2
    return {"value": flops_total / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": 3 * tb, "d2h_bytes_per_step": tb, "steps": steps,
            "path": "C-ABI radial_cuda_attn_fwd_host (pinned host bf16 in/out)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="hunyuan33")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--bwd", action="store_true", help=argparse.SUPPRESS)  # the backward is timed by default
    ap.add_argument("--no-bwd", action="store_true", help="skip the backward (K3) record")
    ap.add_argument("--no-extra", action="store_true", help="skip the Mochi-28 fwd+bwd record")
    ap.add_argument("--no-gather", action="store_true", help="skip the N > 1 output reassembly timings")
    ap.add_argument("--weak", action="store_true", help="every rank runs all heads (weak scaling)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / rank plumbing only (gloo, no GPU): prints the ranks' head split")
    ap.add_argument("--gather", action="store_true",
                    help="reassemble O [H, n, d] on every rank in each step when N > 1 (C1): the kernel "
                         "epilogue stores each row into every rank's buffer over peer memory")
    ap.add_argument("--gather-nccl", action="store_true",
                    help="with --gather: NCCL all-gather after the kernel instead (comparison)")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="plumbing test for boxes with one GPU: every rank runs on cuda:0 with gloo "
                         "collectives (no reassembly timings); the line is marked and its timings are not "
                         "a multi-GPU measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        # the reference's CPU path on rank 0 only (others exit 0 without work); no spawn needed
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        run_reference(args, world, rank)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world, rank, local = dist_setup("gloo" if (args.dry_run or args.shared_gpu) else "nccl")
    if args.shared_gpu and not args.dry_run:
        import torch
        torch.cuda.set_device(0)
        local = 0
        args.no_gather = True
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launch has WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.dry_run:
        run_dry(args, world, rank)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
