"""GPU `mask` / `stats` / `bench` subcommands with the reference CLI's flags, JSON keys and exit
codes (reference tools/radial_cli.cpp:40-96 flags, :122-133 stats keys, :143-189 mask/stats,
:390-418 bench, :487-514 exit codes 0 ok / 2 usage or input error).  SURVEY.md 8f row 3.

    python -m paper_2506_19852_b200.cli stats --preset hunyuan-509
    python -m paper_2506_19852_b200.cli mask --frames 256 --tokens 64 --block 64 --out m.ramk --pgm m.pgm
    python -m paper_2506_19852_b200.cli bench --frames 64 --tokens 64 --head-dim 64 --block 64

`verify`, `compare` and `fit` are the reference's analysis tooling (out of scope).
"""
from __future__ import annotations

import argparse
import json
import sys

# presets.hpp:34-43 (latent geometries; config table)
PRESETS = {
    "hunyuan-117": (30, 3600, 128), "hunyuan-253": (64, 3600, 128), "hunyuan-509": (128, 3600, 128),
    "wan-69": (18, 3600, 128), "wan-161": (41, 3600, 128), "mochi-163": (28, 1590, 128),
    "mochi-331": (56, 1590, 128), "mochi-667": (112, 1590, 128),
}
KINDS = ("radial", "dense", "spatial", "temporal", "sta", "power", "harmonic")


class UsageError(Exception):
    pass


def _shape_opts(p, preset=True):
    p.add_argument("--frames", type=int, default=0)
    p.add_argument("--tokens", type=int, default=0)
    p.add_argument("--block", type=int, default=128)
    p.add_argument("--pattern", default="radial")
    p.add_argument("--sink", dest="sink", action="store_true", default=None)
    p.add_argument("--no-sink", dest="sink", action="store_false")
    p.add_argument("--temporal-window", type=int, default=None)
    p.add_argument("--spatial-window", type=int, default=None)
    if preset:
        p.add_argument("--preset", default="")


def _shape(P, a):
    if getattr(a, "preset", ""):
        if a.preset not in PRESETS:
            raise UsageError(f"--preset: unknown preset '{a.preset}'")
        f, s, b = PRESETS[a.preset]
        return P.GridShape(f, s), b
    if a.frames == 0 or a.tokens == 0:
        raise UsageError("--frames/--tokens: shape required (or use --preset)")
    return P.GridShape(a.frames, a.tokens), a.block


def _pattern(P, a):
    if a.pattern not in KINDS:
        raise UsageError(f"--pattern: unknown pattern '{a.pattern}'")
    kind = KINDS.index(a.pattern)
    sink = a.sink if a.sink is not None else kind == 0
    spec = P.PatternSpec(kind, sink, a.temporal_window, a.spatial_window)
    if kind in (2, 4) and a.temporal_window is None:
        raise UsageError(f"--temporal-window: required for pattern '{a.pattern}'")
    if kind in (3, 4) and a.spatial_window is None:
        raise UsageError(f"--spatial-window: required for pattern '{a.pattern}'")
    return spec


def _emit(obj, pretty):
    print(json.dumps(obj, indent=2 if pretty else None))


def stats_json(P, layout, head_dim, heads):
    fl = P.attention_flops(layout, head_dim, heads)
    return {"f": layout.shape.frames, "s": layout.shape.tokens_per_frame, "B": layout.block_size,
            "kept_blocks": layout.kept_blocks(), "sparsity": P.sparsity(layout),
            "dense_flops": fl.dense_flops, "sparse_flops": fl.sparse_flops, "reduction": fl.reduction}


def run_mask(P, a):
    shape, B = _shape(P, a)
    lay = P.blockify(shape, _pattern(P, a), B)  # K1 on the GPU
    with open(a.out, "wb") as fh:
        fh.write(P.serialize(lay))
    if a.pgm:
        R = lay.grid_rows
        if R > 8192:
            raise ValueError(f"render_pgm: grid {R} exceeds 8192")
        import numpy as np
        img = np.full((R, R), 255, np.uint8)
        rows = np.repeat(np.arange(R), np.diff(lay.row_ptr).astype(np.int64))
        img[rows, lay.col_idx] = 0
        with open(a.pgm, "wb") as fh:
            fh.write(f"P5\n{R} {R}\n255\n".encode() + img.tobytes())
    _emit({"kept_blocks": lay.kept_blocks(), "sparsity": P.sparsity(lay)}, a.pretty)
    return 0


def run_stats(P, a):
    if a.in_:
        with open(a.in_, "rb") as fh:
            lay = P.deserialize(fh.read())
    else:
        shape, B = _shape(P, a)
        lay = P.blockify(shape, _pattern(P, a), B)
    _emit(stats_json(P, lay, a.head_dim, a.heads), a.pretty)
    return 0


def run_bench(P, a):
    """dense vs token-exact masked attention (the reference times masked_attention(inst,
    PatternSpec), radial_cli.cpp:403), both on the GPU, one head, seeded N(0,1) inputs."""
    import torch
    shape, B = _shape(P, a)
    pattern = _pattern(P, a)
    n, d = shape.total_tokens(), a.head_dim
    g = torch.Generator(device="cuda").manual_seed(a.seed)
    q, k, v = (torch.randn(1, n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    lay = P.device_layout(shape, pattern, B)

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(reps):
            fn()
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / reps / 1e3

    dense_s = timed(lambda: P.dense_attention(q, k, v, block_size=B))
    masked_s = timed(lambda: P.masked_attention_pattern(q, k, v, shape, pattern, block_size=B))
    red = P.attention_flops(lay.host(), d, 1).reduction
    _emit({"dense_seconds": dense_s, "masked_seconds": masked_s, "speedup": dense_s / masked_s,
           "flops_reduction": red}, a.pretty)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="radial", description="Radial sparse attention masks on B200")
    ap.add_argument("--pretty", action="store_true")
    sub = ap.add_subparsers(dest="cmd", required=True)
    m = sub.add_parser("mask")
    _shape_opts(m)
    m.add_argument("--out", required=True)
    m.add_argument("--pgm", default="")
    s = sub.add_parser("stats")
    _shape_opts(s)
    s.add_argument("--in", dest="in_", default="")
    s.add_argument("--head-dim", type=int, default=64)
    s.add_argument("--heads", type=int, default=1)
    b = sub.add_parser("bench")
    _shape_opts(b, preset=False)
    b.add_argument("--head-dim", type=int, default=64)
    b.add_argument("--seed", type=int, default=0)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        import paper_2506_19852_b200 as P
        return {"mask": run_mask, "stats": run_stats, "bench": run_bench}[a.cmd](P, a)
    except (UsageError, ValueError, RuntimeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
