"""B200-native radial attention (arXiv 2506.19852): Python host mirror of the
reference's C++ API (``/root/reference/proj/include/radial``) over the C-ABI
library ``lib/libradial_cuda.so`` (include/radial_cuda.h).

Names, argument meaning and error behaviour follow the reference:

=============================  ==================================================
reference (C++)                here
=============================  ==================================================
``GridShape`` grid.hpp:16      :class:`GridShape`
``PatternSpec`` grid.hpp:83    :class:`PatternSpec`
``BlockLayout`` block.hpp:23   :class:`BlockLayout` (host CSR, numpy)
``blockify`` block.hpp:59      :func:`blockify` (built by the K1 CUDA kernel)
``masked_attention`` :229      :func:`masked_attention` (K2, torch CUDA tensors)
``dense_attention`` :141       :func:`dense_attention` (K4 comparator)
``attention_flops`` :137       :func:`attention_flops`
``sparsity`` :123              :func:`sparsity`
``serialize``/``deserialize``  :func:`serialize` / :func:`deserialize`
=============================  ==================================================

The reference's ``std::invalid_argument`` maps to :class:`ValueError`,
``std::length_error`` to :class:`LengthError`, ``std::runtime_error`` (empty
softmax row) to :class:`RuntimeError`.  There is no CPU fallback: importing
this package without the built CUDA library raises ``ImportError``.

Device tensors are bf16 ``[heads, n, head_dim]`` (head-major, so a head slice
is contiguous); ``lse`` is fp32 ``[heads, n]``.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "GridShape", "PatternSpec", "PatternKind", "BlockLayout", "DeviceLayout", "FlopsReport",
    "LengthError", "ParseError", "blockify", "device_layout", "masked_attention",
    "dense_attention", "masked_attention_backward", "masked_attention_pattern", "masked_attention_host", "attention_flops",
    "sparsity", "serialize", "deserialize", "library_path",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# RADIAL_CUDA_LIB overrides the in-tree library (used for kernel-variant sweeps)
_LIB_PATH = os.environ.get("RADIAL_CUDA_LIB") or os.path.join(_HERE, "lib", "libradial_cuda.so")


def library_path() -> str:
    return _LIB_PATH


def debug_library_path() -> str:
    """Diagnostics library (tcgen05 / pipe microbenchmarks for scripts/; not the product path)."""
    return os.path.join(os.path.dirname(_LIB_PATH), "libradial_debug.so")


if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"paper_2506_19852_b200: CUDA library {_LIB_PATH} is missing; build it with "
        "`make lib` or `python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")

_lib = C.CDLL(_LIB_PATH)

_u8, _u32, _u64, _i32, _i64, _f32, _f64, _vp = (C.c_uint8, C.c_uint32, C.c_uint64, C.c_int,
                                                C.c_int64, C.c_float, C.c_double, C.c_void_p)


class _LayoutInfo(C.Structure):
    _fields_ = [("frames", _u32), ("tokens_per_frame", _u32), ("block_size", _u32),
                ("grid_rows", _u32), ("kind", _u8), ("sink", _u8), ("kept_blocks", _u64),
                ("first_empty_row", _i64), ("max_row_len", _u32), ("min_row_len", _u32)]


def _sig(name, restype, *argtypes):
    fn = getattr(_lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn


_sig("radial_cuda_abi_version", _i32)
_sig("radial_cuda_last_error", C.c_char_p)
_sig("radial_cuda_mask_build", _i32, _u32, _u32, _u32, _i32, _i32, _u32, _u32, _vp, C.POINTER(_vp))
_sig("radial_cuda_layout_from_csr", _i32, _u32, _u32, _u32, _i32, _i32, _u32, _vp, _vp, _vp,
     C.POINTER(_vp))
_sig("radial_cuda_layout_info", _i32, _vp, C.POINTER(_LayoutInfo))
_sig("radial_cuda_layout_copy_csr", _i32, _vp, _vp, _vp)
_sig("radial_cuda_layout_copy_csc", _i32, _vp, _vp, _vp)
_sig("radial_cuda_layout_device_csr", _i32, _vp, C.POINTER(_vp), C.POINTER(_vp))
_sig("radial_cuda_layout_free", None, _vp)
_sig("radial_cuda_layout_acquire", _i32, _u32, _u32, _u32, _i32, _i32, _u32, _u32, _vp, C.POINTER(_vp))
_sig("radial_cuda_layout_cache_clear", None)
_sig("radial_cuda_kernel_launches", _u64)
_sig("radial_cuda_attn_fwd", _i32, _vp, _vp, _vp, _vp, _vp, _u32, _u64, _u32, _f32, _vp, _vp)
_sig("radial_cuda_attn_fwd_token", _i32, _vp, _vp, _vp, _vp, _vp, _u32, _u64, _u32, _f32, _vp, _vp)
_sig("radial_cuda_attn_fwd_host_multi", _i32, _vp, _vp, _vp, _vp, _vp, _u32, _u64, _u32, _f32, _u32, _u32, _u32,
     _i32, _i32, _u32, _u32, C.POINTER(_i32), _i32)
_sig("radial_cuda_attn_fwd_scatter", _i32, _vp, _vp, _vp, C.POINTER(_vp), _u32, _u32, _u32, _vp, _u32, _u64,
     _u32, _f32, _vp, _vp)
_sig("radial_cuda_attn_fwd_dense", _i32, _vp, _vp, _vp, _vp, _vp, _u32, _u64, _u32, _u32, _f32, _vp)
_sig("radial_cuda_attn_fwd_host", _i32, _vp, _vp, _vp, _vp, _vp, _u32, _u64, _u32, _f32, _vp, _vp)
_sig("radial_cuda_attn_bwd_workspace_size", C.c_size_t, _u32, _u64, _u32)
_sig("radial_cuda_attn_bwd", _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u32, _u64, _u32,
     _f32, _vp, _vp, _vp)
_sig("radial_cuda_attention_flops", _i32, _vp, _u32, _u32, C.POINTER(_f64), C.POINTER(_f64),
     C.POINTER(_f64))
_sig("radial_cuda_sparsity", _f64, _vp)

RADIAL_OK, ERR_INVALID, ERR_EMPTY_ROW, ERR_CUDA, ERR_OOM, ERR_LENGTH = 0, 1, 2, 3, 4, 5
WINDOW_NONE = 0xFFFFFFFF  # RADIAL_WINDOW_NONE: PatternSpec window absent
# GEMMs the backward kernels issue per kept block, in units of the forward's two (QK^T, PV):
# the dQ kernel computes S, dP, dQ and the dK/dV kernel S, dP, dV, dK -> 7 / 2
BWD_EXECUTED_FACTOR = 3.5


def kernel_launches() -> int:
    """CUDA kernels this library has launched in this process (radial_cuda_kernel_launches)."""
    return int(_lib.radial_cuda_kernel_launches())


def _window(w) -> int:
    return WINDOW_NONE if w is None else int(w)


class LengthError(ValueError):
    """std::length_error in the reference (block grid > 2^32 rows, block.hpp:50-52)."""


class ParseError(RuntimeError):
    """Structured .ramk parse failure; ``field`` names the offending part (block.hpp:155-164)."""

    def __init__(self, field_name: str, message: str):
        super().__init__(f"parse error in '{field_name}': {message}")
        self.field = field_name


def _check(rc: int):
    if rc == RADIAL_OK:
        return
    msg = _lib.radial_cuda_last_error().decode()
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_LENGTH:
        raise LengthError(msg)
    if rc == ERR_EMPTY_ROW:
        raise RuntimeError(msg)
    if rc == ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------------------
# grid.hpp
# ---------------------------------------------------------------------------
class PatternKind:
    radial, dense, spatial, temporal, sta, power, harmonic = range(7)
    names = ("radial", "dense", "spatial", "temporal", "sta", "power", "harmonic")


@dataclass(frozen=True)
class GridShape:
    """f frames of s tokens, token (i, k) at i*s + k (grid.hpp:16-42)."""
    frames: int = 1
    tokens_per_frame: int = 1

    def __post_init__(self):
        if self.frames < 1 or self.tokens_per_frame < 1:
            raise ValueError("GridShape: frames and tokens_per_frame must be >= 1")
        if self.frames * self.tokens_per_frame > (1 << 32):
            raise ValueError("GridShape: total tokens exceeds 2^32")

    def total_tokens(self) -> int:
        return self.frames * self.tokens_per_frame

    def frame_of(self, token: int) -> int:
        return token // self.tokens_per_frame

    def pos_of(self, token: int) -> int:
        return token % self.tokens_per_frame


@dataclass(frozen=True)
class PatternSpec:
    """Mask family + parameters (grid.hpp:83-139).  sink defaults on for radial."""
    kind: int = PatternKind.radial
    sink: bool = True
    temporal_window: Optional[int] = None
    spatial_window: Optional[int] = None

    @staticmethod
    def radial(sink: bool = True) -> "PatternSpec":
        return PatternSpec(PatternKind.radial, sink)

    @staticmethod
    def dense() -> "PatternSpec":
        return PatternSpec(PatternKind.dense, False)

    @staticmethod
    def spatial(temporal_window: int, sink: bool = False) -> "PatternSpec":
        return PatternSpec(PatternKind.spatial, sink, temporal_window, None)

    @staticmethod
    def temporal(spatial_window: int, sink: bool = False) -> "PatternSpec":
        return PatternSpec(PatternKind.temporal, sink, None, spatial_window)

    @staticmethod
    def sta(temporal_window: int, spatial_window: int, sink: bool = False) -> "PatternSpec":
        return PatternSpec(PatternKind.sta, sink, temporal_window, spatial_window)

    @staticmethod
    def power(sink: bool = False) -> "PatternSpec":
        return PatternSpec(PatternKind.power, sink)

    @staticmethod
    def harmonic(sink: bool = False) -> "PatternSpec":
        return PatternSpec(PatternKind.harmonic, sink)

    def validate(self):
        name = PatternKind.names[self.kind]
        if self.kind in (PatternKind.spatial, PatternKind.sta) and self.temporal_window is None:
            raise ValueError(f"{name} pattern requires temporal_window")
        if self.kind in (PatternKind.temporal, PatternKind.sta) and self.spatial_window is None:
            raise ValueError(f"{name} pattern requires spatial_window")


# ---------------------------------------------------------------------------
# block.hpp
# ---------------------------------------------------------------------------
@dataclass
class BlockLayout:
    """Host CSR over the ceil(n/B) x ceil(n/B) block grid (block.hpp:23-45)."""
    shape: GridShape
    block_size: int
    grid_rows: int
    row_ptr: np.ndarray  # uint64 [R+1]
    col_idx: np.ndarray  # uint32 [nnz], strictly increasing per row
    kind: int = PatternKind.radial
    sink: bool = True

    def kept_blocks(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0

    def total_blocks(self) -> int:
        return self.grid_rows * self.grid_rows

    def block_at(self, row: int, col: int) -> bool:
        seg = self.col_idx[int(self.row_ptr[row]):int(self.row_ptr[row + 1])]
        i = int(np.searchsorted(seg, col))
        return i < len(seg) and int(seg[i]) == col

    def __eq__(self, other):
        return (isinstance(other, BlockLayout) and self.shape == other.shape
                and self.block_size == other.block_size and self.grid_rows == other.grid_rows
                and self.kind == other.kind and bool(self.sink) == bool(other.sink)
                and np.array_equal(self.row_ptr, other.row_ptr)
                and np.array_equal(self.col_idx, other.col_idx))


def grid_rows_for(shape: GridShape, block_size: int) -> int:
    rows = (shape.total_tokens() + block_size - 1) // block_size
    if rows > 0xFFFFFFFF:
        raise LengthError("block grid exceeds 2^32 rows")
    return rows


class DeviceLayout:
    """Owning handle of a device-resident layout (CSR + CSC + kernel work lists)."""

    def __init__(self, handle: int, shape: GridShape, block_size: int, kind: int, sink: bool):
        self._h = C.c_void_p(handle)
        self.shape, self.block_size, self.kind, self.sink = shape, block_size, kind, bool(sink)
        info = _LayoutInfo()
        _check(_lib.radial_cuda_layout_info(self._h, C.byref(info)))
        self.grid_rows = info.grid_rows
        self.kept = int(info.kept_blocks)
        self.first_empty_row = int(info.first_empty_row)
        self.max_row_len, self.min_row_len = int(info.max_row_len), int(info.min_row_len)

    @property
    def handle(self):
        return self._h

    def kept_blocks(self) -> int:
        return self.kept

    def host(self) -> BlockLayout:
        R = self.grid_rows
        rp = np.zeros(R + 1, np.uint64)
        ci = np.zeros(max(self.kept, 1), np.uint32)
        _check(_lib.radial_cuda_layout_copy_csr(self._h, rp.ctypes.data, ci.ctypes.data))
        return BlockLayout(self.shape, self.block_size, R, rp, ci[:self.kept], self.kind, self.sink)

    def csc(self):
        R = self.grid_rows
        cp = np.zeros(R + 1, np.uint64)
        ri = np.zeros(max(self.kept, 1), np.uint32)
        _check(_lib.radial_cuda_layout_copy_csc(self._h, cp.ctypes.data, ri.ctypes.data))
        return cp, ri[:self.kept]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:  # _lib is None at interpreter teardown
            _lib.radial_cuda_layout_free(h)
            self._h = C.c_void_p(0)


_cache_lock = threading.Lock()
_layout_cache: dict = {}


def _stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def device_layout(shape: GridShape, pattern: PatternSpec, block_size: int, *, cache: bool = True,
                  stream=None) -> DeviceLayout:
    """Builds (or returns the cached) device layout on the current CUDA device (K1)."""
    import torch
    if block_size < 1:
        raise ValueError("blockify: block_size must be >= 1")
    pattern.validate()
    grid_rows_for(shape, block_size)
    dev = torch.cuda.current_device()
    key = (dev, shape, pattern, block_size)
    if cache:
        with _cache_lock:
            hit = _layout_cache.get(key)
        if hit is not None:
            return hit
    h = C.c_void_p()
    _check(_lib.radial_cuda_mask_build(shape.frames, shape.tokens_per_frame, block_size,
                                       pattern.kind, int(pattern.sink), _window(pattern.temporal_window),
                                       _window(pattern.spatial_window), _stream_ptr(stream), C.byref(h)))
    lay = DeviceLayout(h.value, shape, block_size, pattern.kind, pattern.sink)
    if cache:
        with _cache_lock:
            _layout_cache[key] = lay
    return lay


def layout_from_host(layout: BlockLayout, stream=None) -> DeviceLayout:
    """Uploads a host CSR (e.g. from :func:`deserialize`) as a device layout."""
    h = C.c_void_p()
    rp = np.ascontiguousarray(layout.row_ptr, np.uint64)
    ci = np.ascontiguousarray(layout.col_idx if len(layout.col_idx) else np.zeros(1, np.uint32),
                              np.uint32)
    _check(_lib.radial_cuda_layout_from_csr(layout.shape.frames, layout.shape.tokens_per_frame,
                                            layout.block_size, layout.kind, int(layout.sink),
                                            layout.grid_rows, rp.ctypes.data, ci.ctypes.data,
                                            _stream_ptr(stream), C.byref(h)))
    return DeviceLayout(h.value, layout.shape, layout.block_size, layout.kind, layout.sink)


def blockify(shape: GridShape, pattern: PatternSpec, block_size: int) -> BlockLayout:
    """radial::blockify (block.hpp:59): computed on the GPU by K1, returned as host CSR."""
    return device_layout(shape, pattern, block_size).host()


def sparsity(layout) -> float:
    """1 - kept / R^2 (block.hpp:123-126)."""
    R = layout.grid_rows
    return 1.0 - layout.kept_blocks() / float(R * R)


@dataclass
class FlopsReport:
    dense_flops: float = 0.0
    sparse_flops: float = 0.0
    reduction: float = 0.0


def attention_flops(layout, head_dim: int, num_heads: int) -> FlopsReport:
    """QK^T + PV FLOPs, whole B x B blocks (block.hpp:137-148)."""
    if head_dim < 1:
        raise ValueError("attention_flops: head_dim must be >= 1")
    if num_heads < 1:
        raise ValueError("attention_flops: num_heads must be >= 1")
    n = float(layout.shape.total_tokens())
    B = float(layout.block_size)
    dense = 4.0 * n * n * head_dim * num_heads
    sparse = 4.0 * float(layout.kept_blocks()) * B * B * head_dim * num_heads
    return FlopsReport(dense, sparse, dense / sparse if sparse else float("inf"))


# ---------------------------------------------------------------------------
# .ramk serialization (block.hpp:218-307)
# ---------------------------------------------------------------------------
def serialize(layout: BlockLayout) -> bytes:
    head = b"RAMK" + struct.pack("<HIIIBBI", 1, layout.shape.frames, layout.shape.tokens_per_frame,
                                 layout.block_size, layout.kind, 1 if layout.sink else 0,
                                 layout.grid_rows)
    return (head + np.ascontiguousarray(layout.row_ptr, "<u8").tobytes()
            + np.ascontiguousarray(layout.col_idx, "<u4").tobytes())


def deserialize(data: bytes) -> BlockLayout:
    pos = 0

    def take(fieldname: str, nbytes: int) -> bytes:
        nonlocal pos
        if len(data) - pos < nbytes:
            raise ParseError(fieldname, f"truncated: need {nbytes} bytes, have {len(data) - pos}")
        out = data[pos:pos + nbytes]
        pos += nbytes
        return out

    magic = take("magic", 4)
    if magic != b"RAMK":
        raise ParseError("magic", 'expected "RAMK"')
    (version,) = struct.unpack("<H", take("version", 2))
    if version != 1:
        raise ParseError("version", f"unsupported version {version}")
    (f,) = struct.unpack("<I", take("frames", 4))
    (s,) = struct.unpack("<I", take("tokens_per_frame", 4))
    (B,) = struct.unpack("<I", take("block_size", 4))
    kind = take("kind", 1)[0]
    sink = take("sink", 1)[0]
    (R,) = struct.unpack("<I", take("grid_rows", 4))
    if f < 1:
        raise ParseError("frames", "must be >= 1")
    if s < 1:
        raise ParseError("tokens_per_frame", "must be >= 1")
    if f * s > (1 << 32):
        raise ParseError("tokens_per_frame", "shape exceeds 2^32 tokens")
    if B < 1:
        raise ParseError("block_size", "must be >= 1")
    if kind > PatternKind.harmonic:
        raise ParseError("kind", f"unknown pattern kind {kind}")
    if sink > 1:
        raise ParseError("sink", "must be 0 or 1")
    shape = GridShape(f, s)
    expect = grid_rows_for(shape, B)
    if R != expect:
        raise ParseError("grid_rows", f"expected {expect} for this shape, got {R}")
    # The reference reads entry by entry (block.hpp:276-294): validate the complete
    # entries that are present first, then report truncation.
    m = min(R + 1, (len(data) - pos) // 8)
    row_ptr = np.frombuffer(data[pos:pos + 8 * m], "<u8").astype(np.uint64)
    pos += 8 * m
    bad = np.nonzero(row_ptr[1:] < row_ptr[:-1])[0]
    if len(bad):
        raise ParseError("row_ptr", f"not nondecreasing at row {int(bad[0]) + 1}")
    if m < R + 1:
        take("row_ptr", 8)
    nnz = int(row_ptr[-1])
    if nnz > R * R:
        raise ParseError("row_ptr", "kept-block count exceeds grid capacity")
    m = min(nnz, (len(data) - pos) // 4)
    col_idx = np.frombuffer(data[pos:pos + 4 * m], "<u4").astype(np.uint32)
    pos += 4 * m
    oob = np.nonzero(col_idx >= R)[0]
    if len(oob):
        e = int(oob[0])
        raise ParseError("col_idx", f"column {int(col_idx[e])} out of range at entry {e}")
    if m < nnz:
        take("col_idx", 4)
    for row in range(R):
        seg = col_idx[int(row_ptr[row]):int(row_ptr[row + 1])].astype(np.int64)
        if len(seg) > 1 and (np.diff(seg) <= 0).any():
            raise ParseError("col_idx", f"not strictly increasing in row {row}")
    if pos != len(data):
        raise ParseError("trailer", f"{len(data) - pos} trailing bytes")
    return BlockLayout(shape, B, R, row_ptr, col_idx, kind, bool(sink))


# ---------------------------------------------------------------------------
# attention.hpp (device path)
# ---------------------------------------------------------------------------
def _check_qkv(q, k, v):
    import torch
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError(f"masked_attention: {name} must be a CUDA tensor")
        if t.dtype != torch.bfloat16:
            raise ValueError(f"masked_attention: {name} must be bfloat16")
        if t.dim() != 3 or not t.is_contiguous():
            raise ValueError(f"masked_attention: {name} must be contiguous [heads, n, head_dim]")
    if not (q.shape == k.shape == v.shape):
        raise ValueError("masked_attention: Q, K and V must have the same shape")
    return q.shape


def _check_out(o, lse, q, who: str):
    """Caller-provided outputs must match what the kernel writes: O bf16 contiguous with q's
    shape and device, lse fp32 contiguous [heads, n] on the same device."""
    import torch
    H, n, _ = q.shape
    if o is not None:
        if (not isinstance(o, torch.Tensor) or o.dtype != torch.bfloat16 or tuple(o.shape) != tuple(q.shape)
                or o.device != q.device or not o.is_contiguous()):
            raise ValueError(f"{who}: out must be a contiguous bfloat16 tensor of shape {tuple(q.shape)} on {q.device}")
    if lse is not None:
        if (not isinstance(lse, torch.Tensor) or lse.dtype != torch.float32 or tuple(lse.shape) != (H, n)
                or lse.device != q.device or not lse.is_contiguous()):
            raise ValueError(f"{who}: lse must be a contiguous float32 tensor of shape {(H, n)} on {q.device}")


def _as_device_layout(layout) -> DeviceLayout:
    if isinstance(layout, DeviceLayout):
        return layout
    if isinstance(layout, BlockLayout):
        return layout_from_host(layout)
    raise ValueError("masked_attention: layout must be a DeviceLayout or BlockLayout")


def masked_attention(q, k, v, layout, scale: Optional[float] = None, *, out=None, lse=None,
                     return_lse: bool = False, stream=None):
    """radial::masked_attention(inst, layout) (attention.hpp:229-270) for all heads.

    q, k, v: bf16 CUDA [heads, n, head_dim] (head_dim 64 or 128); layout: DeviceLayout
    (block 64 or 128) or host BlockLayout.  Returns O (bf16) [and lse fp32 [heads, n]]."""
    import torch
    H, n, d = _check_qkv(q, k, v)
    L = _as_device_layout(layout)
    if L.shape.total_tokens() != n:
        raise ValueError("masked_attention: layout shape mismatch")
    _check_out(out, lse, q, "masked_attention")
    o = out if out is not None else torch.empty_like(q)
    if return_lse and lse is None:
        lse = torch.empty((H, n), dtype=torch.float32, device=q.device)
    _check(_lib.radial_cuda_attn_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                     lse.data_ptr() if lse is not None else None, H, n, d,
                                     float(scale or 0.0), L.handle, _stream_ptr(stream)))
    return (o, lse) if return_lse else o


def masked_attention_scatter(q, k, v, layout, dst_ptrs, head_base: int, heads_full: int,
                             scale: Optional[float] = None, *, lse=None, stream=None):
    """Head-parallel forward with the reassembly fused into the kernel epilogue: every O
    row of these heads is stored into each buffer of `dst_ptrs` (1..8 device pointers to bf16
    [heads_full, n, head_dim], e.g. every rank's full-O buffer mapped as peer memory) at
    head `head_base + h`.  The caller synchronises the ranks afterwards."""
    H, n, d = _check_qkv(q, k, v)
    L = _as_device_layout(layout)
    if L.shape.total_tokens() != n:
        raise ValueError("masked_attention: layout shape mismatch")
    _check_out(None, lse, q, "masked_attention_scatter")
    ptrs = (_vp * len(dst_ptrs))(*[int(x) for x in dst_ptrs])
    _check(_lib.radial_cuda_attn_fwd_scatter(q.data_ptr(), k.data_ptr(), v.data_ptr(), ptrs, len(dst_ptrs),
                                             head_base, heads_full,
                                             lse.data_ptr() if lse is not None else None, H, n, d,
                                             float(scale or 0.0), L.handle, _stream_ptr(stream)))


def masked_attention_pattern(q, k, v, shape: GridShape, pattern: PatternSpec, scale: Optional[float] = None,
                             *, block_size: int = 128, out=None, lse=None, return_lse: bool = False,
                             stream=None):
    """radial::masked_attention(inst, PatternSpec) (attention.hpp:184-225): the token-exact
    mask (no block over-approximation).  The kernel walks the blocks of the pattern's
    block layout and keeps exactly the token pairs of the keep rule (mask.hpp:105-154)."""
    import torch
    H, n, d = _check_qkv(q, k, v)
    if shape.total_tokens() != n:
        raise ValueError("masked_attention: layout shape mismatch")
    L = device_layout(shape, pattern, block_size, stream=stream)
    _check_out(out, lse, q, "masked_attention")
    o = out if out is not None else torch.empty_like(q)
    if return_lse and lse is None:
        lse = torch.empty((H, n), dtype=torch.float32, device=q.device)
    _check(_lib.radial_cuda_attn_fwd_token(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                           lse.data_ptr() if lse is not None else None, H, n, d,
                                           float(scale or 0.0), L.handle, _stream_ptr(stream)))
    return (o, lse) if return_lse else o


def dense_attention(q, k, v, scale: Optional[float] = None, *, block_size: int = 128, out=None,
                    lse=None, return_lse: bool = False, stream=None):
    """radial::dense_attention (attention.hpp:141-163): the dense comparator kernel (K4)."""
    import torch
    H, n, d = _check_qkv(q, k, v)
    _check_out(out, lse, q, "dense_attention")
    o = out if out is not None else torch.empty_like(q)
    if return_lse and lse is None:
        lse = torch.empty((H, n), dtype=torch.float32, device=q.device)
    _check(_lib.radial_cuda_attn_fwd_dense(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                           lse.data_ptr() if lse is not None else None, H, n, d,
                                           block_size, float(scale or 0.0), _stream_ptr(stream)))
    return (o, lse) if return_lse else o


def masked_attention_host(q: np.ndarray, k: np.ndarray, v: np.ndarray, layout,
                          scale: Optional[float] = None, *, o: Optional[np.ndarray] = None,
                          lse: Optional[np.ndarray] = None):
    """Host-buffer forward through the C-ABI (radial_cuda_attn_fwd_host): q/k/v are bf16
    bit patterns (numpy uint16) [heads, n, head_dim] in host memory; H2D, kernel, D2H."""
    for name, a in (("q", q), ("k", k), ("v", v)):
        if a.dtype != np.uint16 or a.ndim != 3 or not a.flags.c_contiguous:
            raise ValueError(f"masked_attention_host: {name} must be contiguous uint16 (bf16 bits)"
                             " [heads, n, head_dim]")
    if not (q.shape == k.shape == v.shape):
        raise ValueError("masked_attention_host: Q, K and V must have the same shape")
    H, n, d = q.shape
    L = _as_device_layout(layout)
    if o is None:
        o = np.empty_like(q)
    elif o.dtype != np.uint16 or o.shape != q.shape or not o.flags.c_contiguous or not o.flags.writeable:
        raise ValueError(f"masked_attention_host: o must be a writeable contiguous uint16 array of shape {q.shape}")
    if lse is not None and (lse.dtype != np.float32 or lse.shape != (H, n) or not lse.flags.c_contiguous
                            or not lse.flags.writeable):
        raise ValueError(f"masked_attention_host: lse must be a writeable contiguous float32 array of shape {(H, n)}")
    _check(_lib.radial_cuda_attn_fwd_host(q.ctypes.data, k.ctypes.data, v.ctypes.data, o.ctypes.data,
                                          lse.ctypes.data if lse is not None else None, H, n, d,
                                          float(scale or 0.0), L.handle, None))
    return o


def masked_attention_backward(q, k, v, o, lse, dout, layout, scale: Optional[float] = None, *,
                              stream=None):
    """Gradients (dq, dk, dv) of :func:`masked_attention` over the same layout (K3)."""
    import torch
    H, n, d = _check_qkv(q, k, v)
    if o is None or lse is None or dout is None:
        raise ValueError("masked_attention_backward: o, lse (the forward's return_lse=True outputs) and dout "
                         "are required")
    _check_out(o, lse, q, "masked_attention_backward")
    _check_out(dout, None, q, "masked_attention_backward (dout)")
    L = _as_device_layout(layout)
    dq = torch.empty_like(q)
    dk = torch.empty_like(k)
    dv = torch.empty_like(v)
    ws_bytes = _lib.radial_cuda_attn_bwd_workspace_size(H, n, d)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    _check(_lib.radial_cuda_attn_bwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                     lse.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(),
                                     dv.data_ptr(), H, n, d, float(scale or 0.0), L.handle,
                                     ws.data_ptr(), _stream_ptr(stream)))
    return dq, dk, dv


def _radial_attention_function():
    """torch.autograd.Function over K2 (forward) and K3 (backward), built lazily so that
    importing the package does not require torch."""
    global _RadialAttnFn
    if _RadialAttnFn is not None:
        return _RadialAttnFn
    import torch

    class RadialAttentionFn(torch.autograd.Function):
        @staticmethod
        def forward(ctx, q, k, v, layout, scale):
            q, k, v = (x.contiguous() for x in (q, k, v))
            o, lse = masked_attention(q, k, v, layout, scale, return_lse=True)
            ctx.save_for_backward(q, k, v, o, lse)
            ctx.layout, ctx.scale = layout, scale
            return o

        @staticmethod
        def backward(ctx, do):
            q, k, v, o, lse = ctx.saved_tensors
            dq, dk, dv = masked_attention_backward(q, k, v, o, lse, do.contiguous(), ctx.layout, ctx.scale)
            return dq, dk, dv, None, None

    _RadialAttnFn = RadialAttentionFn
    return _RadialAttnFn


_RadialAttnFn = None


def radial_attention(q, k, v, layout, scale: Optional[float] = None):
    """Differentiable radial attention for training (the paper's LoRA length-extension
    tuning): O = masked_attention(q, k, v, layout) with autograd through the
    K3 backward.  q, k, v bf16 CUDA [heads, n, head_dim] (head_dim 64 / 128, block 128 for
    the backward); gradients come back bf16 in the same layout."""
    return _radial_attention_function().apply(q, k, v, layout, scale)
