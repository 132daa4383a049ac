"""TEST INFRASTRUCTURE ONLY -- the parity checker for the radial hot path.

Two checkers, both loaded through ctypes:

* ``C``   -- ``_build/libradial_oracle.so``: the plain-C restatement of the
  reference algorithm (``radial_oracle.c``; each function cites the
  reference file:line it follows).
* ``REF`` -- ``_ref/libradial_ref.so``: the unmodified reference headers
  (``/root/reference/proj/include``) behind an ``extern "C"`` shim, built by
  ``oracle/Makefile`` with the reference's Release flags.  Used to pin the
  restatement and as the CPU baseline (``cpu_baseline.kind = "reference"``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline
/ reference-arm legs may import this package; the product package
(``paper_2506_19852_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libradial_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libradial_ref.so")

KIND = {"radial": 0, "dense": 1, "spatial": 2, "temporal": 3, "sta": 4, "power": 5, "harmonic": 6}

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32, _u64, _i32, _i64, _f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_double


def _load_c():
    lib = C.CDLL(ORACLE_SO)
    lib.ro_kept_span.restype = _i32
    lib.ro_kept_span.argtypes = [_i32, _i32, _u32, _u32, _u32, _u32, _u32, _u32, _u32,
                                 C.POINTER(_u32), C.POINTER(_u32)]
    lib.ro_radial_keep.restype = _i32
    lib.ro_radial_keep.argtypes = [_u32, _u32, _u32, _u32, _u32, _i32]
    lib.ro_grid_rows.restype = _u64
    lib.ro_grid_rows.argtypes = [_u32, _u32, _u32]
    lib.ro_blockify_rowptr.restype = _i64
    lib.ro_blockify_rowptr.argtypes = [_u32, _u32, _u32, _i32, _i32, _u32, _u32, _u64p]
    lib.ro_blockify_colidx.restype = _i32
    lib.ro_blockify_colidx.argtypes = [_u32, _u32, _u32, _i32, _i32, _u32, _u32, _u64p, _u32p]
    lib.ro_serialize.restype = C.c_size_t
    lib.ro_serialize.argtypes = [_u32, _u32, _u32, _i32, _i32, _u64, _u64p, _u32p, C.c_void_p]
    lib.ro_random_instance.restype = None
    lib.ro_random_instance.argtypes = [_u64, _u32, _u64, _f64p, _f64p, _f64p]
    for name, fp in (("ro_attention_rows_f32", _f32p), ("ro_attention_rows_f64", _f64p)):
        fn = getattr(lib, name)
        fn.restype = _i32
        fn.argtypes = [_u64, _u32, fp, fp, fp, _u32, C.c_void_p, C.c_void_p, _u64p, _u64, _f64,
                       _f64p, C.c_void_p, C.POINTER(_u64)]
    lib.ro_token_attention_rows_f32.restype = _i32
    lib.ro_token_attention_rows_f32.argtypes = [_u64, _u32, _f32p, _f32p, _f32p, _u32, _u32, _i32, _i32,
                                                _u32, _u32, _u64p, _u64, _f64, _f64p, C.c_void_p]
    lib.ro_attention_bwd_f32.restype = _i32
    lib.ro_attention_bwd_f32.argtypes = [_u64, _u32, _f32p, _f32p, _f32p, _f32p, _u32, C.c_void_p,
                                         C.c_void_p, _f64, _f64p, _f64p, _f64p]
    return lib


def _load_ref():
    lib = C.CDLL(REF_SO)
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_blockify_serialize.restype = _i64
    lib.ref_blockify_serialize.argtypes = [_u32, _u32, _u32, _i32, _i32, _u32, _u32, C.c_void_p, _u64]
    lib.ref_radial_keep.restype = _i32
    lib.ref_radial_keep.argtypes = [_u32, _u32, _u32, _u32, _u32, _u32, _i32]
    lib.ref_count_kept.restype = _i64
    lib.ref_count_kept.argtypes = [_u32, _u32, _i32, _i32, _u32, _u32]
    lib.ref_random_instance.restype = _i32
    lib.ref_random_instance.argtypes = [_u32, _u32, _u32, _u64, _f64p, _f64p, _f64p]
    lib.ref_masked_attention.restype = _i32
    lib.ref_masked_attention.argtypes = [_u32, _u32, _u32, _f64p, _f64p, _f64p, _u32, _u32, _u64p,
                                         _u32p, _f64p]
    lib.ref_dense_attention.restype = _i32
    lib.ref_dense_attention.argtypes = [_u32, _u32, _u32, _f64p, _f64p, _f64p, _f64p]
    lib.ref_attention_flops.restype = _i32
    lib.ref_attention_flops.argtypes = [_u32, _u32, _u32, _i32, _u32, _u32] + [C.POINTER(_f64)] * 4
    lib.ref_masked_attention_pattern.restype = _i32
    lib.ref_masked_attention_pattern.argtypes = [_u32, _u32, _u32, _f64p, _f64p, _f64p, _i32, _i32, _u32,
                                                 _u32, _f64p]
    lib.ref_instance_create.restype = C.c_void_p
    lib.ref_instance_create.argtypes = [_u32, _u32, _u32, _u64]
    lib.ref_instance_free.restype = None
    lib.ref_instance_free.argtypes = [C.c_void_p]
    lib.ref_masked_attention_inst.restype = _i32
    lib.ref_masked_attention_inst.argtypes = [C.c_void_p, _u32, _u32, _u64p, _u32p, C.c_void_p]
    return lib


_C = None
_REF = None


def c():
    global _C
    if _C is None:
        _C = _load_c()
    return _C


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _REF
    if _REF is None:
        _REF = _load_ref()
    return _REF


# --------------------------------------------------------------------------
# Layouts
# --------------------------------------------------------------------------
def blockify(f, s, B, kind="radial", sink=True, tw=0, sw=0):
    """C restatement of blockify (block.hpp:59-120) -> (row_ptr u64[R+1], col_idx u32[nnz])."""
    lib = c()
    R = int(lib.ro_grid_rows(f, s, B))
    row_ptr = np.zeros(R + 1, np.uint64)
    nnz = lib.ro_blockify_rowptr(f, s, B, KIND[kind], int(sink), tw, sw, row_ptr)
    if nnz < 0:
        raise ValueError("blockify: bad arguments")
    col_idx = np.zeros(max(nnz, 1), np.uint32)
    lib.ro_blockify_colidx(f, s, B, KIND[kind], int(sink), tw, sw, row_ptr, col_idx)
    return row_ptr, col_idx[:nnz]


def serialize(f, s, B, kind, sink, row_ptr, col_idx) -> bytes:
    """.ramk bytes (block.hpp:218-237) of a CSR layout."""
    lib = c()
    R = len(row_ptr) - 1
    ci = np.ascontiguousarray(col_idx if len(col_idx) else np.zeros(1, np.uint32), np.uint32)
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    size = lib.ro_serialize(f, s, B, KIND[kind], int(sink), R, rp, ci, None)
    buf = np.zeros(size, np.uint8)
    lib.ro_serialize(f, s, B, KIND[kind], int(sink), R, rp, ci, buf.ctypes.data)
    return buf.tobytes()


def layout_sha256(f, s, B, kind="radial", sink=True, tw=0, sw=0) -> str:
    rp, ci = blockify(f, s, B, kind, sink, tw, sw)
    return hashlib.sha256(serialize(f, s, B, kind, sink, rp, ci)).hexdigest()


def ref_serialize(f, s, B, kind="radial", sink=True, tw=0, sw=0) -> bytes:
    """The reference's own serialize(blockify(...)) bytes."""
    lib = ref()
    size = lib.ref_blockify_serialize(f, s, B, KIND[kind], int(sink), tw, sw, None, 0)
    if size < 0:
        raise ValueError(lib.ref_last_error().decode())
    buf = np.zeros(size, np.uint8)
    lib.ref_blockify_serialize(f, s, B, KIND[kind], int(sink), tw, sw, buf.ctypes.data, size)
    return buf.tobytes()


def parse_ramk(data: bytes):
    """Minimal .ramk reader for tests: -> dict(f, s, B, kind, sink, R, row_ptr, col_idx)."""
    assert data[:4] == b"RAMK"
    f, s, B = np.frombuffer(data[6:18], "<u4")
    kind, sink = data[18], data[19]
    R = int(np.frombuffer(data[20:24], "<u4")[0])
    row_ptr = np.frombuffer(data[24:24 + 8 * (R + 1)], "<u8").astype(np.uint64)
    col_idx = np.frombuffer(data[24 + 8 * (R + 1):], "<u4").astype(np.uint32)
    return dict(f=int(f), s=int(s), B=int(B), kind=int(kind), sink=int(sink), R=R,
                row_ptr=row_ptr, col_idx=col_idx)


# --------------------------------------------------------------------------
# Instances and attention
# --------------------------------------------------------------------------
def random_instance(n, d, seed):
    """C restatement of random_instance (attention.hpp:89-104) -> q, k, v (n, d) float64."""
    q = np.empty((n, d), np.float64)
    k = np.empty((n, d), np.float64)
    v = np.empty((n, d), np.float64)
    c().ro_random_instance(n, d, seed, q, k, v)
    return q, k, v


def ref_random_instance(f, s, d, seed):
    n = f * s
    q = np.empty((n, d), np.float64)
    k = np.empty((n, d), np.float64)
    v = np.empty((n, d), np.float64)
    if ref().ref_random_instance(f, s, d, seed, q, k, v) != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return q, k, v


def attention_rows(q, k, v, B, row_ptr, col_idx, rows, scale=0.0, want_lse=False):
    """fp64 restatement of masked_attention(inst, layout) (attention.hpp:229-270) for the
    given query token rows; row_ptr=None means dense (attention.hpp:141-163)."""
    n, d = q.shape
    rows = np.ascontiguousarray(rows, np.uint64)
    out = np.zeros((len(rows), d), np.float64)
    lse = np.zeros(len(rows), np.float64) if want_lse else None
    bad = _u64(0)
    if q.dtype == np.float32:
        fn = c().ro_attention_rows_f32
    else:
        fn = c().ro_attention_rows_f64
        q, k, v = (np.ascontiguousarray(x, np.float64) for x in (q, k, v))
    rp = None if row_ptr is None else np.ascontiguousarray(row_ptr, np.uint64)
    ci = None if row_ptr is None else np.ascontiguousarray(
        col_idx if len(col_idx) else np.zeros(1, np.uint32), np.uint32)
    st = fn(n, d, q, k, v, B, None if rp is None else rp.ctypes.data,
            None if ci is None else ci.ctypes.data, rows, len(rows), scale, out,
            None if lse is None else lse.ctypes.data, C.byref(bad))
    if st == 2:
        raise RuntimeError(f"masked_attention: query row {bad.value} keeps no keys")
    return (out, lse) if want_lse else out


def token_attention_rows(q, k, v, f, s, rows, kind="radial", sink=True, tw=0, sw=0, scale=0.0,
                         want_lse=False):
    """fp64 restatement of masked_attention(inst, PatternSpec) (attention.hpp:184-225), the
    token-exact path, for the given query rows (fp32 inputs)."""
    n, d = q.shape
    rows = np.ascontiguousarray(rows, np.uint64)
    out = np.zeros((len(rows), d), np.float64)
    lse = np.zeros(len(rows), np.float64) if want_lse else None
    f32 = lambda x: np.ascontiguousarray(x, np.float32)
    st = c().ro_token_attention_rows_f32(n, d, f32(q), f32(k), f32(v), f, s, KIND[kind], int(sink), tw,
                                         sw, rows, len(rows), scale, out,
                                         None if lse is None else lse.ctypes.data)
    if st != 0:
        raise RuntimeError("token_attention_rows failed")
    return (out, lse) if want_lse else out


def ref_masked_attention_pattern(f, s, q, k, v, kind="radial", sink=True, tw=0, sw=0):
    """The reference's own token-exact masked_attention(inst, PatternSpec)."""
    n, d = q.shape
    out = np.zeros((n, d), np.float64)
    st = ref().ref_masked_attention_pattern(f, s, d, np.ascontiguousarray(q, np.float64),
                                            np.ascontiguousarray(k, np.float64),
                                            np.ascontiguousarray(v, np.float64), KIND[kind], int(sink),
                                            tw, sw, out)
    if st != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return out


def attention_bwd(q, k, v, do, B, row_ptr, col_idx, scale=0.0):
    """fp64 gradients (dq, dk, dv) of the block-masked attention (no reference exists)."""
    n, d = q.shape
    f32 = lambda x: np.ascontiguousarray(x, np.float32)
    dq = np.zeros((n, d)); dk = np.zeros((n, d)); dv = np.zeros((n, d))
    rp = None if row_ptr is None else np.ascontiguousarray(row_ptr, np.uint64)
    ci = None if row_ptr is None else np.ascontiguousarray(
        col_idx if len(col_idx) else np.zeros(1, np.uint32), np.uint32)
    st = c().ro_attention_bwd_f32(n, d, f32(q), f32(k), f32(v), f32(do), B,
                                  None if rp is None else rp.ctypes.data,
                                  None if ci is None else ci.ctypes.data, scale, dq, dk, dv)
    if st != 0:
        raise RuntimeError("attention_bwd: empty row")
    return dq, dk, dv


def ref_masked_attention(f, s, q, k, v, B, row_ptr, col_idx):
    """The reference's own masked_attention(inst, layout) on float64 q/k/v."""
    n, d = q.shape
    out = np.zeros((n, d), np.float64)
    ci = np.ascontiguousarray(col_idx if len(col_idx) else np.zeros(1, np.uint32), np.uint32)
    st = ref().ref_masked_attention(f, s, d, np.ascontiguousarray(q, np.float64),
                                    np.ascontiguousarray(k, np.float64),
                                    np.ascontiguousarray(v, np.float64), B, len(row_ptr) - 1,
                                    np.ascontiguousarray(row_ptr, np.uint64), ci, out)
    if st == 1:
        raise ValueError(ref().ref_last_error().decode())
    if st != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return out


def ref_dense_attention(f, s, q, k, v):
    n, d = q.shape
    out = np.zeros((n, d), np.float64)
    st = ref().ref_dense_attention(f, s, d, np.ascontiguousarray(q, np.float64),
                                   np.ascontiguousarray(k, np.float64),
                                   np.ascontiguousarray(v, np.float64), out)
    if st != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32 (what the GPU receives)."""
    a = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    a = (a + 0x7FFF + ((a >> 16) & 1)) & 0xFFFF0000
    return a.astype(np.uint32).view(np.float32)


# --------------------------------------------------------------------------
# CPU baseline: the reference's masked_attention on a bounded sample
# --------------------------------------------------------------------------
def sample_layout(row_ptr, col_idx, n, B, threads, per_thread=1):
    """A layout for timing the reference on a bounded sample of the real workload:
    `per_thread` query blocks inside each of the reference's static parallel_for chunks
    (parallel.hpp:42-47, chunk = ceil(n/threads) tokens) keep their true KV lists; every
    other block row keeps only its first kept block (so no row is empty).  Returns
    (row_ptr, col_idx, kept_blocks_executed, sampled_blocks)."""
    R = len(row_ptr) - 1
    threads = max(1, min(threads, n))
    chunk = -(-n // threads)
    sampled = set()
    for t in range(threads):
        lo, hi = t * chunk, min(n, (t + 1) * chunk)
        if lo >= hi:
            break
        for p in range(per_thread):
            u = lo + (2 * p + 1) * (hi - lo) // (2 * per_thread)
            sampled.add(min(u // B, R - 1))
    lens = np.diff(row_ptr.astype(np.int64))
    new_lens = np.where(np.isin(np.arange(R), sorted(sampled)), lens, np.minimum(lens, 1))
    rp = np.concatenate([[0], np.cumsum(new_lens)]).astype(np.uint64)
    ci = np.empty(int(rp[-1]), np.uint32)
    for I in range(R):
        a = int(row_ptr[I])
        ci[int(rp[I]):int(rp[I + 1])] = col_idx[a:a + int(new_lens[I])]
    return rp, ci, int(rp[-1]), sorted(sampled)


class RefInstance:
    """A persistent reference AttentionInstance (random_instance(f, s, d, seed))."""

    def __init__(self, f, s, d, seed):
        self.f, self.s, self.d = f, s, d
        self.h = ref().ref_instance_create(f, s, d, seed)
        if not self.h:
            raise RuntimeError(ref().ref_last_error().decode())

    def masked_attention(self, B, row_ptr, col_idx):
        st = ref().ref_masked_attention_inst(self.h, B, len(row_ptr) - 1,
                                             np.ascontiguousarray(row_ptr, np.uint64),
                                             np.ascontiguousarray(col_idx, np.uint32), None)
        if st != 0:
            raise RuntimeError(ref().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_instance_free(self.h)
            self.h = None
