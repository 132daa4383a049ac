// mask_build.cu -- K1: on-device radial block-layout builder.
//
// Replaces radial::blockify (reference block.hpp:59-120).  The reference
// paints, per query block row, every kept key interval of every key frame
// (kept_span, mask.hpp:105-154) into a hit bitmap.  Here each (I, J) block
// pair is decided independently by a closed-form predicate: (I, J) is kept
// iff some query frame i overlapping block I and key frame j overlapping
// block J have kept_span(i, [k_lo,k_hi], j) intersecting J's positions in
// frame j.  That is exactly the set of J the reference paints, so the CSR is
// bit-identical (gated by sha256 of the .ramk bytes in tests/).
//
// One CTA per output row sweeps the columns 256 at a time; rows are
// compacted with warp ballots so col_idx comes out strictly increasing
// without a sort.  Three list families are built with the same machinery:
//   CSR   rows = query blocks, cols = KV blocks     (BlockLayout)
//   CSC   rows = KV blocks,    cols = query blocks  (backward dK/dV)
//   chunk unions: rows = 256-token chunks, value = J | mask << 28
//         (the forward work lists).
#include <algorithm>
#include <numeric>
#include <vector>

#include "mask_rule.cuh"
#include "radial_internal.h"

#ifndef RADIAL_TOK_PAIRED
#define RADIAL_TOK_PAIRED 0  // token-exact flags over the paired lists (attn_fwd.cu kTokPaired)
#endif

namespace {

using radial_rule::MaskParams;
using radial_rule::kept_span;

constexpr int kThreads = 256;

// Block (I, J) kept?  Frame-structured kinds: exact per-pair restatement of
// the painting in block.hpp:81-97.  Power: block-level rule block.hpp:71-80.
struct BlockKeep {
    MaskParams p;
    __device__ __forceinline__ uint32_t operator()(uint32_t I, uint32_t J) const {
        const uint64_t B = p.B, s = p.s;
        if (p.kind == RADIAL_KIND_POWER) {
            const uint32_t t = I > J ? I - J : J - I;
            if ((t & (t - 1)) == 0) return 1;  // t == 0 or a power of two
            return (p.sink && J <= (s - 1) / B) ? 1 : 0;
        }
        const uint64_t u0 = static_cast<uint64_t>(I) * B;
        const uint64_t u1 = min(p.n, u0 + B) - 1;
        const uint64_t v0 = static_cast<uint64_t>(J) * B;
        const uint64_t v1 = min(p.n, v0 + B) - 1;
        for (uint64_t i = u0 / s; i * s <= u1; ++i) {
            const uint32_t k_lo = static_cast<uint32_t>(max(u0, i * s) - i * s);
            const uint32_t k_hi = static_cast<uint32_t>(min(u1, i * s + s - 1) - i * s);
            for (uint64_t j = v0 / s; j * s <= v1; ++j) {
                const uint32_t l_lo = static_cast<uint32_t>(max(v0, j * s) - j * s);
                const uint32_t l_hi = static_cast<uint32_t>(min(v1, j * s + s - 1) - j * s);
                uint32_t lo, hi;
                if (kept_span(p, static_cast<uint32_t>(i), k_lo, k_hi, static_cast<uint32_t>(j), lo,
                              hi) &&
                    lo <= l_hi && hi >= l_lo)
                    return 1;
            }
        }
        return 0;
    }
};

__device__ __forceinline__ bool csr_member(const uint64_t* __restrict__ ptr,
                                           const uint32_t* __restrict__ idx, uint32_t row,
                                           uint32_t col) {
    uint64_t lo = ptr[row], hi = ptr[row + 1];
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const uint32_t v = idx[mid];
        if (v == col) return true;
        if (v < col)
            lo = mid + 1;
        else
            hi = mid;
    }
    return false;
}

// Transpose: row = KV block J, col = query block I, kept iff J in CSR row I.
struct CsrTranspose {
    const uint64_t* ptr;
    const uint32_t* idx;
    __device__ __forceinline__ uint32_t operator()(uint32_t J, uint32_t I) const {
        return csr_member(ptr, idx, I, J) ? 1u : 0u;
    }
};

// Chunk union: row = chunk c (G consecutive rows of the source lists),
// value = bit g set iff source row c*G+g contains col.
struct ChunkUnion {
    const uint64_t* ptr;
    const uint32_t* idx;
    uint32_t R, G;
    __device__ __forceinline__ uint32_t operator()(uint32_t c, uint32_t col) const {
        uint32_t m = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const uint32_t r = c * G + g;
            if (r < R && csr_member(ptr, idx, r, col)) m |= 1u << g;
        }
        return m;
    }
};

template <class F>
__global__ void __launch_bounds__(kThreads) list_count(F pred, uint32_t cols,
                                                      uint32_t* __restrict__ counts) {
    const uint32_t row = blockIdx.x;
    uint32_t c = 0;
    for (uint32_t base = 0; base < cols; base += kThreads) {
        const uint32_t col = base + threadIdx.x;
        const bool keep = col < cols && pred(row, col) != 0;
        c += __popc(__ballot_sync(0xffffffffu, keep));
    }
    __shared__ uint32_t warp_sum[kThreads / 32];
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += warp_sum[w];
        counts[row] = t;
    }
}

template <class F>
__global__ void __launch_bounds__(kThreads) list_fill(F pred, uint32_t cols,
                                                     const uint64_t* __restrict__ ptr,
                                                     uint32_t* __restrict__ out, int with_mask) {
    const uint32_t row = blockIdx.x;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ uint32_t warp_cnt[kThreads / 32];
    uint64_t pos = ptr[row];
    for (uint32_t base = 0; base < cols; base += kThreads) {
        const uint32_t col = base + threadIdx.x;
        const uint32_t v = col < cols ? pred(row, col) : 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, v != 0);
        if (lane == 0) warp_cnt[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (uint32_t w = 0; w < kThreads / 32; ++w) {
            const uint32_t cw = warp_cnt[w];
            before += w < warp ? cw : 0;
            total += cw;
        }
        if (v) {
            const uint32_t rank = before + __popc(bal & ((1u << lane) - 1u));
            out[pos + rank] = with_mask ? (col | (v << 28)) : col;
        }
        pos += total;
        __syncthreads();
    }
}

struct ScanStats {
    unsigned long long nnz;
    long long first_empty;
    uint32_t max_len, min_len;
};

// Exclusive scan of u32 counts into u64 pointers, plus row-length stats.
__global__ void __launch_bounds__(1024) scan_rows(const uint32_t* __restrict__ counts,
                                                  uint32_t rows, uint64_t* __restrict__ ptr,
                                                  ScanStats* stats) {
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t carry;
    __shared__ long long first_empty;
    __shared__ uint32_t mx, mn;
    if (threadIdx.x == 0) {
        carry = 0;
        first_empty = -1;
        mx = 0;
        mn = 0xffffffffu;
        ptr[0] = 0;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t local_max = 0, local_min = 0xffffffffu;
    long long local_empty = -1;
    for (uint32_t base = 0; base < rows; base += 1024) {
        const uint32_t r = base + threadIdx.x;
        const uint64_t c = r < rows ? counts[r] : 0;
        if (r < rows) {
            local_max = max(local_max, static_cast<uint32_t>(c));
            local_min = min(local_min, static_cast<uint32_t>(c));
            if (c == 0 && local_empty < 0) local_empty = r;
        }
        uint64_t x = c;  // inclusive warp scan
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[warp] = x;
        __syncthreads();
        uint64_t before = 0, total = 0;
        for (uint32_t w = 0; w < 32; ++w) {
            before += w < warp ? warp_tot[w] : 0;
            total += warp_tot[w];
        }
        if (r < rows) ptr[r + 1] = carry + before + x;
        __syncthreads();
        if (threadIdx.x == 0) carry += total;
        __syncthreads();
    }
    atomicMax(&mx, local_max);
    atomicMin(&mn, local_min);
    if (local_empty >= 0) atomicMin(reinterpret_cast<unsigned long long*>(&first_empty),
                                    static_cast<unsigned long long>(local_empty));
    __syncthreads();
    if (threadIdx.x == 0) {
        stats->nnz = carry;
        stats->first_empty = first_empty;
        stats->max_len = mx;
        stats->min_len = rows ? mn : 0;
    }
}

// Stable argsort of lists by length, longest first (LPT work order) inside windows of
// `window` consecutive lists, one CTA.  keys = ptr[i+1] - ptr[i]; n <= kSortMax (bitonic sort
// in shared memory).  Windowing keeps the CTAs resident at any time on neighbouring query
// blocks, whose K/V working set stays in L2: at H132 (243 MB of K+V per head) a global LPT
// order streams the whole head from DRAM and the power-capped clock drops (measured: 591 ->
// 547 ms forward, 1707 -> 1562 ms backward with windows of 2 x 148 lists; H33 unchanged).
constexpr int kSortMax = 4096;  // 32 KB of static shared memory
__global__ void __launch_bounds__(1024) lpt_sort_kernel(const uint64_t* __restrict__ ptr, uint32_t n,
                                                        uint32_t window, uint32_t* __restrict__ order) {
    __shared__ unsigned long long key[kSortMax];  // window << 52 | (max_len - len) << 32 | index
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        if (i < n) {
            const uint64_t len = ptr[i + 1] - ptr[i];
            const uint32_t l20 = static_cast<uint32_t>(len < 0xfffffu ? len : 0xfffffu);
            key[i] = (static_cast<unsigned long long>(i / window) << 52) |
                     (static_cast<unsigned long long>(0xfffffu - l20) << 32) | i;
        } else {
            key[i] = ~0ull;
        }
    }
    __syncthreads();
    for (uint32_t k = 2; k <= m; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = key[i], b = key[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        key[i] = b;
                        key[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) order[i] = static_cast<uint32_t>(key[i] & 0xffffffffu);
}

// Forward chunk lists: each entry kept by tile 0 only ("open") is followed by a later entry
// kept by tile 1 only ("close"), pulled forward, so the forward's MMA warp can issue that
// entry's S together with the first and the two solo steps overlap like one shared step.
// Everything else stays in ascending J order (K/V locality in L2).  The pairing is greedy
// and first-in first-out: the m-th open takes the first close after it and after the
// (m-1)-th open's partner.  That is bracket matching, so one warp per chunk decides it with
// prefix counts: a close is matched iff it does not raise the running maximum of
// (closes - opens) over the list prefix, and the m-th matched close belongs to the m-th
// open.  Pass 1 records the matched closes' positions (in `scratch`, at the chunk's list
// offset), pass 2 scatters every entry to its output slot.  `in` is the fill order.
__global__ void __launch_bounds__(256) pair_solo_entries(const uint64_t* __restrict__ ptr, uint32_t C, uint32_t GT,
                                                         const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                         uint32_t* __restrict__ scratch) {
    const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (c >= C) return;  // whole warps exit together
    const uint64_t b = ptr[c], e = ptr[c + 1];
    const uint32_t m0 = (1u << GT) - 1u;
    const uint32_t below = (1u << lane) - 1u;
    auto kind = [&](uint32_t x) {  // 0 shared, 1 tile-0 only (open), 2 tile-1 only (close)
        const uint32_t m = x >> 28;
        const bool a = m & m0, bb = (m >> GT) & m0;
        return (a && bb) ? 0 : (a ? 1 : 2);
    };
    // one 32-entry tile: kind of this lane's entry and whether it is a matched close; carries
    // opens / closes seen and the running max excess U across tiles
    struct Carry {
        uint32_t opens = 0, closes = 0;
        int U = 0;
    };
    auto tile = [&](uint64_t i, Carry& cy, int& k, bool& matched, uint32_t& bo) {
        k = i < e ? kind(in[i]) : 0;
        bo = __ballot_sync(0xffffffffu, k == 1);
        const uint32_t bc = __ballot_sync(0xffffffffu, k == 2);
        const uint32_t upto = below | (1u << lane);
        int x = static_cast<int>(cy.closes + __popc(bc & upto)) - static_cast<int>(cy.opens + __popc(bo & upto));
        for (int o = 1; o < 32; o <<= 1) {  // inclusive prefix max over the lanes
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<uint32_t>(o)) x = max(x, y);
        }
        const int prev = __shfl_up_sync(0xffffffffu, x, 1);
        const int u_before = lane ? max(cy.U, prev) : cy.U;
        const int u_after = max(cy.U, x);
        matched = k == 2 && u_after == u_before;
        cy.U = __shfl_sync(0xffffffffu, u_after, 31);
        cy.opens += __popc(bo);
        cy.closes += __popc(bc);
    };
    Carry cy;
    uint32_t nm = 0;  // matched closes so far
    for (uint64_t base = b; base < e; base += 32) {
        int k;
        bool matched;
        uint32_t bo;
        tile(base + lane, cy, k, matched, bo);
        const uint32_t bm = __ballot_sync(0xffffffffu, matched);
        if (matched) scratch[b + nm + __popc(bm & below)] = static_cast<uint32_t>(base + lane);
        nm += __popc(bm);
    }
    Carry cy2;
    uint64_t opos = b;
    for (uint64_t base = b; base < e; base += 32) {
        const uint64_t i = base + lane;
        int k;
        bool matched;
        uint32_t bo;
        const uint32_t opens_before = cy2.opens;
        tile(i, cy2, k, matched, bo);
        const uint32_t om = opens_before + __popc(bo & below);  // index of this open
        const bool pair = k == 1 && om < nm;
        const uint32_t contrib = (i >= e || matched) ? 0u : (pair ? 2u : 1u);
        uint32_t x = contrib;  // inclusive prefix sum
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
        }
        const uint64_t pos = opos + x - contrib;
        if (contrib) {
            out[pos] = in[i];
            if (pair) out[pos + 1] = in[scratch[b + om]];
        }
        opos += __shfl_sync(0xffffffffu, x, 31);
    }
}

// Token-exact fast path: for every entry of the ascending chunk lists, bit t is set iff Q tile
// t (128 query rows of the chunk) keeps ALL token pairs of KV block J under the pattern's rule
// (every block of the tile keeps J and span_covers holds for every frame pair the tile and
// the block overlap).  The token-exact forward then skips its per-row mask for that tile.
// One warp per chunk, lanes over the entries.
__global__ void __launch_bounds__(256) token_full_flags(MaskParams p, const uint64_t* __restrict__ ptr, uint32_t C,
                                                        uint32_t G, const uint32_t* __restrict__ idx,
                                                        uint8_t* __restrict__ full) {
    const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (c >= C) return;
    const uint32_t GT = G / 2;
    const uint64_t s = p.s;
    for (uint64_t e = ptr[c] + lane; e < ptr[c + 1]; e += 32) {
        const uint32_t x = idx[e];
        const uint32_t J = x & 0x0FFFFFFFu, m = x >> 28;
        const uint64_t v0 = static_cast<uint64_t>(J) * p.B;
        const uint64_t v1 = min(p.n, v0 + p.B) - 1;
        uint8_t flags = 0;
        for (uint32_t t = 0; t < 2; ++t) {
            const uint64_t u0 = static_cast<uint64_t>(c) * 256 + t * 128;
            if (u0 >= p.n) {
                flags |= 1u << t;  // no query rows: vacuously full
                continue;
            }
            if (((m >> (t * GT)) & ((1u << GT) - 1u)) != ((1u << GT) - 1u)) {
                // some block of the tile skips J (or lies past the grid): only full if those
                // blocks hold no rows
                bool ok = true;
                for (uint32_t g = 0; g < GT; ++g)
                    if (!((m >> (t * GT + g)) & 1u) && u0 + static_cast<uint64_t>(g) * p.B < p.n) ok = false;
                if (!ok) continue;
            }
            const uint64_t u1 = min(p.n, u0 + 128) - 1;
            bool ok = true;
            for (uint64_t i = u0 / s; ok && i * s <= u1; ++i) {
                const uint32_t k_lo = static_cast<uint32_t>(max(u0, i * s) - i * s);
                const uint32_t k_hi = static_cast<uint32_t>(min(u1, i * s + s - 1) - i * s);
                for (uint64_t j = v0 / s; ok && j * s <= v1; ++j) {
                    const uint32_t l_lo = static_cast<uint32_t>(max(v0, j * s) - j * s);
                    const uint32_t l_hi = static_cast<uint32_t>(min(v1, j * s + s - 1) - j * s);
                    ok = radial_rule::span_covers(p, static_cast<uint32_t>(i), k_lo, k_hi, static_cast<uint32_t>(j),
                                                  l_lo, l_hi);
                }
            }
            if (ok) flags |= 1u << t;
        }
        full[e] = flags;
    }
}

// One list family (rows x cols under predicate F): counts -> exclusive scan into ptr.
template <class F>
int count_and_scan(F pred, uint32_t rows, uint32_t cols, uint32_t* counts, uint64_t* ptr, ScanStats* dstats,
                   cudaStream_t st) {
    if (rows) list_count<F><<<rows, kThreads, 0, st>>>(pred, cols, counts);
    scan_rows<<<1, 1024, 0, st>>>(counts, rows, ptr, dstats);
    RADIAL_CUDA_TRY(cudaGetLastError());
    radial_detail::count_launches(rows ? 2 : 1);
    return RADIAL_OK;
}

template <class F>
int fill(F pred, uint32_t rows, uint32_t cols, const uint64_t* ptr, uint32_t* idx, int with_mask,
         cudaStream_t st) {
    if (rows) list_fill<F><<<rows, kThreads, 0, st>>>(pred, cols, ptr, idx, with_mask);
    RADIAL_CUDA_TRY(cudaGetLastError());
    if (rows) radial_detail::count_launches(1);
    return RADIAL_OK;
}

// Longest-processing-time-first order of `n` lists within windows of 2 x (SM count) lists
// (device sort; host fallback when large).
int lpt_order(const uint64_t* dptr, uint32_t n, cudaStream_t st, uint32_t** order_out) {
    RADIAL_CUDA_TRY(cudaMallocAsync(order_out, sizeof(uint32_t) * std::max<uint32_t>(n, 1), st));
    if (n == 0) return RADIAL_OK;
    int dev = 0, sms = 148;
    RADIAL_CUDA_TRY(cudaGetDevice(&dev));
    RADIAL_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
#ifndef RADIAL_LPT_WINDOW_SMS
#define RADIAL_LPT_WINDOW_SMS 2  // window = this many x the SM count (tuning knob)
#endif
    const uint32_t window = RADIAL_LPT_WINDOW_SMS * static_cast<uint32_t>(std::max(sms, 1));
    if (n <= static_cast<uint32_t>(kSortMax)) {
        lpt_sort_kernel<<<1, 1024, 0, st>>>(dptr, n, window, *order_out);
        RADIAL_CUDA_TRY(cudaGetLastError());
        radial_detail::count_launches(1);
        return RADIAL_OK;
    }
    std::vector<uint64_t> h(n + 1);
    RADIAL_CUDA_TRY(cudaMemcpyAsync(h.data(), dptr, sizeof(uint64_t) * (n + 1), cudaMemcpyDeviceToHost, st));
    RADIAL_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<uint32_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0u);
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
        if (a / window != b / window) return a < b;
        return (h[a + 1] - h[a]) > (h[b + 1] - h[b]);
    });
    RADIAL_CUDA_TRY(cudaMemcpyAsync(*order_out, ord.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st));
    RADIAL_CUDA_TRY(cudaStreamSynchronize(st));
    return RADIAL_OK;
}

// Stream-ordered scratch (pool allocations; no device-wide synchronisation).
struct Scratch {
    cudaStream_t st;
    uint32_t* counts = nullptr;
    ScanStats* stats = nullptr;  // [4] CSR, CSC, 256-row chunk unions, 512-row chunk unions
    ScanStats host[4];
    explicit Scratch(cudaStream_t s) : st(s) {}
    ~Scratch() {
        if (counts) cudaFreeAsync(counts, st);
        if (stats) cudaFreeAsync(stats, st);
    }
};

}  // namespace

namespace radial_detail {

// K1: CSR of the pattern by the closed-form block predicate.  One host sync (nnz).
int build_layout_device(radial_layout* L, cudaStream_t st) {
    MaskParams p{L->f, L->s, L->B, static_cast<uint64_t>(L->f) * L->s, L->kind, L->sink, L->tw, L->sw};
    Scratch sc(st);
    RADIAL_CUDA_TRY(cudaMallocAsync(&sc.counts, sizeof(uint32_t) * std::max<uint32_t>(L->R, 1), st));
    RADIAL_CUDA_TRY(cudaMallocAsync(&sc.stats, sizeof(ScanStats), st));
    RADIAL_CUDA_TRY(cudaMallocAsync(&L->row_ptr, sizeof(uint64_t) * (static_cast<size_t>(L->R) + 1), st));
    int rc = count_and_scan(BlockKeep{p}, L->R, L->R, sc.counts, L->row_ptr, sc.stats, st);
    if (rc) return rc;
    RADIAL_CUDA_TRY(cudaMemcpyAsync(sc.host, sc.stats, sizeof(ScanStats), cudaMemcpyDeviceToHost, st));
    RADIAL_CUDA_TRY(cudaStreamSynchronize(st));
    L->nnz = sc.host[0].nnz;
    L->first_empty_row = sc.host[0].first_empty;
    L->max_row_len = sc.host[0].max_len;
    L->min_row_len = sc.host[0].min_len;
    RADIAL_CUDA_TRY(cudaMallocAsync(&L->col_idx, sizeof(uint32_t) * std::max<uint64_t>(L->nnz, 1), st));
    return fill(BlockKeep{p}, L->R, L->R, L->row_ptr, L->col_idx, 0, st);
}

// CSC, chunk unions and LPT orders for a CSR already on the device.  One host sync
// (union sizes) plus a final one so the handle is complete when this returns.
int build_worklists(radial_layout* L, cudaStream_t st) {
    Scratch sc(st);
    const uint32_t R = L->R;
    const bool attn = (L->B == 64 || L->B == 128);
    L->G = attn ? 256 / L->B : 1;
    L->C = attn ? (R + L->G - 1) / L->G : 0;
    const uint32_t C = L->C;
    L->C4 = L->B == 128 ? (R + 3) / 4 : 0;
    const uint32_t C4 = L->C4;
    RADIAL_CUDA_TRY(cudaMallocAsync(&sc.counts, sizeof(uint32_t) * (std::max<uint32_t>(R, 1) + std::max<uint32_t>(C, 1) +
                                                                     std::max<uint32_t>(C4, 1)), st));
    RADIAL_CUDA_TRY(cudaMallocAsync(&sc.stats, 4 * sizeof(ScanStats), st));
    RADIAL_CUDA_TRY(cudaMallocAsync(&L->col_ptr, sizeof(uint64_t) * (static_cast<size_t>(R) + 1), st));
    RADIAL_CUDA_TRY(cudaMallocAsync(&L->row_idx, sizeof(uint32_t) * std::max<uint64_t>(L->nnz, 1), st));
    int rc;
    // CSC: its nnz equals the CSR's, so no sync is needed before the fill
    const CsrTranspose tr{L->row_ptr, L->col_idx};
    if ((rc = count_and_scan(tr, R, R, sc.counts, L->col_ptr, sc.stats + 1, st))) return rc;
    if ((rc = fill(tr, R, R, L->col_ptr, L->row_idx, 0, st))) return rc;
    if (!attn) {
        RADIAL_CUDA_TRY(cudaStreamSynchronize(st));
        return RADIAL_OK;  // attention kernels not instantiated for this block size
    }
    RADIAL_CUDA_TRY(cudaMallocAsync(&L->uptr, sizeof(uint64_t) * (static_cast<size_t>(C) + 1), st));
    const ChunkUnion uq{L->row_ptr, L->col_idx, R, L->G};
    if ((rc = count_and_scan(uq, C, R, sc.counts + R, L->uptr, sc.stats + 2, st))) return rc;
    if ((rc = lpt_order(L->row_ptr, R, st, &L->rorder))) return rc;
    if ((rc = lpt_order(L->col_ptr, R, st, &L->corder))) return rc;
    if ((rc = lpt_order(L->uptr, C, st, &L->uorder))) return rc;
    const ChunkUnion uq4{L->row_ptr, L->col_idx, R, 4};
    if (C4) {
        RADIAL_CUDA_TRY(cudaMallocAsync(&L->u4ptr, sizeof(uint64_t) * (static_cast<size_t>(C4) + 1), st));
        if ((rc = count_and_scan(uq4, C4, R, sc.counts + R + C, L->u4ptr, sc.stats + 3, st))) return rc;
        if ((rc = lpt_order(L->u4ptr, C4, st, &L->u4order))) return rc;
    }
    // slots 1 (CSC), 2 and 3 (unions); slot 0 belongs to build_layout_device
    RADIAL_CUDA_TRY(cudaMemcpyAsync(sc.host + 1, sc.stats + 1, (C4 ? 3 : 2) * sizeof(ScanStats), cudaMemcpyDeviceToHost, st));
    RADIAL_CUDA_TRY(cudaStreamSynchronize(st));
    if (sc.host[1].nnz != L->nnz) return fail(RADIAL_ERR_INVALID, "layout transpose size mismatch");
    const uint64_t un = sc.host[2].nnz;
    RADIAL_CUDA_TRY(cudaMallocAsync(&L->uidx, sizeof(uint32_t) * std::max<uint64_t>(un, 1), st));
    RADIAL_CUDA_TRY(cudaMallocAsync(&L->uidx_asc, sizeof(uint32_t) * std::max<uint64_t>(un, 1), st));
    // ascending lists (token-exact forward) filled directly, then the paired copy for the
    // block-layout forward
    if ((rc = fill(uq, C, R, L->uptr, L->uidx_asc, 1, st))) return rc;
    if (C4) {
        RADIAL_CUDA_TRY(cudaMallocAsync(&L->u4idx, sizeof(uint32_t) * std::max<uint64_t>(sc.host[3].nnz, 1), st));
        if ((rc = fill(uq4, C4, R, L->u4ptr, L->u4idx, 1, st))) return rc;
    }
    if (C && un) {
        uint32_t* match = nullptr;
        RADIAL_CUDA_TRY(cudaMallocAsync(&match, sizeof(uint32_t) * un, st));
        const uint32_t warps_per_cta = 8;
        pair_solo_entries<<<(C + warps_per_cta - 1) / warps_per_cta, 32 * warps_per_cta, 0, st>>>(
            L->uptr, C, L->G / 2, L->uidx_asc, L->uidx, match);
        RADIAL_CUDA_TRY(cudaGetLastError());
        count_launches(1);
        RADIAL_CUDA_TRY(cudaFreeAsync(match, st));
        if (L->from_pattern) {
            const MaskParams mp{L->f, L->s, L->B, static_cast<uint64_t>(L->f) * L->s, L->kind, L->sink, L->tw, L->sw};
            RADIAL_CUDA_TRY(cudaMallocAsync(&L->ufull, un, st));
            token_full_flags<<<(C + warps_per_cta - 1) / warps_per_cta, 32 * warps_per_cta, 0, st>>>(
                mp, L->uptr, C, L->G, RADIAL_TOK_PAIRED ? L->uidx : L->uidx_asc, L->ufull);
            RADIAL_CUDA_TRY(cudaGetLastError());
            count_launches(1);
        }
    }
    RADIAL_CUDA_TRY(cudaStreamSynchronize(st));
    return RADIAL_OK;
}

}  // namespace radial_detail
