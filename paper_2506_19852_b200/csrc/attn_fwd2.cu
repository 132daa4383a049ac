// attn_fwd2.cu -- K2 / K4 on CTA pairs (tcgen05 cta_group::2), head_dim 128, block 128.
//
// Same computation as attn_fwd.cu (radial::masked_attention(inst, layout), reference
// attention.hpp:229-270, and dense_attention, :141-163), with every MMA issued for a pair
// of SMs: M = 256 query rows, 128 from each CTA of a 2-CTA cluster.  The pair shares each
// K / V tile, and each CTA holds and loads only HALF of it (the B operand of a pair MMA is
// split along N): K_j rows [64 r, 64 r + 64) (N = keys for S = Q K^T) and V_j columns
// [64 r, 64 r + 64) (N = head dims for O += P V), r = CTA rank.  So every SM receives half
// the K / V bytes of the one-CTA kernel and its shared-memory port carries half the B-operand
// traffic.  (Measured on the one-CTA kernel: delivering half of every tile raises the
// power-capped clock from ~1580 to ~1870 MHz.)
//
// Work item = (head, chunk of 512 query rows = 4 blocks) per cluster.  Pair tile A = blocks
// 4c (CTA 0) and 4c + 1 (CTA 1), pair tile B = 4c + 2 / 4c + 3.  The KV loop runs over the
// union of the four blocks' lists (entry = J | mask << 28, bit g = block 4c + g keeps J); a
// pair tile computes S for J when either of its blocks keeps it, and the rows of a block
// that does not keep J are masked (their share of that MMA is the price of the pairing: the
// union of two adjacent blocks' lists is 5-16% longer than their mean length).
//
// Roles (384 threads per CTA, one CTA per SM):
//   warp 0      TMA producer (both CTAs): own Q tiles, own halves of K_j / V_j, completion
//               counted on the LEADER's (rank 0) barriers
//   warp 1      MMA issuer (leader only): S_T = Q_T K^T, O_T += P_T V (TS, P from TMEM)
//   warp 2      TMEM allocator (cta_group::2, both CTAs)
//   warps 4-11  softmax + epilogue, as in attn_fwd.cu, for this CTA's 128 rows of each tile;
//               P-ready arrivals go to the leader's barrier (remote arrive from rank 1)
// MMA completions are committed to the barriers at the same offset in both CTAs (multicast).
#include <cmath>
#include <type_traits>

#include "radial_internal.h"
#include "sm100.cuh"

#ifndef RADIAL_FWD2_SLOTS
#define RADIAL_FWD2_SLOTS 9
#endif

using namespace radial_sm100;

namespace {

constexpr int kThreads = 384;
constexpr uint32_t kTmem = 0;
constexpr int D = 128, BK = 128;
constexpr int kSlots = RADIAL_FWD2_SLOTS;  // half-tile ring (K_j half, V_j half, ...): 16 KB each
constexpr int kPParts = 2;
constexpr float kRescaleThreshold = 8.0f;
constexpr int kMaxDst = 8;

constexpr int kQBytes = 128 * D * 2;            // one 128-row Q tile (32 KB)
constexpr int kQAtomBytes = 128 * 128;          // 64 d-columns of it
constexpr int kHalfBytes = 16384;               // half a K or V tile
constexpr int kKHalfAtomBytes = 64 * 128;       // 64 keys x 64 d-columns (K half, 2 atoms)
constexpr int kSmemQ = 0;
constexpr int kSmemKV = 2 * kQBytes;
constexpr int kSmemBar = kSmemKV + kSlots * kHalfBytes;
constexpr int kNumBars = 1 + 2 * kSlots + 2 + 2 * kPParts + 2;
constexpr int kSmemBytes = kSmemBar + kNumBars * 8 + 16;
constexpr int kSmemAlloc = kSmemBytes + 1024;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO0 = 256, kColO1 = 384;
constexpr uint32_t kIdescS = idesc_bf16(256, BK, 0, 0);  // pair M = 256, N = 128 keys
constexpr uint32_t kIdescO = idesc_bf16(256, D, 0, 1);   // pair M = 256, N = 128 dims, V MN-major

struct Fwd2Params {
    __nv_bfloat16* o;
    float* lse;
    __nv_bfloat16* dst[kMaxDst];
    uint32_t n_dst, head_base, heads_full;
    const uint64_t* uptr;   // 512-row chunk unions
    const uint32_t* uidx;
    const uint32_t* order;
    uint64_t n;
    uint32_t heads, R, C;   // C = 512-row chunks
    float scale_log2;
    int dense;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    radial_attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                                const __grid_constant__ CUtensorMap tm_v, const Fwd2Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBar);
    uint64_t* bar_q = bars;                          // leader: both CTAs' Q tiles landed
    uint64_t* bar_full = bars + 1;                   // leader: both halves of a ring slot landed
    uint64_t* bar_empty = bar_full + kSlots;         // both: slot free (pair MMAs done)
    uint64_t* bar_sfull = bar_empty + kSlots;        // both: S_T computed
    uint64_t* bar_pready = bar_sfull + 2;            // leader: P_T part h published by 8 warps
    uint64_t* bar_ofull = bar_pready + 2 * kPParts;  // both: O_T final
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_ofull + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;

    const uint32_t item = blockIdx.x >> 1;
    const uint32_t head = item / p.C;
    const uint32_t chunk = p.order ? p.order[item % p.C] : item % p.C;
    const uint64_t row0 = static_cast<uint64_t>(chunk) * 512;
    uint64_t ebase = 0;
    uint32_t L;
    uint32_t dense_mask = 0;
    if (p.dense) {
        L = p.R;
        for (int g = 0; g < 4; ++g)
            if (chunk * 4 + g < p.R) dense_mask |= 1u << g;
    } else {
        ebase = p.uptr[chunk];
        L = static_cast<uint32_t>(p.uptr[chunk + 1] - ebase);
    }
    auto entry = [&](uint32_t j) -> uint32_t {
        return p.dense ? (j | (dense_mask << 28)) : __ldg(p.uidx + ebase + j);
    };

    if (warp == 0 && lane == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&bar_sfull[t], 1);
            for (int h = 0; h < kPParts; ++h) mbar_init(&bar_pready[kPParts * t + h], 8);  // 4 warps x 2 CTAs
            mbar_init(&bar_ofull[t], 1);
        }
        fence_barrier_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
    }
    if (warp == 2) tmem_alloc2(tmem_slot, 512);  // both CTAs, same warp: the pair's 2 x 512 columns
    tc_fence_before();
    cluster_sync();  // barriers initialised and TMEM allocated in both CTAs before any remote use
    tc_fence_after();

    if (warp < 4) {
        regs_dec<72>();
        if (warp == 0) {
            // ------------------------------------------------------------ producer (both CTAs)
            if (lane == 0) {
                const uint32_t q_bar = mapa_shared(smem_u32(bar_q), 0);
                if (leader) mbar_arrive_expect_tx(bar_q, 4 * kQBytes);  // two tiles in each CTA
                for (int t = 0; t < 2; ++t)
                    for (int a = 0; a < 2; ++a)
                        tma_load_3d_2sm(smem + kSmemQ + t * kQBytes + a * kQAtomBytes, &tm_q, q_bar, a * 64,
                                        static_cast<int32_t>(row0 + 256 * t + 128 * rank), head);
                for (uint32_t t = 0; t < 2 * L; ++t) {
                    const int32_t J = static_cast<int32_t>(entry(t >> 1) & 0x0FFFFFFFu);
                    const uint32_t slot = t % kSlots;
                    mbar_wait(&bar_empty[slot], ((t / kSlots) & 1) ^ 1);
                    if (leader) mbar_arrive_expect_tx(&bar_full[slot], 2 * kHalfBytes);
                    const uint32_t fb = mapa_shared(smem_u32(&bar_full[slot]), 0);
                    uint8_t* dst = smem + kSmemKV + slot * kHalfBytes;
                    if ((t & 1) == 0) {
                        // K_j rows [64 rank, 64 rank + 64): the pair MMA's B operand, N = keys
                        for (int a = 0; a < 2; ++a)
                            tma_load_3d_2sm(dst + a * kKHalfAtomBytes, &tm_k, fb, a * 64, J * BK + 64 * rank, head);
                    } else {
                        // V_j columns [64 rank, 64 rank + 64), all 128 keys: B operand, N = dims
                        tma_load_3d_2sm(dst, &tm_v, fb, 64 * rank, J * BK, head);
                    }
                }
            }
        } else if (warp == 1 && leader) {
            // ------------------------------------------------------------ MMA issuer (leader)
            mbar_wait(bar_q, 0);
            tc_fence_after();
            const uint64_t dq = sdesc_sw128(smem_u32(smem + kSmemQ), 16, 1024);
            const uint64_t dk = sdesc_sw128(smem_u32(smem + kSmemKV), 16, 1024);
            const uint64_t dv = sdesc_sw128(smem_u32(smem + kSmemKV), kHalfBytes, 1024);
            bool pend0 = false, pend1 = false;
            uint32_t acc0 = 0, acc1 = 0, pphase0 = 0, pphase1 = 0;
            uint32_t e_next = L > 0 ? __shfl_sync(0xffffffffu, entry(0), 0) : 0u;
            auto step = [&](uint32_t j, auto PC) {
                constexpr int PH = decltype(PC)::value;               // == j % kSlots
                constexpr int KSL = (2 * PH) % kSlots;                 // slot of K_j
                constexpr int VSL = (2 * PH + kSlots - 1) % kSlots;   // slot of V_{j-1}
                uint32_t tf0 = 0, tf1 = 0;
                if (j < L) {
                    const uint32_t m = e_next >> 28;
                    if (j + 1 < L) e_next = __shfl_sync(0xffffffffu, entry(j + 1), 0);
                    tf0 = m & 3u;
                    tf1 = (m >> 2) & 3u;
                }
                if (j > 0) mbar_wait(&bar_full[VSL], ((2 * j - 1) / kSlots) & 1);
                tc_fence_after();
                auto pv = [&](auto TC, uint32_t& acc, uint32_t& pphase) {
                    constexpr int T = decltype(TC)::value;
                    constexpr uint32_t p_col = T ? kColS1 : kColS0;
                    constexpr uint32_t o_col = T ? kColO1 : kColO0;
                    static_for<kPParts>([&](auto HC) {
                        constexpr int h = decltype(HC)::value;
                        constexpr int kk0 = h * 4;  // four 16-key K-steps per part
                        mbar_wait(&bar_pready[kPParts * T + h], pphase);
                        tc_fence_after();
                        mma2_ts_x4<((VSL * kHalfBytes + kk0 * 16 * 128) >> 4), 128>(
                            kTmem + o_col, kTmem + p_col + kk0 * 8, dv, kIdescO, (acc | kk0) ? 1u : 0u);
                    });
                    pphase ^= 1;
                    acc = 1;
                };
                auto qk = [&](auto TC) {
                    constexpr int T = decltype(TC)::value;
                    constexpr uint32_t s_col = T ? kColS1 : kColS0;
                    static_for<2>([&](auto AC) {
                        constexpr int at = decltype(AC)::value;
                        mma2_ss_x4<((T * kQBytes + at * kQAtomBytes) >> 4),
                                   ((KSL * kHalfBytes + at * kKHalfAtomBytes) >> 4)>(kTmem + s_col, dq, dk, kIdescS,
                                                                                     at ? 1u : 0u);
                    });
                    mma2_commit_mc(&bar_sfull[T]);
                };
                if (pend0) {
                    pv(std::integral_constant<int, 0>{}, acc0, pphase0);
                    pend0 = false;
                }
                if (j < L) {
                    mbar_wait(&bar_full[KSL], ((2 * j) / kSlots) & 1);
                    tc_fence_after();
                }
                if (tf0) {
                    qk(std::integral_constant<int, 0>{});
                    pend0 = true;
                }
                if (pend1) {
                    pv(std::integral_constant<int, 1>{}, acc1, pphase1);
                    pend1 = false;
                }
                if (j > 0) mma2_commit_mc(&bar_empty[VSL]);
                if (tf1) {
                    qk(std::integral_constant<int, 1>{});
                    pend1 = true;
                }
                if (j < L) mma2_commit_mc(&bar_empty[KSL]);
            };
            for (uint32_t j = 0; j <= L; j += kSlots) {
                static_for<kSlots>([&](auto PC) {
                    if (j + decltype(PC)::value <= L) step(j + decltype(PC)::value, PC);
                });
            }
            mma2_commit_mc(&bar_ofull[0]);
            mma2_commit_mc(&bar_ofull[1]);
        }
    } else {
        regs_inc<216>();
        // ------------------------------------------------------------ softmax (both CTAs)
        const int t = (warp - 4) >> 2;
        const int r = ((warp & 3) << 5) + lane;
        const uint32_t lane_addr = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t s_addr = kTmem + lane_addr + (t ? kColS1 : kColS0);
        const uint32_t o_addr = kTmem + lane_addr + (t ? kColO1 : kColO0);
        const int my_bit = 2 * t + static_cast<int>(rank);
        const uint64_t grow = row0 + 256 * t + 128 * rank + r;
        uint32_t pready_addr[kPParts];
        for (int h = 0; h < kPParts; ++h) pready_addr[h] = mapa_shared(smem_u32(&bar_pready[kPParts * t + h]), 0);
        const float sl2 = p.scale_log2;
        float m = -INFINITY, l = 0.f;
        uint32_t sphase = 0;
        uint32_t e_next = L > 0 ? entry(0) : 0u;
        for (uint32_t j = 0; j < L; ++j) {
            const uint32_t e = e_next;
            if (j + 1 < L) e_next = entry(j + 1);
            const uint32_t mask = e >> 28;
            if (((mask >> (2 * t)) & 3u) == 0) continue;  // the pair tile skips J
            const uint32_t J = e & 0x0FFFFFFFu;
            mbar_wait(&bar_sfull[t], sphase);
            sphase ^= 1;
            tc_fence_after();
            float s[BK];
            {
                uint32_t u[64];
                tmem_ld64(s_addr, u);
#pragma unroll
                for (int x = 0; x < 64; ++x) s[x] = __uint_as_float(u[x]);
            }
            tmem_wait_ld();
            float mh[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) mh[x] = s[x];
            {
                uint32_t u[64];
                tmem_ld64(s_addr + 64, u);
#pragma unroll
                for (int x = 0; x < 64; ++x) s[64 + x] = __uint_as_float(u[x]);
            }
#pragma unroll
            for (int c = 8; c < BK / 2; c += 8)
#pragma unroll
                for (int x = 0; x < 8; ++x) mh[x] = fmaxf(mh[x], s[c + x]);
            tmem_wait_ld();
            const bool active = (mask >> my_bit) & 1;
            const uint64_t kv0 = static_cast<uint64_t>(J) * BK;
            const int valid = (kv0 + BK <= p.n) ? BK : static_cast<int>(p.n - kv0);
            const bool full = active && valid == BK;
            if (!full) {
#pragma unroll
                for (int c = 0; c < BK; ++c) s[c] = (active && c < valid) ? s[c] : -INFINITY;
            }
            float mm[8];
            if (full) {
#pragma unroll
                for (int x = 0; x < 8; ++x) mm[x] = mh[x];
            } else {
#pragma unroll
                for (int x = 0; x < 8; ++x) mm[x] = s[x];
#pragma unroll
                for (int c = 8; c < BK / 2; c += 8)
#pragma unroll
                    for (int x = 0; x < 8; ++x) mm[x] = fmaxf(mm[x], s[c + x]);
            }
#pragma unroll
            for (int c = BK / 2; c < BK; c += 8)
#pragma unroll
                for (int x = 0; x < 8; ++x) mm[x] = fmaxf(mm[x], s[c + x]);
            const float mx = fmaxf(fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])),
                                   fmaxf(fmaxf(mm[4], mm[5]), fmaxf(mm[6], mm[7])));
            const float m_cand = mx * sl2;
            const bool need = active && (m == -INFINITY || m_cand > m + kRescaleThreshold);
            const bool rescale = need && m != -INFINITY;
            if (__any_sync(0xffffffffu, rescale)) {
                const float alpha = rescale ? ex2(m - m_cand) : 1.f;
#pragma unroll
                for (int c = 0; c < D; c += 32) {
                    uint32_t u[32];
                    tmem_ld32(o_addr + c, u);
                    tmem_wait_ld();
#pragma unroll
                    for (int x = 0; x < 32; ++x) u[x] = __float_as_uint(__uint_as_float(u[x]) * alpha);
                    tmem_st32(o_addr + c, u);
                }
                if (rescale) l *= alpha;
            }
            if (need) m = m_cand;
            const float mb = (m == -INFINITY) ? 0.f : m;
            float2 r2a = make_float2(0.f, 0.f), r2b = make_float2(0.f, 0.f);
            const float2 sl = make_float2(sl2, sl2), nm = make_float2(-mb, -mb);
#pragma unroll
            for (int h = 0; h < kPParts; ++h) {
                constexpr int CP = BK / kPParts;
                uint32_t pk[CP / 2];
#pragma unroll
                for (int c = h * CP; c < (h + 1) * CP; c += 2) {
                    if (c > h * CP && (c - h * CP) % 32 == 0)
                        tmem_st16(s_addr + h * (CP / 2) + (c - h * CP) / 2 - 16, pk + (c - h * CP) / 2 - 16);
                    const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), sl, nm);
                    float2 pr;
                    pr.x = ex2(x.x);
                    pr.y = ex2(x.y);
                    if ((c >> 1) & 1)
                        r2b = __fadd2_rn(r2b, pr);
                    else
                        r2a = __fadd2_rn(r2a, pr);
                    pk[(c - h * CP) / 2] = pack_bf16(pr.x, pr.y);
                }
                tmem_st16(s_addr + h * (CP / 2) + CP / 2 - 16, pk + CP / 2 - 16);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (leader)
                        mbar_arrive(&bar_pready[kPParts * t + h]);
                    else
                        mbar_arrive_cluster(pready_addr[h]);
                }
            }
            l += (r2a.x + r2a.y) + (r2b.x + r2b.y);
        }
        // ------------------------------------------------------------ epilogue
        mbar_wait(&bar_ofull[t], 0);
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        __nv_bfloat16* orow = p.o + (static_cast<uint64_t>(head) * p.n + grow) * D;
        const uint64_t frow = (static_cast<uint64_t>(p.head_base + head) * p.n + grow) * D;
#pragma unroll
        for (int c = 0; c < D; c += 32) {
            uint32_t u[32];
            tmem_ld32(o_addr + c, u);
            tmem_wait_ld();
            uint32_t w[16];
#pragma unroll
            for (int x = 0; x < 16; ++x)
                w[x] = pack_bf16(__uint_as_float(u[2 * x]) * inv, __uint_as_float(u[2 * x + 1]) * inv);
            if (grow < p.n) {
                if (p.n_dst == 0) {
                    uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
                    for (int x = 0; x < 4; ++x) dst[x] = make_uint4(w[4 * x], w[4 * x + 1], w[4 * x + 2], w[4 * x + 3]);
                } else {
                    for (uint32_t rr = 0; rr < p.n_dst; ++rr) {
                        uint4* dst = reinterpret_cast<uint4*>(p.dst[rr] + frow + c);
#pragma unroll
                        for (int x = 0; x < 4; ++x)
                            dst[x] = make_uint4(w[4 * x], w[4 * x + 1], w[4 * x + 2], w[4 * x + 3]);
                    }
                }
            }
        }
        if (p.lse && grow < p.n)
            p.lse[static_cast<uint64_t>(head) * p.n + grow] = l > 0.f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
    }
    tc_fence_before();
    cluster_sync();  // both CTAs done with TMEM and every remote barrier before teardown
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc2(*tmem_slot, 512);
    }
}

}  // namespace

namespace radial_detail {

int make_tmap_bf16_3d(CUtensorMap* m, const void* base, uint64_t n, uint32_t D, uint32_t heads, uint32_t box_rows);

// K2 / K4 on CTA pairs; L == nullptr runs the dense comparator.
int launch_fwd_pair(const void* q, const void* k, const void* v, void* o, float* lse, uint32_t heads, uint64_t n,
                    float scale, const radial_layout* L, cudaStream_t st, const FwdScatter* sc) {
    const uint64_t R64 = (n + BK - 1) / BK;
    const uint32_t R = static_cast<uint32_t>(R64);
    CUtensorMap tq, tk, tv;
    int rc;
    if ((rc = make_tmap_bf16_3d(&tq, q, n, D, heads, 128))) return rc;
    if ((rc = make_tmap_bf16_3d(&tk, k, n, D, heads, 64))) return rc;   // half a K tile: 64 keys
    if ((rc = make_tmap_bf16_3d(&tv, v, n, D, heads, 128))) return rc;  // half a V tile: 64 dims x 128 keys
    Fwd2Params p{};
    p.o = static_cast<__nv_bfloat16*>(o);
    p.lse = lse;
    if (sc) {
        p.n_dst = sc->n_dst;
        p.head_base = sc->head_base;
        p.heads_full = sc->heads_full;
        for (uint32_t r = 0; r < sc->n_dst; ++r) p.dst[r] = static_cast<__nv_bfloat16*>(sc->dst[r]);
    }
    p.n = n;
    p.heads = heads;
    p.R = R;
    p.C = (R + 3) / 4;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.dense = L == nullptr;
    if (L) {
        if (!L->u4ptr) return fail(RADIAL_ERR_INVALID, "masked_attention: layout has no 512-row work lists");
        p.uptr = L->u4ptr;
        p.uidx = L->u4idx;
        p.order = L->u4order;
    }
    auto kern = radial_attn_fwd_pair_kernel;
    RADIAL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc));
    const uint64_t items = static_cast<uint64_t>(p.C) * heads;
    if (items == 0) return RADIAL_OK;
    if (2 * items > 0x7fffffffull) return fail(RADIAL_ERR_INVALID, "too many work items");
    kern<<<static_cast<unsigned>(2 * items), kThreads, kSmemAlloc, st>>>(tq, tk, tv, p);
    RADIAL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    note_use(L, st);
    return RADIAL_OK;
}

}  // namespace radial_detail
