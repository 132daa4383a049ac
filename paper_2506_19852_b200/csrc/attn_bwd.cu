// attn_bwd.cu -- K3: backward of the block-sparse radial forward over the same
// layout (no reference exists: the paper's LoRA length-extension path is out
// of the reference's scope).  Gradients of attention.hpp:229-270:
//
//   P  = exp(S - lse),  S = scale * Q K^T on kept B x B blocks
//   dV = P^T dO          dP = dO V^T          D = rowsum(dO o O)
//   dS = P o (dP - D)    dQ = scale * dS K    dK = scale * dS^T Q
//
// Deterministic, no atomics, three launches:
//   bwd_prep    D and lse*log2(e) per query row, padded to whole 128-row blocks
//               (+inf lse / 0 D beyond n, so padded rows contribute exactly 0)
//   bwd_dq      one CTA per (head, query block I) over its CSR row: S = Q K^T (Q resident in
//               TMEM), dP = dO V^T, dS (bf16) into its own TMEM columns, dQ += dS K
//   bwd_dkdv    one CTA per (head, KV block J) over its CSC column: S^T, dP^T, then
//               dV += P^T dO and dK += dS^T Q with P^T / dS^T in the consumed dP^T columns
// Every MMA is 128 x 128 x 16 (128 x 64 MMAs run at 61% of the tensor rate); the elementwise
// warpgroups split the 128 columns of each block and release S / dP as soon as they have
// loaded them, so the tensor core computes the next block while they work.
// Block size 128 only (the layouts of the BASELINE backward configs).
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "radial_internal.h"
#include "sm100.cuh"

// setmaxnreg split: producer/MMA warpgroup vs elementwise warpgroups (384 threads x 168 =
// 128 x LO + 256 x HI must hold)
#ifndef RADIAL_REGS_LO
#define RADIAL_REGS_LO 104
#define RADIAL_REGS_HI 200
#endif

using namespace radial_sm100;

namespace radial_detail {
int make_tmap_bf16_3d(CUtensorMap* m, const void* base, uint64_t n, uint32_t D, uint32_t heads,
                      uint32_t box_rows);
}

#ifdef RADIAL_TRACE
__device__ unsigned long long* g_btrace = nullptr;
#define BTRACE(ev, j)                                                                         \
    do {                                                                                      \
        if (g_btrace && blockIdx.x < 4 && (j) < 64)                                           \
            g_btrace[(blockIdx.x * 64 + (j)) * 16 + (ev)] = clock64();                       \
    } while (0)
#else
#define BTRACE(ev, j) \
    do {              \
    } while (0)
#endif

#ifndef RADIAL_BWD_DQ_POLY
#define RADIAL_BWD_DQ_POLY 1  // column pairs per 8 whose exp2 runs on the FMA pipe in the dQ kernel (measured best)
#endif
#ifndef RADIAL_BWD_DQ_SPLIT_S
#define RADIAL_BWD_DQ_SPLIT_S 0  // dQ kernel: load S in two 32-column halves, the second under the first's exps
#endif
#ifndef RADIAL_BWD_DQ_EARLY_DP
#define RADIAL_BWD_DQ_EARLY_DP 48  // dQ kernel: column index at which dP is loaded under the exponentials (0 = after)
#endif
#ifndef RADIAL_BWD_DKDV_EARLY_DP
#define RADIAL_BWD_DKDV_EARLY_DP 0  // dK/dV kernel: column at which dP^T is loaded under the exponentials
#endif
#ifndef RADIAL_BWD_DKDV_POLY
#define RADIAL_BWD_DKDV_POLY 0  // column quads per 8 whose exp2 runs on the FMA pipe in the dK/dV kernel
#endif
#ifndef RADIAL_BWD_L2HINTS
#define RADIAL_BWD_L2HINTS 0  // L2 eviction hints (tiles read once evict-first, re-read tiles evict-last): measured neutral, off
#endif
#if RADIAL_BWD_L2HINTS
#define BWD_LOAD(dst, map, bar, c0, c1, c2, pol) tma_load_3d_hint(dst, map, bar, c0, c1, c2, pol)
#else
#define BWD_LOAD(dst, map, bar, c0, c1, c2, pol) tma_load_3d(dst, map, bar, c0, c1, c2)
#endif

namespace {

constexpr int kThreads = 384;   // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warps 4-11 elementwise
constexpr int kBlk = 128;       // layout block = rows per resident tile
constexpr uint32_t kTmem = 0;   // whole-SM TMEM allocation starts at column 0
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
    const __nv_bfloat16* q;     // dQ kernel: Q and dO rows go straight to TMEM
    const __nv_bfloat16* dout;
    __nv_bfloat16* dq;
    __nv_bfloat16* dk;
    __nv_bfloat16* dv;
    const float* lse2;   // [H][Rpad] lse * log2(e), +inf padded
    const float* dvec;   // [H][Rpad] D, 0 padded
    const uint64_t* ptr;  // CSR (dq) or CSC (dkdv)
    const uint32_t* idx;
    const uint32_t* order;
    uint64_t n, rpad;
    uint32_t heads, R;
    float scale, scale_log2;
};

// ---------------------------------------------------------------- preprocess
__global__ void bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                const float* __restrict__ lse, float* __restrict__ lse2,
                                float* __restrict__ dvec, uint64_t n, uint64_t rpad, uint32_t D,
                                uint32_t heads) {
    // one warp per padded row
    const uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= static_cast<uint64_t>(heads) * rpad) return;
    const uint64_t h = w / rpad, i = w % rpad;
    float acc = 0.f;
    if (i < n) {
        const __nv_bfloat16* orow = o + (h * n + i) * D;
        const __nv_bfloat16* drow = dout + (h * n + i) * D;
        for (uint32_t c = lane * 2; c < D; c += 64) {
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(orow + c));
            const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(drow + c));
            acc += a.x * b.x + a.y * b.y;
        }
    }
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
        dvec[w] = i < n ? acc : 0.f;
        lse2[w] = i < n ? lse[h * n + i] * kLog2e : INFINITY;
    }
}

template <int D>
struct BwdCfg {
    static constexpr int kAtoms = D / 64;
    static constexpr int kAtomBytes = kBlk * 128;      // 128 rows x 128 B
    static constexpr int kTileBytes = kBlk * D * 2;    // one 128-row bf16 tile
    static constexpr uint32_t kIdAcc = idesc_bf16(128, D, 0, 1);   // 128 x D x 16, B MN-major
    static constexpr uint32_t kIdAcc128 = idesc_bf16(128, kBlk, 0, 0);  // 128 x 128 x 16, K-major both
};

// Base descriptors: an MMA's descriptor = base + (byte offset >> 4); the 14-bit start
// address field never carries (all offsets stay inside the 227 KB of shared memory).
// Keeping every offset a compile-time constant keeps the tcgen05 operands uniform.
__device__ __forceinline__ uint64_t kbase(uint32_t smem_addr) { return sdesc_sw128(smem_addr, 16, 1024); }
__device__ __forceinline__ uint64_t mnbase(uint32_t smem_addr) { return sdesc_sw128(smem_addr, kBlk * 128, 1024); }
__host__ __device__ constexpr uint32_t koff(int kk, int row0) {
    return static_cast<uint32_t>(((kk >> 2) * (kBlk * 128) + row0 * 128 + (kk & 3) * 32) >> 4);
}
__host__ __device__ constexpr uint32_t mnoff(int row0) { return static_cast<uint32_t>((row0 * 128) >> 4); }

// ============================================================================ dQ
// CTA per (head, query block I) over its CSR row.  Q is resident in TMEM (A operand of
// S = Q K^T), dO in shared memory (A operand of dP = dO V^T); K_j / V_j stream through
// 3- / 2-stage rings.  Every MMA is 128 x 128 x 16.
// TMEM: S [0,128) dP [128,256) dQ [256,256+D) dS [256+D, 320+D) Q [320+D, 320+D+D/2).
// Warpgroup g owns key columns [64g, 64g+64).  The warpgroups release S and dP as soon
// as they have loaded them, so the tensor core computes S(j+1) and dP(j+1) while they
// turn block j into dS(j); dS has its own columns, freed when dQ(j) has consumed it.
// MMA issue order per block j:  S(j), dP(j), dQ(j-1).
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    radial_attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                              const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                              const BwdParams p) {
    using Cfg = BwdCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int T = Cfg::kTileBytes;
    constexpr int kKS = 4, kVS = 2;  // ring depths (K is held from S(j) to dQ(j): deeper)
    constexpr int kUnroll = 4;       // lcm of the ring depths: slots are compile-time constants
    // [dO | K0..K3 | V0 V1 | barriers]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (1 + kKS + kVS) * T);
    uint64_t* bar_q = bars;                   // Q rows stored into TMEM (8 warp arrivals)
    uint64_t* bar_do = bars + 1;              // dO landed
    uint64_t* bar_kfull = bars + 2;           // [kKS]
    uint64_t* bar_kempty = bar_kfull + kKS;   // [kKS] K_j free (dQ(j) done)
    uint64_t* bar_vfull = bar_kempty + kKS;   // [kVS]
    uint64_t* bar_vempty = bar_vfull + kVS;   // [kVS] V_j free (dP(j) done)
    uint64_t* bar_s = bar_vempty + kVS;       // S(j) computed
    uint64_t* bar_dp = bar_s + 1;             // dP(j) computed
    uint64_t* bar_sfree = bar_s + 2;          // S(j) loaded by the warpgroups (8)
    uint64_t* bar_dpfree = bar_s + 3;         // dP(j) loaded (8)
    uint64_t* bar_ds = bar_s + 4;             // dS(j) in TMEM (8)
    uint64_t* bar_dsfree = bar_s + 5;         // dQ(j) done: dS columns free
    uint64_t* bar_acc = bar_s + 6;            // dQ final
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_s + 7);
    constexpr uint32_t kColS = 0, kColDP = 128, kColDQ = 256, kColDS = 256 + D, kColQ = 320 + D;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t head = blockIdx.x / p.R;
    const uint32_t I = p.order[blockIdx.x % p.R];
    const uint64_t e0 = p.ptr[I];
    const uint32_t L = static_cast<uint32_t>(p.ptr[I + 1] - e0);

    if (warp == 0 && lane == 0) {
        mbar_init(bar_q, 8);
        mbar_init(bar_do, 1);
        for (int i = 0; i < kKS; ++i) {
            mbar_init(&bar_kfull[i], 1);
            mbar_init(&bar_kempty[i], 1);
        }
        for (int i = 0; i < kVS; ++i) {
            mbar_init(&bar_vfull[i], 1);
            mbar_init(&bar_vempty[i], 1);
        }
        mbar_init(bar_s, 1);
        mbar_init(bar_dp, 1);
        mbar_init(bar_sfree, 8);
        mbar_init(bar_dpfree, 8);
        mbar_init(bar_ds, 8);
        mbar_init(bar_dsfree, 1);
        mbar_init(bar_acc, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();  // all 512 columns allocated: the base is column 0 by construction

    if (warp < 4) {
        regs_dec<RADIAL_REGS_LO>();
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------ producer
            // dO_I is read once (evict-first); K_j / V_j are re-read by every query block of
            // their CSC column (evict-last)
            [[maybe_unused]] const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
            mbar_arrive_expect_tx(bar_do, T);
            for (int a = 0; a < Cfg::kAtoms; ++a)
                BWD_LOAD(smem + a * Cfg::kAtomBytes, &tm_do, bar_do, a * 64, I * kBlk, head, pol_first);
            for (uint32_t j = 0; j < L; ++j) {
                const int32_t J = static_cast<int32_t>(__ldg(p.idx + e0 + j));
                const int ks = j % kKS, vs = j % kVS;
                mbar_wait(&bar_kempty[ks], ((j / kKS) & 1) ^ 1);
                mbar_arrive_expect_tx(&bar_kfull[ks], T);
                for (int a = 0; a < Cfg::kAtoms; ++a)
                    BWD_LOAD(smem + (1 + ks) * T + a * Cfg::kAtomBytes, &tm_k, &bar_kfull[ks], a * 64, J * kBlk, head, pol_last);
                mbar_wait(&bar_vempty[vs], ((j / kVS) & 1) ^ 1);
                mbar_arrive_expect_tx(&bar_vfull[vs], T);
                for (int a = 0; a < Cfg::kAtoms; ++a)
                    BWD_LOAD(smem + (1 + kKS + vs) * T + a * Cfg::kAtomBytes, &tm_v, &bar_vfull[vs], a * 64,
                                J * kBlk, head, pol_last);
            }
        } else if (warp == 1) {  // whole warp, converged (elected issue)
            // ------------------------------------------------ MMA issuer
            mbar_wait(bar_q, 0);
            mbar_wait(bar_do, 0);
            tc_fence_after();
            const uint64_t dkm = kbase(smem_u32(smem));  // K-major view of every tile
            const uint64_t dmn = mnbase(smem_u32(smem));  // MN-major view
            // dQ += dS(j) K_j  (A = dS from TMEM, B = K_j MN-major, K = 128 keys)
            auto dq_mma = [&](auto KSC, bool first) {
                constexpr int ks = decltype(KSC)::value;
                // 8 K-steps (16 keys each) as two groups of four (grouped elected issue)
                mma_ts_x4<(((1 + ks) * T) >> 4) + mnoff(0), mnoff(16)>(kTmem + kColDQ, kTmem + kColDS, dmn,
                                                                      Cfg::kIdAcc, first ? 0u : 1u);
                mma_ts_x4<(((1 + ks) * T) >> 4) + mnoff(64), mnoff(16)>(kTmem + kColDQ, kTmem + kColDS + 32, dmn,
                                                                       Cfg::kIdAcc, 1u);
            };
            // step j: ring slots are compile-time constants (the loop is unrolled by kUnroll)
            auto block = [&](uint32_t j, auto PC) {
                constexpr int P6 = decltype(PC)::value;  // == j % kUnroll
                constexpr int ks = P6 % kKS, vs = P6 % kVS, ksp = (P6 + kKS - 1) % kKS;
                // S(j) = Q K_j^T  (TS: Q from TMEM)
                mbar_wait(&bar_kfull[ks], (j / kKS) & 1);
                if (j > 0) mbar_wait(bar_sfree, (j - 1) & 1);
                tc_fence_after();
                static_for<Cfg::kAtoms>([&](auto AC) {
                    constexpr int at = decltype(AC)::value;  // four K-steps per 64-column atom of d
                    mma_ts_x4<koff(4 * at, 0) + (((1 + ks) * T) >> 4), 2>(kTmem + kColS, kTmem + kColQ + 32 * at, dkm,
                                                                          Cfg::kIdAcc128, at ? 1u : 0u);
                });
                mma_commit_w(bar_s);
                BTRACE(1, j);
                // dP(j) = dO V_j^T  (SS)
                mbar_wait(&bar_vfull[vs], (j / kVS) & 1);
                if (j > 0) mbar_wait(bar_dpfree, (j - 1) & 1);
                tc_fence_after();
                static_for<Cfg::kAtoms>([&](auto AC) {
                    constexpr int at = decltype(AC)::value;
                    mma_ss_x4<koff(4 * at, 0), koff(4 * at, 0) + (((1 + kKS + vs) * T) >> 4)>(kTmem + kColDP, dkm, dkm,
                                                                                             Cfg::kIdAcc128, at ? 1u : 0u);
                });
                mma_commit_w(bar_dp);
                mma_commit_w(&bar_vempty[vs]);
                BTRACE(2, j);
                // dQ += dS(j-1) K_{j-1}
                if (j > 0) {
                    mbar_wait(bar_ds, (j - 1) & 1);
                    BTRACE(3, j);
                    tc_fence_after();
                    dq_mma(std::integral_constant<int, ksp>{}, j == 1);
                    mma_commit_w(&bar_kempty[ksp]);
                    mma_commit_w(bar_dsfree);
                }
            };
            for (uint32_t j = 0; j < L; j += kUnroll) {
                static_for<kUnroll>([&](auto UC) {
                    if (j + decltype(UC)::value < L) block(j + decltype(UC)::value, UC);
                });
            }
            if (L > 0) {
                mbar_wait(bar_ds, (L - 1) & 1);
                tc_fence_after();
                static_for<kKS>([&](auto KC) {
                    if ((L - 1) % kKS == decltype(KC)::value) dq_mma(KC, L == 1);
                });
            }
            mma_commit_w(bar_acc);
        }
    } else {
        regs_inc<RADIAL_REGS_HI>();
        // ---------------------------------------------------- elementwise
        const int wg = (warp - 4) >> 2;  // key columns [64 wg, 64 wg + 64)
        const int r = ((warp & 3) << 5) + lane;
        const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint64_t row = static_cast<uint64_t>(I) * kBlk + r;
        const uint64_t prow = static_cast<uint64_t>(head) * p.rpad + row;
        {
            // resident A operand: this row of Q as packed bf16 pairs in TMEM (lane = row,
            // column c = elements 2c, 2c+1); warpgroup g stores elements [D/2 g, D/2 (g+1))
            const __nv_bfloat16* src = p.q + (static_cast<uint64_t>(head) * p.n + row) * D + wg * (D / 2);
#pragma unroll
            for (int c = 0; c < D / 4; c += 16) {
                uint32_t w[16];
                if (row < p.n) {
                    const uint4* g = reinterpret_cast<const uint4*>(src + 2 * c);
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const uint4 u = __ldg(g + x);
                        w[4 * x] = u.x;
                        w[4 * x + 1] = u.y;
                        w[4 * x + 2] = u.z;
                        w[4 * x + 3] = u.w;
                    }
                } else {
#pragma unroll
                    for (int x = 0; x < 16; ++x) w[x] = 0u;
                }
                tmem_st16(kTmem + la + kColQ + wg * (D / 4) + c, w);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_q);
        }
        const float lse2 = p.lse2[prow];
        const float dval = p.dvec[prow];
        const float sl2 = p.scale_log2;
        for (uint32_t j = 0; j < L; ++j) {
            const uint32_t J = __ldg(p.idx + e0 + j);
            mbar_wait(bar_s, j & 1);
            if (warp == 4 && lane == 0) BTRACE(5, j);
            tc_fence_after();
            uint32_t sv[64];
            uint32_t dp[64];
            const uint64_t key0 = static_cast<uint64_t>(J) * kBlk + wg * 64;
            const int valid = key0 + 64 <= p.n ? 64 : (key0 < p.n ? static_cast<int>(p.n - key0) : 0);
            float pv[64];
            const float2 sl = make_float2(sl2, sl2), nl = make_float2(-lse2, -lse2);
#if RADIAL_BWD_DQ_SPLIT_S
            // the first 32 columns, then the second half's load runs under their exponentials
            tmem_ld32(kTmem + la + kColS + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_wait_ld();
            tmem_ld32(kTmem + la + kColS + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
#else
            tmem_ld64(kTmem + la + kColS + wg * 64, sv);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_sfree);
#endif
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
#if RADIAL_BWD_DQ_SPLIT_S
                if (c == 32) {
                    tmem_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_sfree);
                }
#endif
#if RADIAL_BWD_DQ_EARLY_DP
                if (c == RADIAL_BWD_DQ_EARLY_DP) {
                    // dP(j) (computed right after S(j)) is loaded under the last exponentials
                    mbar_wait(bar_dp, j & 1);
                    tc_fence_after();
                    tmem_ld64(kTmem + la + kColDP + wg * 64, dp);
                }
#endif
                const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sl, nl);
                if (((c >> 1) & 7) < RADIAL_BWD_DQ_POLY) {
                    // a share of the exponentials on the FMA pipe: this loop's chain is bound by
                    // the MUFU queue (two warps x 64 ex2 per sub-partition), not by issue slots
                    const float2 pr = ex2_poly2(x);
                    pv[c] = pr.x;
                    pv[c + 1] = pr.y;
                } else {
                    pv[c] = ex2(x.x);
                    pv[c + 1] = ex2(x.y);
                }
            }
            if (valid < 64) {
#pragma unroll
                for (int c = 0; c < 64; ++c) pv[c] = c < valid ? pv[c] : 0.f;
            }
#if !RADIAL_BWD_DQ_EARLY_DP
            mbar_wait(bar_dp, j & 1);
            tc_fence_after();
#ifdef RADIAL_BWD_LD32
            tmem_ld32(kTmem + la + kColDP + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(dp));
            tmem_ld32(kTmem + la + kColDP + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(dp + 32));
#else
            tmem_ld64(kTmem + la + kColDP + wg * 64, dp);
#endif
#endif
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_dpfree);
            uint32_t pk[32];
            const float2 nd = make_float2(-dval, -dval);
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
                const float2 g = __fadd2_rn(make_float2(__uint_as_float(dp[c]), __uint_as_float(dp[c + 1])), nd);
                const float2 ds = __fmul2_rn(make_float2(pv[c], pv[c + 1]), g);
                pk[c / 2] = pack_bf16(ds.x, ds.y);
            }
            if (j > 0) mbar_wait(bar_dsfree, (j - 1) & 1);
            tc_fence_after();
            tmem_st16(kTmem + la + kColDS + wg * 32, pk);
            tmem_st16(kTmem + la + kColDS + wg * 32 + 16, pk + 16);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_ds);
            if (warp == 4 && lane == 0) BTRACE(6, j);
        }
        // ---------------------------------------------------- epilogue: dQ * scale
        mbar_wait(bar_acc, 0);
        tc_fence_after();
        constexpr int kHalf = D / 2;
#pragma unroll
        for (int c = 0; c < kHalf; c += 32) {
            uint32_t u[32];
            tmem_ld32(kTmem + la + kColDQ + wg * kHalf + c, u);
            tmem_wait_ld();
            if (row < p.n) {
                uint32_t w[16];
#pragma unroll
                for (int x = 0; x < 16; ++x)
                    w[x] = L ? pack_bf16(__uint_as_float(u[2 * x]) * p.scale, __uint_as_float(u[2 * x + 1]) * p.scale) : 0u;
                uint4* dst = reinterpret_cast<uint4*>(p.dq + (static_cast<uint64_t>(head) * p.n + row) * D + wg * kHalf + c);
#pragma unroll
                for (int x = 0; x < 4; ++x) dst[x] = make_uint4(w[4 * x], w[4 * x + 1], w[4 * x + 2], w[4 * x + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(*tmem_slot, 512);
    }
}

// ========================================================================== dK/dV
// CTA per (head, KV block J) over its CSC column; K_J, V_J resident in shared memory,
// Q_I through a 3-stage ring, dO_I (+ lse2 / D of its rows) through a 2-stage ring.
// Every MMA is 128 x 128 x 16 (N = 64 MMAs run at ~53 instead of 32 clk on B200).
// TMEM: S^T [0,128) dP^T [128,256) dV [256,384) dK [384,512).
// The warpgroups release S^T(i) as soon as they have loaded it, so S^T(i+1) is computed
// while they work on block i.  Warpgroup g owns query columns [64g, 64g+64); once it has
// loaded its dP^T(i) columns it writes P^T(i) (bf16) to [128+64g, +32) and dS^T(i) to
// [128+64g+32, +32) -- inside its own range, never over values the other one still reads.
// MMA issue order per query block i:  dP^T(i), S^T(i+1), dV(i), dK(i).  The warpgroups'
// exponentials for block i run while the tensor core computes dK(i-1) and dP^T(i).
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    radial_attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                                const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                                const BwdParams p) {
    using Cfg = BwdCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    // the dynamic window starts 1 KB-aligned on sm_100 (checked): no alignment slack, the
    // 3 + 2 stage rings use 226 KB of the 227 KB
    if (smem_u32(smem_raw) & 1023u) __trap();
    uint8_t* smem = smem_raw;
    constexpr int T = Cfg::kTileBytes;
    constexpr int kQS = 3, kDS = 2;
    // [K | V | Q0 Q1 Q2 | dO0 dO1 | lse2/D for dO stage 0 (1 KB), stage 1 (1 KB) | barriers]
    constexpr int kOffQ = 2 * T, kOffDO = kOffQ + kQS * T;
    float* vec = reinterpret_cast<float*>(smem + kOffDO + kDS * T);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffDO + kDS * T + 2048);
    uint64_t* bar_res = bars;          // K, V landed
    uint64_t* bar_qfull = bars + 1;    // [3] Q_i landed
    uint64_t* bar_qempty = bars + 4;   // [3] Q_i free (dK(i) done)
    uint64_t* bar_dofull = bars + 7;   // [2] dO_i + lse2/D landed
    uint64_t* bar_doempty = bars + 9;  // [2] dO_i free (dV(i) done; the warpgroups are past block i)
    uint64_t* bar_s = bars + 11;       // S^T(i) computed
    uint64_t* bar_sfree = bars + 12;   // S^T(i) loaded by the warpgroups (8)
    uint64_t* bar_dp = bars + 13;      // dP^T(i) computed
    uint64_t* bar_p = bars + 14;       // [2] P^T(i) query halves in TMEM (8 each)
    uint64_t* bar_ds = bars + 16;      // dS^T(i) in TMEM (8)
    uint64_t* bar_acc = bars + 17;     // dV, dK final
    uint64_t* bar_vecempty = bars + 18;  // [2] the stage's lse2 / D read by the 8 elementwise warps
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t head = blockIdx.x / p.R;
    const uint32_t J = p.order[blockIdx.x % p.R];
    const uint64_t e0 = p.ptr[J];
    const uint32_t L = static_cast<uint32_t>(p.ptr[J + 1] - e0);

    if (warp == 0 && lane == 0) {
        mbar_init(bar_res, 1);
        for (int i = 0; i < kQS; ++i) {
            mbar_init(&bar_qfull[i], 1);
            mbar_init(&bar_qempty[i], 1);
        }
        for (int i = 0; i < kDS; ++i) {
            mbar_init(&bar_dofull[i], 1);
            mbar_init(&bar_doempty[i], 1);   // the MMA warp's commit: dV(i), dK(i) done with dO_i
            // every thread of the 8 elementwise warps, done reading the stage's lse2 / D (generic
            // proxy); a barrier of their own, so the next bulk load into the stage is ordered
            // after those reads by plain thread arrivals (not mixed with the tcgen05.commit)
            mbar_init(&bar_vecempty[i], 8 * 32);
        }
        mbar_init(bar_s, 1);
        mbar_init(bar_sfree, 8);
        mbar_init(bar_dp, 1);
        mbar_init(&bar_p[0], 8);
        mbar_init(&bar_p[1], 8);
        mbar_init(bar_ds, 8);
        mbar_init(bar_acc, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();  // all 512 columns allocated: the base is column 0 by construction
    constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 384;

    if (warp < 4) {
        regs_dec<RADIAL_REGS_LO>();
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------ producer
            // K_J / V_J are read once (evict-first); Q_I / dO_I are re-read by every KV block
            // of their CSR row (evict-last)
            [[maybe_unused]] const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
            mbar_arrive_expect_tx(bar_res, 2 * T);
            for (int a = 0; a < Cfg::kAtoms; ++a) {
                BWD_LOAD(smem + a * Cfg::kAtomBytes, &tm_k, bar_res, a * 64, J * kBlk, head, pol_first);
                BWD_LOAD(smem + T + a * Cfg::kAtomBytes, &tm_v, bar_res, a * 64, J * kBlk, head, pol_first);
            }
            for (uint32_t i = 0; i < L; ++i) {
                const int qs = i % kQS, ds = i % kDS;
                const uint32_t Iq = __ldg(p.idx + e0 + i);
                mbar_wait(&bar_qempty[qs], ((i / kQS) & 1) ^ 1);
                mbar_arrive_expect_tx(&bar_qfull[qs], T);
                for (int a = 0; a < Cfg::kAtoms; ++a)
                    BWD_LOAD(smem + kOffQ + qs * T + a * Cfg::kAtomBytes, &tm_q, &bar_qfull[qs], a * 64,
                                Iq * kBlk, head, pol_last);
                mbar_wait(&bar_doempty[ds], ((i / kDS) & 1) ^ 1);
                mbar_wait(&bar_vecempty[ds], ((i / kDS) & 1) ^ 1);
                mbar_arrive_expect_tx(&bar_dofull[ds], T + 2 * kBlk * 4);
                for (int a = 0; a < Cfg::kAtoms; ++a)
                    BWD_LOAD(smem + kOffDO + ds * T + a * Cfg::kAtomBytes, &tm_do, &bar_dofull[ds], a * 64,
                                Iq * kBlk, head, pol_last);
                const uint64_t off = static_cast<uint64_t>(head) * p.rpad + static_cast<uint64_t>(Iq) * kBlk;
                bulk_load(vec + ds * 256, p.lse2 + off, kBlk * 4, &bar_dofull[ds]);
                bulk_load(vec + ds * 256 + 128, p.dvec + off, kBlk * 4, &bar_dofull[ds]);
            }
        } else if (warp == 1) {  // whole warp, converged (elected issue)
            // ------------------------------------------------ MMA issuer
            mbar_wait(bar_res, 0);
            tc_fence_after();
            const uint64_t dkm = kbase(smem_u32(smem));        // K-major view of every tile
            const uint64_t dmn = mnbase(smem_u32(smem));       // MN-major view
            constexpr uint32_t kK = 0, kV = T;                 // tile byte offsets
            // S^T(i) = K Q_i^T  (M = 128 keys, N = 128 queries, K = d)
            auto s_mma = [&](uint32_t i, auto QC) {
                constexpr int qs = decltype(QC)::value;
                mbar_wait(&bar_qfull[qs], (i / kQS) & 1);
                if (i > 0) mbar_wait(bar_sfree, (i - 1) & 1);
                tc_fence_after();
                static_for<Cfg::kAtoms>([&](auto AC) {
                    constexpr int at = decltype(AC)::value;
                    mma_ss_x4<koff(4 * at, 0) + (kK >> 4), koff(4 * at, 0) + ((kOffQ + qs * T) >> 4)>(
                        kTmem + kColS, dkm, dkm, Cfg::kIdAcc128, at ? 1u : 0u);
                });
                mma_commit_w(bar_s);
                BTRACE(0, i);
            };
            // step i (P6 = i % 6 keeps every ring slot a compile-time constant)
            auto block = [&](uint32_t i, auto PC) {
                constexpr int P6 = decltype(PC)::value;
                constexpr int qs = P6 % kQS, ds = P6 % kDS, qn = (P6 + 1) % kQS;
                // dP^T(i) = V dO_i^T
                mbar_wait(&bar_dofull[ds], (i / kDS) & 1);
                tc_fence_after();
                static_for<Cfg::kAtoms>([&](auto AC) {
                    constexpr int at = decltype(AC)::value;
                    mma_ss_x4<koff(4 * at, 0) + (kV >> 4), koff(4 * at, 0) + ((kOffDO + ds * T) >> 4)>(
                        kTmem + kColDP, dkm, dkm, Cfg::kIdAcc128, at ? 1u : 0u);
                });
                mma_commit_w(bar_dp);
                BTRACE(2, i);
                if (i + 1 < L) s_mma(i + 1, std::integral_constant<int, qn>{});
                // dV += P^T(i) dO_i, in two query halves (h = 0: queries 0-31 and 64-95,
                // h = 1: 32-63 and 96-127)
                static_for<2>([&](auto HC) {
                    constexpr int h = decltype(HC)::value;
                    mbar_wait(&bar_p[h], i & 1);
                    if (h == 0) BTRACE(3, i);
                    tc_fence_after();
                    // K-steps 2h, 2h+1 (warpgroup 0's queries), then 4+2h, 5+2h (warpgroup 1's)
                    mma_ts_x2<((kOffDO + ds * T) >> 4) + mnoff(32 * h), mnoff(16)>(
                        kTmem + kColDV, kTmem + kColDP + 16 * h, dmn, Cfg::kIdAcc, (i > 0 || h) ? 1u : 0u);
                    mma_ts_x2<((kOffDO + ds * T) >> 4) + mnoff(64 + 32 * h), mnoff(16)>(
                        kTmem + kColDV, kTmem + kColDP + 64 + 16 * h, dmn, Cfg::kIdAcc, 1u);
                });
                BTRACE(4, i);
                // dK += dS^T(i) Q_i  (A = dS^T from TMEM, B = Q_i MN-major, K = 128 queries)
                mbar_wait(bar_ds, i & 1);
                tc_fence_after();
                // queries 0-63 (warpgroup 0's dS^T columns), then 64-127 (warpgroup 1's)
                mma_ts_x4<((kOffQ + qs * T) >> 4) + mnoff(0), mnoff(16)>(kTmem + kColDK, kTmem + kColDP + 32, dmn,
                                                                        Cfg::kIdAcc, i > 0 ? 1u : 0u);
                mma_ts_x4<((kOffQ + qs * T) >> 4) + mnoff(64), mnoff(16)>(kTmem + kColDK, kTmem + kColDP + 96, dmn,
                                                                         Cfg::kIdAcc, 1u);
                mma_commit_w(&bar_doempty[ds]);
                mma_commit_w(&bar_qempty[qs]);
                BTRACE(1, i);
            };
            if (L > 0) s_mma(0, std::integral_constant<int, 0>{});
            for (uint32_t i = 0; i < L; i += 6) {
                block(i, std::integral_constant<int, 0>{});
                if (i + 1 < L) block(i + 1, std::integral_constant<int, 1>{});
                if (i + 2 < L) block(i + 2, std::integral_constant<int, 2>{});
                if (i + 3 < L) block(i + 3, std::integral_constant<int, 3>{});
                if (i + 4 < L) block(i + 4, std::integral_constant<int, 4>{});
                if (i + 5 < L) block(i + 5, std::integral_constant<int, 5>{});
            }
            mma_commit_w(bar_acc);
        }
    } else {
        regs_inc<RADIAL_REGS_HI>();
        const int wg = (warp - 4) >> 2;  // query columns [64 wg, 64 wg + 64)
        const int r = ((warp & 3) << 5) + lane;  // key row of the tile
        const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint64_t krow = static_cast<uint64_t>(J) * kBlk + r;
        const float sl2 = p.scale_log2;
        for (uint32_t i = 0; i < L; ++i) {
            const int ds = i % kDS;
            mbar_wait(bar_s, i & 1);
            if (warp == 4 && lane == 0) BTRACE(5, i);
            tc_fence_after();
            uint32_t sv[64];
#ifdef RADIAL_BWD_LD32
            tmem_ld32(kTmem + la + kColS + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_ld32(kTmem + la + kColS + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
#else
            tmem_ld64(kTmem + la + kColS + wg * 64, sv);
#endif
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_sfree);
            // lse2 / D of this block's queries travel with dO_i
            mbar_wait(&bar_dofull[ds], (i / kDS) & 1);
            const float4* lv = reinterpret_cast<const float4*>(vec + ds * 256 + wg * 64);
            float pv[64];
            const float2 sl = make_float2(sl2, sl2);
            uint32_t dp[64];
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
#if RADIAL_BWD_DKDV_EARLY_DP
                if (c4 == RADIAL_BWD_DKDV_EARLY_DP / 4) {  // dP^T(i) loaded under the last exponentials
                    mbar_wait(bar_dp, i & 1);
                    tc_fence_after();
                    tmem_ld64(kTmem + la + kColDP + wg * 64, dp);
                }
#endif
                const float4 l4 = lv[c4];
                const float2 xa = __ffma2_rn(make_float2(__uint_as_float(sv[4 * c4]), __uint_as_float(sv[4 * c4 + 1])),
                                             sl, make_float2(-l4.x, -l4.y));
                const float2 xb = __ffma2_rn(make_float2(__uint_as_float(sv[4 * c4 + 2]), __uint_as_float(sv[4 * c4 + 3])),
                                             sl, make_float2(-l4.z, -l4.w));
                if ((c4 & 7) < RADIAL_BWD_DKDV_POLY) {  // a share of the exp2 on the FMA pipe
                    const float2 pa = ex2_poly2(xa), pb = ex2_poly2(xb);
                    pv[4 * c4 + 0] = pa.x;
                    pv[4 * c4 + 1] = pa.y;
                    pv[4 * c4 + 2] = pb.x;
                    pv[4 * c4 + 3] = pb.y;
                } else {
                    pv[4 * c4 + 0] = ex2(xa.x);
                    pv[4 * c4 + 1] = ex2(xa.y);
                    pv[4 * c4 + 2] = ex2(xb.x);
                    pv[4 * c4 + 3] = ex2(xb.y);
                }
            }
            if ((warp == 4 || warp == 8) && lane == 0) BTRACE(warp == 4 ? 7 : 10, i);
#if !RADIAL_BWD_DKDV_EARLY_DP
            mbar_wait(bar_dp, i & 1);
            if (warp == 4 && lane == 0) BTRACE(8, i);
            tc_fence_after();
#ifdef RADIAL_BWD_LD32
            tmem_ld32(kTmem + la + kColDP + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(dp));
            tmem_ld32(kTmem + la + kColDP + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(dp + 32));
#else
            tmem_ld64(kTmem + la + kColDP + wg * 64, dp);
#endif
#endif
            tmem_wait_ld();
            // P^T into the (now consumed) dP^T columns, in two query halves
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t pp[16];
#pragma unroll
                for (int x = 0; x < 16; ++x) pp[x] = pack_bf16(pv[32 * h + 2 * x], pv[32 * h + 2 * x + 1]);
                tmem_st16(kTmem + la + kColDP + wg * 64 + 16 * h, pp);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_p[h]);
            }
            const float4* dvv = reinterpret_cast<const float4*>(vec + ds * 256 + 128 + wg * 64);
            uint32_t pd[32];
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
                const float4 d4 = dvv[c4];
                const float2 ga = __fadd2_rn(make_float2(__uint_as_float(dp[4 * c4]), __uint_as_float(dp[4 * c4 + 1])),
                                             make_float2(-d4.x, -d4.y));
                const float2 gb = __fadd2_rn(make_float2(__uint_as_float(dp[4 * c4 + 2]), __uint_as_float(dp[4 * c4 + 3])),
                                             make_float2(-d4.z, -d4.w));
                const float2 a = __fmul2_rn(make_float2(pv[4 * c4], pv[4 * c4 + 1]), ga);
                const float2 b = __fmul2_rn(make_float2(pv[4 * c4 + 2], pv[4 * c4 + 3]), gb);
                pd[2 * c4] = pack_bf16(a.x, a.y);
                pd[2 * c4 + 1] = pack_bf16(b.x, b.y);
            }
            tmem_st16(kTmem + la + kColDP + wg * 64 + 32, pd);
            tmem_st16(kTmem + la + kColDP + wg * 64 + 48, pd + 16);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            fence_proxy_async_smem();  // the stage's lse2 / D reads before the next bulk load into it
            // every lane releases its own reads of the stage (an elected arrive after __syncwarp
            // is equally correct, but compute-sanitizer racecheck does not model __syncwarp and
            // reports it: scripts/racecheck_probe.py mode 1)
            mbar_arrive(&bar_vecempty[ds]);
            if (lane == 0) mbar_arrive(bar_ds);  // dS^T stores: ordered by the __syncwarp above
            if ((warp == 4 || warp == 8) && lane == 0) BTRACE(warp == 4 ? 9 : 11, i);
        }
        // ---------------------------------------------------- epilogue: wg0 -> dV, wg1 -> dK * scale
        mbar_wait(bar_acc, 0);
        tc_fence_after();
        const float mul = wg ? p.scale : 1.f;
        __nv_bfloat16* out = (wg ? p.dk : p.dv) + (static_cast<uint64_t>(head) * p.n + krow) * D;
#pragma unroll
        for (int c = 0; c < D; c += 32) {
            uint32_t u[32];
            tmem_ld32(kTmem + la + (wg ? kColDK : kColDV) + c, u);
            tmem_wait_ld();
            if (krow < p.n) {
                uint32_t w[16];
#pragma unroll
                for (int x = 0; x < 16; ++x)
                    w[x] = L ? pack_bf16(__uint_as_float(u[2 * x]) * mul, __uint_as_float(u[2 * x + 1]) * mul) : 0u;
                uint4* dst = reinterpret_cast<uint4*>(out + c);
#pragma unroll
                for (int x = 0; x < 4; ++x) dst[x] = make_uint4(w[4 * x], w[4 * x + 1], w[4 * x + 2], w[4 * x + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(*tmem_slot, 512);
    }
}

template <int D>
int launch_bwd_t(const void* q, const void* k, const void* v, const void* o, const float* lse,
                 const void* dout, void* dq, void* dk, void* dv, uint32_t heads, uint64_t n,
                 float scale, const radial_layout* L, void* workspace, cudaStream_t st) {
    using namespace radial_detail;
    const uint64_t R = L->R;
    const uint64_t rpad = R * kBlk;
    float* lse2 = static_cast<float*>(workspace);
    float* dvec = lse2 + heads * rpad;
    {
        const uint64_t warps = heads * rpad;
        const unsigned blocks = static_cast<unsigned>((warps * 32 + 255) / 256);
        bwd_prep_kernel<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                                 static_cast<const __nv_bfloat16*>(dout), lse, lse2, dvec, n,
                                                 rpad, D, heads);
        RADIAL_CUDA_TRY(cudaGetLastError());
    }
    CUtensorMap tq, tdo, tk, tv;
    int rc;
    if ((rc = make_tmap_bf16_3d(&tq, q, n, D, heads, kBlk))) return rc;
    if ((rc = make_tmap_bf16_3d(&tdo, dout, n, D, heads, kBlk))) return rc;
    if ((rc = make_tmap_bf16_3d(&tk, k, n, D, heads, kBlk))) return rc;
    if ((rc = make_tmap_bf16_3d(&tv, v, n, D, heads, kBlk))) return rc;
    BwdParams p{};
    p.q = static_cast<const __nv_bfloat16*>(q);
    p.dout = static_cast<const __nv_bfloat16*>(dout);
    p.dq = static_cast<__nv_bfloat16*>(dq);
    p.dk = static_cast<__nv_bfloat16*>(dk);
    p.dv = static_cast<__nv_bfloat16*>(dv);
    p.lse2 = lse2;
    p.dvec = dvec;
    p.n = n;
    p.rpad = rpad;
    p.heads = heads;
    p.R = static_cast<uint32_t>(R);
    p.scale = scale;
    p.scale_log2 = scale * kLog2e;
    const uint64_t items = heads * R;
    if (items > 0x7fffffffull) return fail(RADIAL_ERR_INVALID, "attn_bwd: too many work items");
    const int T = BwdCfg<D>::kTileBytes;
    {
        const int smem = 7 * T + 256 + 1024;  // dO, 4 K + 2 V stages, barriers
        auto kern = radial_attn_bwd_dq_kernel<D>;
        RADIAL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        p.ptr = L->row_ptr;
        p.idx = L->col_idx;
        p.order = L->rorder;
        kern<<<static_cast<unsigned>(items), kThreads, smem, st>>>(tq, tdo, tk, tv, p);
        RADIAL_CUDA_TRY(cudaGetLastError());
    }
#ifdef RADIAL_TRACE
    if (getenv("RADIAL_BWD_DQ_ONLY")) return RADIAL_OK;  // trace builds: time the dQ kernel alone
#endif
    {
        const int smem = 7 * T + 2048 + 176;  // K, V, 3 Q, 2 dO, lse2/D, 20 barriers + TMEM slot (no align slack)
        auto kern = radial_attn_bwd_dkdv_kernel<D>;
        RADIAL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        p.ptr = L->col_ptr;
        p.idx = L->row_idx;
        p.order = L->corder;
        kern<<<static_cast<unsigned>(items), kThreads, smem, st>>>(tq, tdo, tk, tv, p);
        RADIAL_CUDA_TRY(cudaGetLastError());
    }
    count_launches(3);
    note_use(L, st);
    return RADIAL_OK;
}

}  // namespace

namespace radial_detail {

size_t bwd_workspace_bytes(uint32_t heads, uint64_t n, uint32_t D) {
    (void)D;
    const uint64_t rpad = ((n + kBlk - 1) / kBlk) * kBlk;
    return static_cast<size_t>(2) * heads * rpad * sizeof(float) + 256;
}

int launch_bwd(const void* q, const void* k, const void* v, const void* o, const float* lse,
               const void* dout, void* dq, void* dk, void* dv, uint32_t heads, uint64_t n, uint32_t D,
               float scale, const radial_layout* L, void* workspace, cudaStream_t st) {
    if (!workspace) return fail(RADIAL_ERR_INVALID, "attn_bwd: null workspace");
    if (L->B != kBlk) return fail(RADIAL_ERR_INVALID, "attn_bwd: block_size must be 128 on the device path");
    if (!L->rorder || !L->corder) return fail(RADIAL_ERR_INVALID, "attn_bwd: layout has no work lists");
    if (D == 128) return launch_bwd_t<128>(q, k, v, o, lse, dout, dq, dk, dv, heads, n, scale, L, workspace, st);
    if (D == 64) return launch_bwd_t<64>(q, k, v, o, lse, dout, dq, dk, dv, heads, n, scale, L, workspace, st);
    return fail(RADIAL_ERR_INVALID, "attn_bwd: head_dim must be 64 or 128");
}

#ifdef RADIAL_TRACE
extern "C" int radial_cuda_debug_btrace(void* buf) {
    RADIAL_CUDA_TRY(cudaMemcpyToSymbol(g_btrace, &buf, sizeof(void*)));
    return RADIAL_OK;
}
#endif

}  // namespace radial_detail
