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
//   bwd_dq      one CTA per (head, query block I) over its CSR row: S, dP on
//               tcgen05 into TMEM, dS (bf16) written back to TMEM, dQ += dS K (TS MMA)
//   bwd_dkdv    one CTA per (head, KV block J) over its CSC column: S^T, dP^T,
//               then dV += P^T dO and dK += dS^T Q with P^T / dS^T in TMEM
// Both stream the other operand in 128-row blocks split into two 64-row
// sub-steps whose S / dP TMEM buffers alternate, so the tensor core computes
// sub-step s+1 while warpgroup (s mod 2) does the elementwise work of s.
// Block size 128 only (the layouts of the BASELINE backward configs).
#include <cmath>
#include <type_traits>

#include "radial_internal.h"
#include "sm100.cuh"

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

namespace {

constexpr int kThreads = 384;   // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warps 4-11 elementwise
constexpr int kBlk = 128;       // layout block = rows per resident tile
constexpr int kSub = 64;        // streamed rows per sub-step
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
    static constexpr uint32_t kIdS = idesc_bf16(128, kSub, 0, 0);  // 128 x 64 x 16, K-major both
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

// K-major descriptor of MMA k-step kk (16 elements of d) for a 128-row tile,
// optionally starting at row `row0` (multiple of 8).
__device__ __forceinline__ uint64_t kdesc(uint32_t tile, int kk, int row0) {
    return sdesc_sw128(tile + (kk >> 2) * (kBlk * 128) + row0 * 128 + (kk & 3) * 32, 16, 1024);
}
// MN-major descriptor (B operand with N = d) of 16 rows starting at `row0`.
__device__ __forceinline__ uint64_t mndesc(uint32_t tile, int row0) {
    return sdesc_sw128(tile + row0 * 128, kBlk * 128, 1024);
}

// ============================================================================ dQ
// TMEM: S0 [0,64) S1 [64,128) dP0 [128,192) dP1 [192,256) dQ [256,256+D) Q [384,448) dO [448,512)
constexpr uint32_t kColQ = 384, kColDO = 448;
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    radial_attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                              const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                              const BwdParams p) {
    using Cfg = BwdCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int T = Cfg::kTileBytes;
    // [Q | dO | K0 V0 | K1 V1]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * T);
    uint64_t* bar_res = bars;          // Q, dO landed
    uint64_t* bar_full = bars + 1;     // [2] K/V stage landed
    uint64_t* bar_empty = bars + 3;    // [2] K/V stage free
    uint64_t* bar_s = bars + 5;        // [2] S/dP sub-buffer computed
    uint64_t* bar_ds = bars + 7;       // [2] dS sub-buffer written
    uint64_t* bar_acc = bars + 9;      // dQ final
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t head = blockIdx.x / p.R;
    const uint32_t I = p.order[blockIdx.x % p.R];
    const uint64_t e0 = p.ptr[I];
    const uint32_t L = static_cast<uint32_t>(p.ptr[I + 1] - e0);

    if (warp == 0 && lane == 0) {
        mbar_init(bar_res, 8);  // Q / dO rows stored into TMEM by the 8 elementwise warps
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_full[i], 1);
            mbar_init(&bar_empty[i], 1);
            mbar_init(&bar_s[i], 1);
            mbar_init(&bar_ds[i], 4);
        }
        mbar_init(bar_acc, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (*tmem_slot != 0) __trap();

    if (warp < 4) {
        regs_dec<104>();
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------ producer
            for (uint32_t j = 0; j < L; ++j) {
                const int st = j & 1;
                const int32_t J = static_cast<int32_t>(__ldg(p.idx + e0 + j));
                mbar_wait(&bar_empty[st], ((j >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&bar_full[st], 2 * T);
                uint8_t* kd = smem + (2 + 2 * st) * T;
                for (int a = 0; a < Cfg::kAtoms; ++a) {
                    tma_load_3d(kd + a * Cfg::kAtomBytes, &tm_k, &bar_full[st], a * 64, J * kBlk, head);
                    tma_load_3d(kd + T + a * Cfg::kAtomBytes, &tm_v, &bar_full[st], a * 64, J * kBlk, head);
                }
            }
        } else if (warp == 1) {  // whole warp, converged (elected issue)
            // ------------------------------------------------ MMA issuer
            mbar_wait(bar_res, 0);
            tc_fence_after();
            const uint64_t dkv_k = kbase(smem_u32(smem + 2 * T));  // K/V stages, K-major view
            const uint64_t dkv_mn = mnbase(smem_u32(smem + 2 * T));  // K/V stages, MN-major view
            uint32_t dsph0 = 0, dsph1 = 0;
            bool acc = false;
            uint32_t dq_j = 0;  // block index of the dS being consumed (trace only)
            (void)dq_j;
            // dQ += dS(sub-buffer b) . K(rows of that sub-step), K in stage STG
            auto dq_mma = [&](auto BC, auto SC) {
                constexpr int b = decltype(BC)::value;
                constexpr int STG = decltype(SC)::value;
                uint32_t& ph = b ? dsph1 : dsph0;
                mbar_wait(&bar_ds[b], ph);
                BTRACE(3 + b, dq_j);
                ph ^= 1;
                tc_fence_after();
                static_for<kSub / 16>([&](auto KK) {
                    constexpr int kk = decltype(KK)::value;
                    mma_ts_w<((STG * 2 * T) >> 4) + mnoff(b * kSub + kk * 16)>(
                        kTmem + 256, kTmem + b * 64 + kk * 8, dkv_mn, Cfg::kIdAcc, (acc || kk) ? 1u : 0u);
                });
                acc = true;
            };
            auto block = [&](uint32_t j, auto SC) {
                constexpr int STG = decltype(SC)::value;  // == j % 2
                mbar_wait(&bar_full[STG], (j >> 1) & 1);
                BTRACE(0, j);
                tc_fence_after();
                auto sub = [&](auto BC) {
                    constexpr int b = decltype(BC)::value;
                    // S_b = Q K_sub^T ; dP_b = dO V_sub^T   (128 x 64, K = d): TS MMAs with
                    // Q / dO read from TMEM, so only the 64-row K / V sub-tile streams from
                    // shared memory (an SS MMA at N = 64 is shared-memory bound)
                    static_for<D / 16>([&](auto KK) {
                        constexpr int kk = decltype(KK)::value;
                        mma_ts_w<((STG * 2 * T) >> 4) + koff(kk, b * kSub)>(
                            kTmem + b * 64, kTmem + kColQ + kk * 8, dkv_k, Cfg::kIdS, kk ? 1u : 0u);
                    });
                    static_for<D / 16>([&](auto KK) {
                        constexpr int kk = decltype(KK)::value;
                        mma_ts_w<((STG * 2 * T + T) >> 4) + koff(kk, b * kSub)>(
                            kTmem + 128 + b * 64, kTmem + kColDO + kk * 8, dkv_k, Cfg::kIdS, kk ? 1u : 0u);
                    });
                    mma_commit_w(&bar_s[b]);
                    BTRACE(1 + b, j);
                };
                sub(std::integral_constant<int, 0>{});
                if (j > 0) {  // previous block's second sub-step, then free its K/V stage
                    dq_j = j - 1;
                    dq_mma(std::integral_constant<int, 1>{}, std::integral_constant<int, STG ^ 1>{});
                    mma_commit_w(&bar_empty[STG ^ 1]);
                }
                sub(std::integral_constant<int, 1>{});
                dq_j = j;
                dq_mma(std::integral_constant<int, 0>{}, std::integral_constant<int, STG>{});
            };
            for (uint32_t j = 0; j < L; j += 2) {
                block(j, std::integral_constant<int, 0>{});
                if (j + 1 < L) block(j + 1, std::integral_constant<int, 1>{});
            }
            if (L > 0) {
                if ((L - 1) & 1)
                    dq_mma(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
                else
                    dq_mma(std::integral_constant<int, 1>{}, std::integral_constant<int, 0>{});
            }
            mma_commit_w(bar_acc);
        }
    } else {
        regs_inc<200>();
        // ---------------------------------------------------- elementwise
        const int wg = (warp - 4) >> 2;  // sub-buffer this warpgroup owns
        const int r = ((warp & 3) << 5) + lane;
        const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint64_t row = static_cast<uint64_t>(I) * kBlk + r;
        const uint64_t prow = static_cast<uint64_t>(head) * p.rpad + row;
        {
            // resident A operands: warpgroup 0 stores this row of Q, warpgroup 1 of dO, as
            // packed bf16 pairs in TMEM (lane = row, column c = elements 2c, 2c+1)
            const __nv_bfloat16* src = (wg ? p.dout : p.q) + (static_cast<uint64_t>(head) * p.n + row) * D;
            const uint32_t col = wg ? kColDO : kColQ;
#pragma unroll
            for (int c = 0; c < D / 2; c += 16) {
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
                tmem_st16(kTmem + la + col + c, w);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_res);
        }
        const float lse2 = p.lse2[prow];
        const float dval = p.dvec[prow];
        const float sl2 = p.scale_log2;
        for (uint32_t j = 0; j < L; ++j) {
            const uint32_t J = __ldg(p.idx + e0 + j);
            if ((warp & 3) == 0 && lane == 0) BTRACE(5 + 2 * wg, j);
            mbar_wait(&bar_s[wg], j & 1);
            if ((warp & 3) == 0 && lane == 0) BTRACE(5 + 2 * wg, j);
            tc_fence_after();
            uint32_t sv[64], dp[64];
            tmem_ld32(kTmem + la + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_ld32(kTmem + la + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
            tmem_ld32(kTmem + la + 128 + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(dp));
            tmem_ld32(kTmem + la + 128 + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(dp + 32));
            tmem_wait_ld();
            const uint64_t key0 = static_cast<uint64_t>(J) * kBlk + wg * kSub;
            const int valid = key0 + kSub <= p.n ? kSub : (key0 < p.n ? static_cast<int>(p.n - key0) : 0);
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < kSub; c += 2) {
                float p0 = ex2(fmaf(__uint_as_float(sv[c]), sl2, -lse2));
                float p1 = ex2(fmaf(__uint_as_float(sv[c + 1]), sl2, -lse2));
                if (valid < kSub) {
                    p0 = c < valid ? p0 : 0.f;
                    p1 = c + 1 < valid ? p1 : 0.f;
                }
                const float d0 = p0 * (__uint_as_float(dp[c]) - dval);
                const float d1 = p1 * (__uint_as_float(dp[c + 1]) - dval);
                pk[c / 2] = pack_bf16(d0, d1);
            }
            tmem_st16(kTmem + la + wg * 64, pk);
            tmem_st16(kTmem + la + wg * 64 + 16, pk + 16);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_ds[wg]);
            if ((warp & 3) == 0 && lane == 0) BTRACE(6 + 2 * wg, j);
        }
        // ---------------------------------------------------- epilogue: dQ * scale
        mbar_wait(bar_acc, 0);
        tc_fence_after();
        constexpr int kHalf = D / 2;
#pragma unroll
        for (int c = 0; c < kHalf; c += 32) {
            uint32_t u[32];
            tmem_ld32(kTmem + la + 256 + wg * kHalf + c, u);
            tmem_wait_ld();
            if (row < p.n) {
                uint32_t w[16];
#pragma unroll
                for (int x = 0; x < 16; ++x)
                    w[x] = pack_bf16(__uint_as_float(u[2 * x]) * p.scale, __uint_as_float(u[2 * x + 1]) * p.scale);
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
// Q_I / dO_I streamed through two-stage rings.  Every MMA is 128 x 128 x 16 (N = 64
// MMAs run at ~53 instead of 32 clk on B200, scripts/mma_rate.py).
// TMEM: S^T [0,128) dP^T [128,256) dV [256,384) dK [384,512).
// Warpgroup g owns query columns [64g, 64g+64): it writes P^T (bf16) over S^T columns
// [64g, 64g+32) and dS^T over dP^T columns [128+64g, +32) -- inside its own range, so it
// never overwrites values the other warpgroup has still to read.
// MMA issue order per query block i:  S^T(i), dK(i-1), dP^T(i), dV(i), so the tensor core
// computes dK(i-1) and dP^T(i) while the warpgroups turn S^T(i) into P^T(i).
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    radial_attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                                const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                                const BwdParams p) {
    using Cfg = BwdCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int T = Cfg::kTileBytes;
    // [K | V | Q0 dO0 | Q1 dO1 | lse2/D stage0 (1 KB) | stage1 (1 KB) | barriers]
    float* vec = reinterpret_cast<float*>(smem + 6 * T);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * T + 2048);
    uint64_t* bar_res = bars;          // K, V landed
    uint64_t* bar_qfull = bars + 1;    // [2] Q_i (+ lse2/D) landed
    uint64_t* bar_qempty = bars + 3;   // [2] Q_i free (dK(i) done)
    uint64_t* bar_dofull = bars + 5;   // [2]
    uint64_t* bar_doempty = bars + 7;  // [2] dO_i free (dV(i) done)
    uint64_t* bar_s = bars + 9;        // S^T(i) computed
    uint64_t* bar_dp = bars + 10;      // dP^T(i) computed
    uint64_t* bar_p = bars + 11;       // [2] P^T(i) query halves in TMEM (8 warp arrivals each)
    uint64_t* bar_ds = bars + 13;      // dS^T(i) in TMEM (8 warp arrivals)
    uint64_t* bar_acc = bars + 14;     // dV, dK final
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t head = blockIdx.x / p.R;
    const uint32_t J = p.order[blockIdx.x % p.R];
    const uint64_t e0 = p.ptr[J];
    const uint32_t L = static_cast<uint32_t>(p.ptr[J + 1] - e0);

    if (warp == 0 && lane == 0) {
        mbar_init(bar_res, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar_qfull[i], 1);
            mbar_init(&bar_qempty[i], 1);
            mbar_init(&bar_dofull[i], 1);
            mbar_init(&bar_doempty[i], 1);
        }
        mbar_init(bar_s, 1);
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
    tc_fence_after();
    if (*tmem_slot != 0) __trap();
    constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256, kColDK = 384;

    if (warp < 4) {
        regs_dec<104>();
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------ producer
            mbar_arrive_expect_tx(bar_res, 2 * T);
            for (int a = 0; a < Cfg::kAtoms; ++a) {
                tma_load_3d(smem + a * Cfg::kAtomBytes, &tm_k, bar_res, a * 64, J * kBlk, head);
                tma_load_3d(smem + T + a * Cfg::kAtomBytes, &tm_v, bar_res, a * 64, J * kBlk, head);
            }
            for (uint32_t i = 0; i < L; ++i) {
                const int st = i & 1;
                const uint32_t Iq = __ldg(p.idx + e0 + i);
                mbar_wait(&bar_qempty[st], ((i >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&bar_qfull[st], T + 2 * kBlk * 4);
                uint8_t* qd = smem + (2 + 2 * st) * T;
                for (int a = 0; a < Cfg::kAtoms; ++a)
                    tma_load_3d(qd + a * Cfg::kAtomBytes, &tm_q, &bar_qfull[st], a * 64, Iq * kBlk, head);
                const uint64_t off = static_cast<uint64_t>(head) * p.rpad + static_cast<uint64_t>(Iq) * kBlk;
                bulk_load(vec + st * 256, p.lse2 + off, kBlk * 4, &bar_qfull[st]);
                bulk_load(vec + st * 256 + 128, p.dvec + off, kBlk * 4, &bar_qfull[st]);
                mbar_wait(&bar_doempty[st], ((i >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&bar_dofull[st], T);
                for (int a = 0; a < Cfg::kAtoms; ++a)
                    tma_load_3d(qd + T + a * Cfg::kAtomBytes, &tm_do, &bar_dofull[st], a * 64, Iq * kBlk, head);
            }
        } else if (warp == 1) {  // whole warp, converged (elected issue)
            // ------------------------------------------------ MMA issuer
            mbar_wait(bar_res, 0);
            tc_fence_after();
            const uint64_t dkm = kbase(smem_u32(smem));        // K-major view of every tile
            const uint64_t dmn = mnbase(smem_u32(smem));       // MN-major view
            constexpr uint32_t kK = 0, kV = T, kQ0 = 2 * T;    // tile byte offsets
            // dK += dS^T(i) Q_i  (A = dS^T from TMEM, B = Q_i MN-major, K = 128 queries)
            auto dk_mma = [&](auto SC, bool first) {
                constexpr int st = decltype(SC)::value;
                static_for<kBlk / 16>([&](auto KK) {
                    constexpr int kk = decltype(KK)::value;
                    constexpr uint32_t a_col = kColDP + (kk >> 2) * 64 + (kk & 3) * 8;
                    mma_ts_w<((kQ0 + st * 2 * T) >> 4) + mnoff(kk * 16)>(kTmem + kColDK, kTmem + a_col, dmn,
                                                                          Cfg::kIdAcc, (!first || kk) ? 1u : 0u);
                });
            };
            auto block = [&](uint32_t i, auto SC) {
                constexpr int st = decltype(SC)::value;  // == i % 2
                const uint32_t ph = (i >> 1) & 1;
                // S^T(i) = K Q_i^T  (M = 128 keys, N = 128 queries, K = d)
                mbar_wait(&bar_qfull[st], ph);
                tc_fence_after();
                static_for<D / 16>([&](auto KK) {
                    constexpr int kk = decltype(KK)::value;
                    mma_ss_w<koff(kk, 0) + (kK >> 4), koff(kk, 0) + ((kQ0 + st * 2 * T) >> 4)>(
                        kTmem + kColS, dkm, dkm, Cfg::kIdAcc128, kk ? 1u : 0u);
                });
                mma_commit_w(bar_s);
                BTRACE(0, i);
                if (i > 0) {
                    mbar_wait(bar_ds, (i - 1) & 1);
                    tc_fence_after();
                    dk_mma(std::integral_constant<int, st ^ 1>{}, i == 1);
                    mma_commit_w(&bar_qempty[st ^ 1]);
                    BTRACE(1, i);
                }
                // dP^T(i) = V dO_i^T
                mbar_wait(&bar_dofull[st], ph);
                tc_fence_after();
                static_for<D / 16>([&](auto KK) {
                    constexpr int kk = decltype(KK)::value;
                    mma_ss_w<koff(kk, 0) + (kV >> 4), koff(kk, 0) + ((kQ0 + st * 2 * T + T) >> 4)>(
                        kTmem + kColDP, dkm, dkm, Cfg::kIdAcc128, kk ? 1u : 0u);
                });
                mma_commit_w(bar_dp);
                BTRACE(2, i);
                // dV += P^T(i) dO_i, in two query halves (h = 0: queries 0-31 and 64-95,
                // h = 1: 32-63 and 96-127) so the first starts while the second's
                // exponentials are still being computed
                static_for<2>([&](auto HC) {
                    constexpr int h = decltype(HC)::value;
                    mbar_wait(&bar_p[h], i & 1);
                    if (h == 0) BTRACE(3, i);
                    tc_fence_after();
                    static_for<4>([&](auto KK) {
                        constexpr int kk = (decltype(KK)::value >> 1) * 4 + h * 2 + (decltype(KK)::value & 1);
                        constexpr uint32_t a_col = kColS + (kk >> 2) * 64 + (kk & 3) * 8;
                        mma_ts_w<((kQ0 + st * 2 * T + T) >> 4) + mnoff(kk * 16)>(
                            kTmem + kColDV, kTmem + a_col, dmn, Cfg::kIdAcc, (i > 0 || kk) ? 1u : 0u);
                    });
                });
                mma_commit_w(&bar_doempty[st]);
                BTRACE(4, i);
            };
            for (uint32_t i = 0; i < L; i += 2) {
                block(i, std::integral_constant<int, 0>{});
                if (i + 1 < L) block(i + 1, std::integral_constant<int, 1>{});
            }
            if (L > 0) {
                mbar_wait(bar_ds, (L - 1) & 1);
                tc_fence_after();
                if ((L - 1) & 1)
                    dk_mma(std::integral_constant<int, 1>{}, L == 1);
                else
                    dk_mma(std::integral_constant<int, 0>{}, L == 1);
            }
            mma_commit_w(bar_acc);
        }
    } else {
        regs_inc<200>();
        const int wg = (warp - 4) >> 2;  // query columns [64 wg, 64 wg + 64)
        const int r = ((warp & 3) << 5) + lane;  // key row of the tile
        const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint64_t krow = static_cast<uint64_t>(J) * kBlk + r;
        const float sl2 = p.scale_log2;
        for (uint32_t i = 0; i < L; ++i) {
            const int st = i & 1;
            mbar_wait(bar_s, i & 1);
            if (warp == 4 && lane == 0) BTRACE(5, i);
            tc_fence_after();
            uint32_t sv[64];
            tmem_ld32(kTmem + la + kColS + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(sv));
            tmem_ld32(kTmem + la + kColS + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
            tmem_wait_ld();
            const float4* lv = reinterpret_cast<const float4*>(vec + st * 256 + wg * 64);
            float pv[64];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t pp[16];
#pragma unroll
                for (int c4 = 8 * h; c4 < 8 * h + 8; ++c4) {
                    const float4 l4 = lv[c4];
                    pv[4 * c4 + 0] = ex2(fmaf(__uint_as_float(sv[4 * c4 + 0]), sl2, -l4.x));
                    pv[4 * c4 + 1] = ex2(fmaf(__uint_as_float(sv[4 * c4 + 1]), sl2, -l4.y));
                    pv[4 * c4 + 2] = ex2(fmaf(__uint_as_float(sv[4 * c4 + 2]), sl2, -l4.z));
                    pv[4 * c4 + 3] = ex2(fmaf(__uint_as_float(sv[4 * c4 + 3]), sl2, -l4.w));
                    pp[2 * (c4 - 8 * h)] = pack_bf16(pv[4 * c4], pv[4 * c4 + 1]);
                    pp[2 * (c4 - 8 * h) + 1] = pack_bf16(pv[4 * c4 + 2], pv[4 * c4 + 3]);
                }
                tmem_st16(kTmem + la + kColS + wg * 64 + 16 * h, pp);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_p[h]);
            }
            if ((warp == 4 || warp == 8) && lane == 0) BTRACE(warp == 4 ? 7 : 10, i);
            mbar_wait(bar_dp, i & 1);
            if (warp == 4 && lane == 0) BTRACE(8, i);
            tc_fence_after();
            uint32_t dp[64];
            tmem_ld32(kTmem + la + kColDP + wg * 64, *reinterpret_cast<uint32_t(*)[32]>(dp));
            tmem_ld32(kTmem + la + kColDP + wg * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(dp + 32));
            tmem_wait_ld();
            const float4* dvv = reinterpret_cast<const float4*>(vec + st * 256 + 128 + wg * 64);
            uint32_t pd[32];
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
                const float4 d4 = dvv[c4];
                const float a0 = pv[4 * c4 + 0] * (__uint_as_float(dp[4 * c4 + 0]) - d4.x);
                const float a1 = pv[4 * c4 + 1] * (__uint_as_float(dp[4 * c4 + 1]) - d4.y);
                const float a2 = pv[4 * c4 + 2] * (__uint_as_float(dp[4 * c4 + 2]) - d4.z);
                const float a3 = pv[4 * c4 + 3] * (__uint_as_float(dp[4 * c4 + 3]) - d4.w);
                pd[2 * c4] = pack_bf16(a0, a1);
                pd[2 * c4 + 1] = pack_bf16(a2, a3);
            }
            tmem_st16(kTmem + la + kColDP + wg * 64, pd);
            tmem_st16(kTmem + la + kColDP + wg * 64 + 16, pd + 16);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_ds);
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
        const int smem = 6 * T + 128 + 1024;
        auto kern = radial_attn_bwd_dq_kernel<D>;
        RADIAL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        p.ptr = L->row_ptr;
        p.idx = L->col_idx;
        p.order = L->rorder;
        kern<<<static_cast<unsigned>(items), kThreads, smem, st>>>(tq, tdo, tk, tv, p);
        RADIAL_CUDA_TRY(cudaGetLastError());
    }
    {
        const int smem = 6 * T + 2048 + 128 + 1024;
        auto kern = radial_attn_bwd_dkdv_kernel<D>;  // 6 tiles: K, V, 2 x (Q, dO)
        RADIAL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        p.ptr = L->col_ptr;
        p.idx = L->row_idx;
        p.order = L->corder;
        kern<<<static_cast<unsigned>(items), kThreads, smem, st>>>(tq, tdo, tk, tv, p);
        RADIAL_CUDA_TRY(cudaGetLastError());
    }
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
