// attn_fwd.cu -- K2 (block-sparse radial forward) and K4 (dense comparator).
//
// Replaces radial::masked_attention(const AttentionInstance&, const BlockLayout&)
// (reference attention.hpp:229-270) and radial::dense_attention
// (attention.hpp:141-163): O = softmax(Q K^T * scale restricted to the kept
// B x B blocks) V, computed for all heads in one launch.
//
// Work item = (head, chunk of 256 query rows).  A chunk is two 128-row Q
// tiles that share every K/V tile load; the KV loop runs over the UNION of the
// chunk's query-block lists (entry = J | mask << 28) and each tile skips the
// blocks it does not keep, so FLOPs are exactly the kept blocks.
//
// Warp roles (384 threads, one CTA per SM):
//   warp 0      TMA producer: Q tiles once, then K_j, V_j into one 5-slot ring
//   warp 1      MMA issuer (converged warp, elected lane, four K-steps per asm
//               block): S_t = Q_t K_j^T (SS, both operands K-major in smem) and
//               O_t += P_t V_j (TS: P from TMEM, V MN-major in smem),
//               tcgen05.commit -> mbarriers
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1)
//   warps 4-7   softmax + epilogue for Q tile 0 (one thread per row = TMEM lane)
//   warps 8-11  softmax + epilogue for Q tile 1
// P (bf16) is written over its own S columns with tcgen05.st; the MMA issue
// order (PV_t(j-1) before S_t(j)) makes that alias safe.  Online softmax in
// the exp2 domain with lazy (threshold 8) rescaling of O in TMEM.  Optionally the
// epilogue stores O rows straight into several ranks' full-O buffers (fused
// head-parallel reassembly, radial_cuda_attn_fwd_scatter).
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "mask_rule.cuh"
#include "radial_internal.h"
#include "sm100.cuh"

// setmaxnreg split: producer/MMA warpgroup vs elementwise warpgroups (384 threads x 168 =
// 128 x LO + 256 x HI must hold)
#ifndef RADIAL_FWD_REGS_LO
#define RADIAL_FWD_REGS_LO 40   // the producer / MMA warps issue from uniform registers
#define RADIAL_FWD_REGS_HI 232  // 128 x 40 + 256 x 232 = 384 x 168: no spills in any instantiation
#endif

using namespace radial_sm100;

#ifdef RADIAL_TRACE
// Debug-only event trace (compile with -DRADIAL_TRACE): SM clock stamps for the
// first kTraceCtas CTAs, kTraceEv events per KV step.
__device__ unsigned long long* g_trace = nullptr;
constexpr int kTraceCtas = 4, kTraceSteps = 64, kTraceEv = 24;
#define TRACE(ev, j)                                                                         \
    do {                                                                                     \
        if (trace_base && (j) < kTraceSteps) trace_base[(j) * kTraceEv + (ev)] = clock64();   \
    } while (0)
#else
#define TRACE(ev, j) \
    do {             \
    } while (0)
#endif

namespace {

// MMA issue: warp 1 runs converged and elect.sync picks the issuing lane inside the asm;
// the S and PV MMAs are issued four K-steps per asm block (mma_ss_x4 / mma_ts_x4), so ptxas
// emits back-to-back UTCHMMA (+0.8% per clock over single-lane issue, which costs ~16
// instructions per MMA on the sub-partition the MMA warp shares with two softmax warps).
// -DRADIAL_FWD_LANE0 builds the single-lane variant for comparison.
#ifdef RADIAL_FWD_LANE0
#define FWD_MMA_SS mma_ss_off
#define FWD_MMA_TS mma_ts_off
#define FWD_COMMIT mma_commit
#else
#define RADIAL_FWD_WARP_MMA 1
#define FWD_MMA_SS mma_ss_w
#define FWD_MMA_TS mma_ts_w
#define FWD_COMMIT mma_commit_w
#endif

constexpr int kThreads = 384;
constexpr uint32_t kTmem = 0;   // TMEM base address (checked against tcgen05.alloc)
constexpr int kBQ = 128;        // query rows per tile
// K_j and V_j share one ring of kSlots tiles, in load order K0 V0 K1 V1 ...: tile t = 2j
// (K_j) or 2j + 1 (V_j) lives in slot t % kSlots.  The MMA issue order frees them in the
// same order (K_j after S_B(j), V_j after PV_B(j)), so one ring suffices and every tile
// is prefetched kSlots / 2 steps ahead (the L2 -> SM latency under load is ~1 step).
#ifndef RADIAL_FWD_SLOTS
#define RADIAL_FWD_SLOTS 5
#endif
constexpr int kSlots = RADIAL_FWD_SLOTS;  // the MMA loop is unrolled by kSlots steps (constant slot indices)
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef RADIAL_P_PARTS
#define RADIAL_P_PARTS 2
#endif
// P of a tile is published in kPParts key-column parts, each on its own barrier, so the
// PV MMAs of the first parts run while the later parts' exponentials are computed
// (measured at H33: 2 and 4 parts perform the same; 4 needs block size 128).
constexpr int kPParts = RADIAL_P_PARTS;
#ifndef RADIAL_POLY_PAIRS
#define RADIAL_POLY_PAIRS 0  // measured on B200: MUFU-only is fastest with the current pipeline
#endif
constexpr int kPolyPairs = RADIAL_POLY_PAIRS;  // column pairs per 8 using the polynomial exp2

constexpr int kMaxDst = 8;  // fused all-gather: O rows stored into up to 8 ranks' buffers

#ifndef RADIAL_FWD_L2HINTS
#define RADIAL_FWD_L2HINTS 1  // L2 eviction hints: Q evict-first, K/V evict-last, O streaming stores
#endif

#ifndef RADIAL_TOK_PAIRED
#define RADIAL_TOK_PAIRED 0
#endif
// token-exact mode over the paired work lists with the early S issue (as the block path)
// instead of the ascending lists
constexpr bool kTokPaired = RADIAL_TOK_PAIRED != 0;

struct FwdParams {
    __nv_bfloat16* o;
    float* lse;
    // fused reassembly (C1 without a separate collective): when n_dst > 0 each O row is
    // stored into every destination [heads_full][n][D] buffer (peer GPUs' memory over
    // NVLink / NVSwitch) at head head_base + head, instead of into o
    __nv_bfloat16* dst[kMaxDst];
    uint32_t n_dst, head_base, heads_full;
    const uint64_t* uptr;
    const uint32_t* uidx;
    const uint32_t* order;
    const uint8_t* ufull;  // token-exact mode: per entry, bit t = tile t keeps the whole block
    uint64_t n;
    uint32_t heads, R, C;
    float scale_log2;
    int dense;
    radial_rule::MaskParams rule;  // token-exact mode: the pattern's keep rule
    uint32_t s_inv;                // token-exact mode: floor((2^32 - 1) / s), for key frame = key / s
};

template <int D, int BK>
struct FwdCfg {
    static constexpr int G = 256 / BK;        // query blocks per chunk
    static constexpr int GT = G / 2;          // query blocks per tile
    static constexpr int kAtoms = D / 64;     // 64-column (128 B) swizzle atoms
    static constexpr int kQAtomBytes = kBQ * 128;
    static constexpr int kKVAtomBytes = BK * 128;
    static constexpr int kQBytes = kBQ * D * 2;
    static constexpr int kKVBytes = BK * D * 2;
    static constexpr int kSmemQ = 0;
    static constexpr int kSmemKV = kSmemQ + 2 * kQBytes;          // unified K/V ring
    static constexpr int kSmemBar = kSmemKV + kSlots * kKVBytes;
    static constexpr int kNumBars = 1 + 2 * kSlots + 2 + 2 * kPParts + 2;
    static constexpr int kSmemBytes = kSmemBar + kNumBars * 8 + 16;
    static constexpr int kSmemAlloc = kSmemBytes + 1024;  // slack for 1024 B alignment
    // TMEM columns
    static constexpr uint32_t kColS0 = 0, kColS1 = BK, kColO0 = 2 * BK, kColO1 = 2 * BK + D;
    // always all 512 columns: the only possible allocation base is then column 0, which the
    // MMA operands assume (a smaller request could be placed above another kernel's columns)
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kIdescS = idesc_bf16(128, BK, 0, 0);
    static constexpr uint32_t kIdescO = idesc_bf16(128, D, 0, 1);
};

template <int D, int BK, bool TOKEN>
__global__ void __launch_bounds__(kThreads, 1)
    radial_attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                           const __grid_constant__ CUtensorMap tm_k,
                           const __grid_constant__ CUtensorMap tm_v, const FwdParams p) {
    using Cfg = FwdCfg<D, BK>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kSmemBar);
    uint64_t* bar_q = bars;
    uint64_t* bar_full = bars + 1;
    uint64_t* bar_empty = bar_full + kSlots;
    uint64_t* bar_sfull = bar_empty + kSlots;  // [2]
    uint64_t* bar_pready = bar_sfull + 2;          // [2 tiles][kPParts key parts]
    uint64_t* bar_ofull = bar_pready + 2 * kPParts;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_ofull + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
#ifdef RADIAL_TRACE
    // loaded once: a global load per event would perturb the timeline it measures
    unsigned long long* const trace_base =
        (g_trace && blockIdx.x < kTraceCtas) ? g_trace + blockIdx.x * kTraceSteps * kTraceEv : nullptr;
#endif

    // work item: head-major so the CTAs resident at any time share one head's K/V in L2
    // (K+V of a head = 2 n d bytes = 61 MB at n = 118,800); longest chunks first within
    // windows of 2 x (SM count) consecutive chunks (LPT for a short grid tail, windowed so the
    // resident CTAs' K/V stays in L2 when a head does not: H132, 243 MB per head).
    const uint32_t item = blockIdx.x;
    // The work item's list is (re)derived inside each warp role, after its setmaxnreg: values
    // live across the role split were kept in local memory by ptxas (3 LDL per softmax step).
#define FWD_WORK_ITEM                                                                  \
    const uint32_t head = item / p.C;                                                  \
    const uint32_t chunk = p.order ? __ldg(p.order + item % p.C) : item % p.C;         \
    const uint64_t row0 = static_cast<uint64_t>(chunk) * 256;                          \
    uint64_t ebase = 0;                                                                \
    uint32_t L;                                                                        \
    uint32_t dense_mask = 0;                                                           \
    if (p.dense) {                                                                     \
        L = p.R;                                                                       \
        for (int g = 0; g < Cfg::G; ++g)                                               \
            if (chunk * Cfg::G + g < p.R) dense_mask |= 1u << g;                       \
    } else {                                                                           \
        ebase = __ldg(p.uptr + chunk);                                                 \
        L = static_cast<uint32_t>(__ldg(p.uptr + chunk + 1) - ebase);                  \
    }                                                                                  \
    auto entry = [&](uint32_t j) -> uint32_t {                                         \
        return p.dense ? (j | (dense_mask << 28)) : __ldg(p.uidx + ebase + j);        \
    };                                                                                 \
    (void)head;                                                                        \
    (void)row0

    if (warp == 0 && lane == 0) {
        mbar_init(bar_q, 1);
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_empty[s], 1);
        }
        for (int t = 0; t < 2; ++t) {
            mbar_init(&bar_sfull[t], 1);
            for (int q = 0; q < kPParts; ++q) mbar_init(&bar_pready[kPParts * t + q], 4);  // one arrive per softmax warp
            mbar_init(&bar_ofull[t], 1);
        }
        fence_barrier_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
    }
    if (threadIdx.x == 0) TRACE(22, 0);  // CTA start
    if (warp == 2) tmem_alloc(tmem_slot, Cfg::kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // The CTA allocates all 512 TMEM columns of its SM, so the allocation starts at lane 0 /
    // column 0 by construction; the constant base keeps tcgen05 operands uniform.
    constexpr uint32_t tmem = kTmem;
    // producer / MMA / allocator warpgroup needs few registers (the grouped MMA issue keeps
    // its operands in uniform registers); the two softmax warpgroups hold a 128-column S row
    // each (128 x LO + 256 x HI = 384 x 168, the launch allocation; 72 / 216 was +1% over
    // 104 / 200, and 40 / 232 removes the last spills)
    if (warp < 4) {
        regs_dec<RADIAL_FWD_REGS_LO>();
        FWD_WORK_ITEM;
    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
#if RADIAL_FWD_L2HINTS
            const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
#endif
            mbar_arrive_expect_tx(bar_q, 2 * Cfg::kQBytes);
            for (int t = 0; t < 2; ++t)
                for (int a = 0; a < Cfg::kAtoms; ++a)
#if RADIAL_FWD_L2HINTS
                    // Q is read once: evict-first keeps the L2 for the K/V tiles every chunk re-reads
                    tma_load_3d_hint(smem + Cfg::kSmemQ + t * Cfg::kQBytes + a * Cfg::kQAtomBytes, &tm_q,
                                     bar_q, a * 64, static_cast<int32_t>(row0 + t * kBQ), head, pol_first);
#else
                    tma_load_3d(smem + Cfg::kSmemQ + t * Cfg::kQBytes + a * Cfg::kQAtomBytes, &tm_q,
                                bar_q, a * 64, static_cast<int32_t>(row0 + t * kBQ), head);
#endif
            for (uint32_t t = 0; t < 2 * L; ++t) {
                const int32_t J = static_cast<int32_t>(entry(t >> 1) & 0x0FFFFFFFu);
                const uint32_t slot = t % kSlots;
                mbar_wait(&bar_empty[slot], ((t / kSlots) & 1) ^ 1);
                TRACE(18 + (t & 1), t >> 1);
#ifdef RADIAL_FWD_NO_LOADS
                mbar_arrive(&bar_full[slot]);  // timing experiment: stale K/V tiles
                continue;
#endif
                mbar_arrive_expect_tx(&bar_full[slot], Cfg::kKVBytes);
                uint8_t* dst = smem + Cfg::kSmemKV + slot * Cfg::kKVBytes;
                const CUtensorMap* tm = (t & 1) ? &tm_v : &tm_k;
                for (int a = 0; a < Cfg::kAtoms; ++a)
#if RADIAL_FWD_L2HINTS
                    tma_load_3d_hint(dst + a * Cfg::kKVAtomBytes, tm, &bar_full[slot], a * 64, J * BK, head, pol_last);
#else
                    tma_load_3d(dst + a * Cfg::kKVAtomBytes, tm, &bar_full[slot], a * 64, J * BK, head);
#endif
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // One thread issues.  Every tcgen05 operand is (uniform smem base or the
        // constant TMEM base) + a compile-time offset: the step loop is unrolled by
        // the ring depth so stage indices are constants.  That keeps the operands in
        // uniform registers; a per-MMA register->uniform move would otherwise double
        // the issue cost of each 128x128x16 MMA (measured: 114 vs 64 clk).
#ifdef RADIAL_FWD_LANE0
        if (lane == 0) {
#else
        {  // whole warp, converged: elect.sync inside the MMA / commit wrappers
#endif
            mbar_wait(bar_q, 0);
            tc_fence_after();
            // base descriptors; an MMA's descriptor = base + (byte offset >> 4) (the 14-bit
            // start-address field cannot carry: every offset stays inside 256 KB)
            const uint64_t dq = sdesc_sw128(smem_u32(smem + Cfg::kSmemQ), 16, 1024);
            const uint64_t dk = sdesc_sw128(smem_u32(smem + Cfg::kSmemKV), 16, 1024);
            const uint64_t dv = sdesc_sw128(smem_u32(smem + Cfg::kSmemKV), Cfg::kKVAtomBytes, 1024);
            bool pend0 = false, pend1 = false;
            uint32_t acc0 = 0, acc1 = 0;
            uint32_t pphase0 = 0, pphase1 = 0;
            // warp-converged issue: broadcast lane 0's value so the compiler sees a uniform
            // operand for every branch on it (no divergent / waterfall code paths)
            auto uentry = [&](uint32_t j) -> uint32_t {
#ifdef RADIAL_FWD_LANE0
                return entry(j);
#else
                return __shfl_sync(0xffffffffu, entry(j), 0);
#endif
            };
            uint32_t e_next = L > 0 ? uentry(0) : 0u;
            // tile B's pending PV is issued at step pv1_step (normally the step after its S; two
            // steps after when its S was issued one entry early)
            uint32_t pv1_step = 0;
            bool b_done = false;  // the current entry's S_B was issued early, in the previous step
            // step j: PV_A(j-1), S_A(j), PV_B(j-1), S_B(j); each operand is waited for just
            // before its first use and released right after its last use.
            auto step = [&](uint32_t j, auto PC) {
                constexpr int PH = decltype(PC)::value;        // == j % kSlots
                constexpr int KSL = (2 * PH) % kSlots;          // slot of K_j
                constexpr int VSL = (2 * PH + kSlots - 1) % kSlots;  // slot of V_{j-1}
                uint32_t tf0 = 0, tf1 = 0;
                bool early = false;
                if (j < L) {
                    const uint32_t m = e_next >> 28;  // entry(j), loaded one step ahead
                    if (j + 1 < L) e_next = uentry(j + 1);
                    tf0 = m & ((1u << Cfg::GT) - 1);
                    tf1 = (m >> Cfg::GT) & ((1u << Cfg::GT) - 1);
#ifndef RADIAL_FWD_NO_EARLY_S
                    // a tile-A-only entry followed by a tile-B-only one (the worklist pairs solo
                    // entries up this way): issue the next entry's S_B now, so the two tiles'
                    // softmaxes overlap as in a shared step
                    // (block layouts only: the token-exact path keeps ascending lists, whose
                    // solo entries are rarely adjacent, and measured 4% slower with this logic)
                    if ((!TOKEN || kTokPaired) && tf0 && !tf1 && j + 1 < L) {
                        const uint32_t mn = e_next >> 28;
                        early = !(mn & ((1u << Cfg::GT) - 1)) && ((mn >> Cfg::GT) & ((1u << Cfg::GT) - 1));
                    }
#endif
                }
                // every union entry keeps a block of at least one tile, so V_{j-1} is always
                // consumed; it is waited for and released unconditionally (no TMA in flight
                // into a released slot)
                TRACE(20, j);
                if (j > 0) mbar_wait(&bar_full[VSL], ((2 * j - 1) / kSlots) & 1);
                TRACE(17, j);
                tc_fence_after();
                auto pv = [&](auto TC, uint32_t& acc, uint32_t& pphase) {
                    constexpr int T = decltype(TC)::value;
                    constexpr uint32_t p_col = T ? Cfg::kColS1 : Cfg::kColS0;
                    constexpr uint32_t o_col = T ? Cfg::kColO1 : Cfg::kColO0;

                    static_for<kPParts>([&](auto HC) {
                        constexpr int h = decltype(HC)::value;
                        constexpr int KPP = BK / 16 / kPParts;  // K-steps (16 keys) per part
                        mbar_wait(&bar_pready[kPParts * T + h], pphase);
                        TRACE(8 + 2 * T + (h * 2) / kPParts, j - 1);
                        tc_fence_after();
#if defined(RADIAL_FWD_WARP_MMA) && !defined(RADIAL_FWD_NO_GROUP)
                        if constexpr (KPP == 4 || KPP == 2) {
                            // the part's K-steps in one asm block (elected issue)
                            constexpr int kk0 = h * KPP;
                            if constexpr (KPP == 4)
                                mma_ts_x4<((VSL * Cfg::kKVBytes + kk0 * 16 * 128) >> 4), 128>(
                                    kTmem + o_col, kTmem + p_col + kk0 * 8, dv, Cfg::kIdescO, (acc | kk0) ? 1u : 0u);
                            else
                                mma_ts_x2<((VSL * Cfg::kKVBytes + kk0 * 16 * 128) >> 4), 128>(
                                    kTmem + o_col, kTmem + p_col + kk0 * 8, dv, Cfg::kIdescO, (acc | kk0) ? 1u : 0u);
                        } else
#endif
                        static_for<KPP>([&](auto KI) {
                            constexpr int kk = h * KPP + decltype(KI)::value;
                            FWD_MMA_TS<((VSL * Cfg::kKVBytes + kk * 16 * 128) >> 4)>(
                                kTmem + o_col, kTmem + p_col + kk * 8, dv, Cfg::kIdescO, (acc | kk) ? 1u : 0u);
                        });
                    });
                    pphase ^= 1;
                    acc = 1;
                };
                auto qk = [&](auto TC, auto KC_) {
                    constexpr int T = decltype(TC)::value;
                    constexpr int KSL = decltype(KC_)::value;  // slot of the K tile
                    constexpr uint32_t s_col = T ? Cfg::kColS1 : Cfg::kColS0;

#if defined(RADIAL_FWD_WARP_MMA) && !defined(RADIAL_FWD_NO_GROUP)
                    // one asm block per 64-column atom of d: four K-steps each
                    static_for<Cfg::kAtoms>([&](auto AC) {
                        constexpr int at = decltype(AC)::value;
                        mma_ss_x4<((T * Cfg::kQBytes + at * Cfg::kQAtomBytes) >> 4),
                                  ((KSL * Cfg::kKVBytes + at * Cfg::kKVAtomBytes) >> 4)>(
                            kTmem + s_col, dq, dk, Cfg::kIdescS, at ? 1u : 0u);
                    });
#else
                    static_for<D / 16>([&](auto KC) {
                        constexpr int kk = decltype(KC)::value;
                        constexpr uint32_t off_q = (kk >> 2) * Cfg::kQAtomBytes + (kk & 3) * 32;
                        constexpr uint32_t off_k = (kk >> 2) * Cfg::kKVAtomBytes + (kk & 3) * 32;
                        FWD_MMA_SS<((T * Cfg::kQBytes + off_q) >> 4), ((KSL * Cfg::kKVBytes + off_k) >> 4)>(
                            kTmem + s_col, dq, dk, Cfg::kIdescS, kk ? 1u : 0u);
                    });
#endif
                    FWD_COMMIT(&bar_sfull[T]);
                    TRACE(12 + T, j);
                };
                if (pend0) {
                    pv(std::integral_constant<int, 0>{}, acc0, pphase0);
                    pend0 = false;
                }
                if (j < L) {
                    TRACE(21, j);
                    mbar_wait(&bar_full[KSL], ((2 * j) / kSlots) & 1);
                    TRACE(16, j);
                    tc_fence_after();
                }
                if (tf0) {
                    qk(std::integral_constant<int, 0>{}, std::integral_constant<int, KSL>{});
                    pend0 = true;
                }
                if (pend1 && pv1_step == j) {
                    pv(std::integral_constant<int, 1>{}, acc1, pphase1);
                    pend1 = false;
                }
                if (j > 0) FWD_COMMIT(&bar_empty[VSL]);  // V_{j-1} free once its PVs finish
                if (tf1 && !b_done) {
                    qk(std::integral_constant<int, 1>{}, std::integral_constant<int, KSL>{});
                    pend1 = true;
                    pv1_step = j + 1;
                }
                b_done = false;
                if ((!TOKEN || kTokPaired) && early) {
                    constexpr int KSL1 = (2 * PH + 2) % kSlots;  // slot of K_{j+1}
                    mbar_wait(&bar_full[KSL1], ((2 * j + 2) / kSlots) & 1);
                    tc_fence_after();
                    qk(std::integral_constant<int, 1>{}, std::integral_constant<int, KSL1>{});
                    pend1 = true;
                    pv1_step = j + 2;  // V_{j+1} is read at step j + 2
                    b_done = true;
                }
                if (j < L) FWD_COMMIT(&bar_empty[KSL]);
            };
            for (uint32_t j = 0; j <= L; j += kSlots) {
                static_for<kSlots>([&](auto PC) {
                    if (j + decltype(PC)::value <= L) step(j + decltype(PC)::value, PC);
                });
            }
            FWD_COMMIT(&bar_ofull[0]);
            FWD_COMMIT(&bar_ofull[1]);
        }
    }
    } else {
        regs_inc<RADIAL_FWD_REGS_HI>();
        FWD_WORK_ITEM;
        // ------------------------------------------------------------ softmax
        const int t = (warp - 4) >> 2;                 // Q tile
        const int r = ((warp & 3) << 5) + lane;        // row in tile = TMEM lane
        const uint32_t lane_addr = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t s_addr = tmem + lane_addr + (t ? Cfg::kColS1 : Cfg::kColS0);
        const uint32_t o_addr = tmem + lane_addr + (t ? Cfg::kColO1 : Cfg::kColO0);
        const int my_bit = t * Cfg::GT + r / BK;
        const uint64_t grow = row0 + t * kBQ + r;
        // token coordinates (frame, position) of this row, for the token-exact mode
        const uint32_t tok_i = TOKEN ? static_cast<uint32_t>(grow / p.rule.s) : 0u;
        const uint32_t tok_k = TOKEN ? static_cast<uint32_t>(grow % p.rule.s) : 0u;
        const float sl2 = p.scale_log2;
        float m = -INFINITY, l = 0.f;
        uint32_t sphase = 0;
        uint32_t e_next = L > 0 ? entry(0) : 0u;
        for (uint32_t j = 0; j < L; ++j) {
            const uint32_t e = e_next;  // entry(j), loaded one iteration ahead
            if (j + 1 < L) e_next = entry(j + 1);
            const uint32_t mask = e >> 28;
            if (((mask >> (t * Cfg::GT)) & ((1u << Cfg::GT) - 1)) == 0) continue;
            const uint32_t J = e & 0x0FFFFFFFu;
            // the keep mask of this entry depends only on (row, J): it is built before waiting
            // for S, in the time the warp would otherwise spend waiting (token-exact mode)
            const bool active = (mask >> my_bit) & 1;
            const uint64_t kv0 = static_cast<uint64_t>(J) * BK;
            const int valid = (kv0 + BK <= p.n) ? BK : static_cast<int>(p.n - kv0);
            bool full = active && valid == BK;  // common case: no per-column masking
            uint32_t kmask[BK / 32];
            if constexpr (TOKEN) {
                // token-exact mode (masked_attention(inst, PatternSpec), attention.hpp:184-225):
                // keep exactly the key intervals kept_span(i, k, k, j) of this row's token
                // (i, k) in each key frame j the block overlaps (mask.hpp:238-272).  K1 flags the
                // entries whose whole tile keeps the whole block (ufull): those take the
                // block path's unmasked code with no per-row mask.
#ifdef RADIAL_TOK_NOMASK
                const bool tile_full = true;  // timing hook: token kernel without any masking work
#else
                const bool tile_full = (__ldg(p.ufull + ebase + j) >> t) & 1u;
#endif
#pragma unroll
                for (int w = 0; w < BK / 32; ++w) {
                    const int len = min(max(valid - 32 * w, 0), 32);
                    kmask[w] = tile_full ? (len == 32 ? 0xffffffffu : ((1u << len) - 1u)) : 0u;
                }
                if (tile_full) {
                } else if (active && grow < p.n && p.rule.kind == RADIAL_KIND_POWER) {
                    // power rule (mask.hpp:246-270): key v is kept iff |u - v| is 0 or a power of
                    // two, or (sink) v lies in frame 0
                    const uint64_t v0 = static_cast<uint64_t>(J) * BK, vn = static_cast<uint64_t>(valid);
                    auto set = [&](uint64_t v) {
                        if (v < v0 || v - v0 >= vn) return;
                        const uint32_t c = static_cast<uint32_t>(v - v0);
                        // branch-free per-word update: a data-dependent word index would put
                        // kmask in local memory for the whole loop
#pragma unroll
                        for (int w = 0; w < BK / 32; ++w)
                            kmask[w] |= (1u << (c & 31)) & (0u - static_cast<uint32_t>((c >> 5) == static_cast<uint32_t>(w)));
                    };
                    if (p.rule.sink && v0 < p.rule.s) {
                        const uint32_t hi = static_cast<uint32_t>(min(static_cast<uint64_t>(p.rule.s) - v0, vn));
#pragma unroll
                        for (int w = 0; w < BK / 32; ++w) {
                            const int lw = 32 * w, hw = min(static_cast<int>(hi) - 1, 32 * w + 31);
                            if (lw <= hw) {
                                const int len = hw - lw + 1;
                                kmask[w] |= len == 32 ? 0xffffffffu : ((1u << len) - 1u);
                            }
                        }
                    }
                    set(grow);
                    for (uint64_t t = 1; t < p.n; t <<= 1) {
                        if (grow >= t) set(grow - t);
                        if (grow + t < p.n) set(grow + t);
                    }
                } else if (active && grow < p.n) {
                    const uint32_t v0 = J * BK, v1 = v0 + static_cast<uint32_t>(valid) - 1;
                    // key frame of the block's first key: v0 / s through the host-computed
                    // reciprocal (an under-estimate by at most 2, fixed up), any list order
                    uint32_t jf0 = __umulhi(v0, p.s_inv), fs0 = jf0 * p.rule.s;
                    while (fs0 + p.rule.s <= v0) {
                        ++jf0;
                        fs0 += p.rule.s;
                    }
                    uint32_t fs = fs0;
                    for (uint32_t jf = jf0; fs <= v1; ++jf, fs += p.rule.s) {
                        uint32_t lo, hi;
                        if (!radial_rule::kept_span(p.rule, tok_i, tok_k, tok_k, jf, lo, hi)) continue;
                        const uint32_t a = max(fs + lo, v0) - v0;
                        const uint32_t b = min(fs + hi, v1);
                        if (b < v0 || a > b - v0) continue;
                        const uint32_t bb = b - v0;
#pragma unroll
                        for (int w = 0; w < BK / 32; ++w) {
                            const int lw = max(static_cast<int>(a), 32 * w), hw = min(static_cast<int>(bb), 32 * w + 31);
                            if (lw <= hw) {
                                const int len = hw - lw + 1;
                                kmask[w] |= (len == 32 ? 0xffffffffu : ((1u << len) - 1u)) << (lw - 32 * w);
                            }
                        }
                    }
                }
                bool all = true;
#pragma unroll
                for (int w = 0; w < BK / 32; ++w) all = all && kmask[w] == 0xffffffffu;
#ifdef RADIAL_TOK_NOSELECT
                full = active && (all || kmask[0] != 1u);  // timing hook: build masks, skip applying them
#else
                full = active && all;
#endif
            }
            if ((warp & 3) == 0 && lane == 0) TRACE(4 * t + 0, j);
            mbar_wait(&bar_sfull[t], sphase);
            if ((warp & 3) == 0 && lane == 0) TRACE(4 * t + 1, j);
            sphase ^= 1;
            tc_fence_after();
#ifdef RADIAL_FWD_MMA_ONLY
            // timing experiment: no softmax at all (P = stale TMEM contents); measures the
            // MMA + TMA pipeline alone
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                for (int h = 0; h < kPParts; ++h) mbar_arrive(&bar_pready[kPParts * t + h]);
            continue;
#endif
            float s[BK];
            // first half, wait, then the second half's load overlaps the first half's max; one
            // 64-column tcgen05.ld per half (+1.5% over two 32-column loads)
#if !defined(RADIAL_FWD_LD32)
            if constexpr (BK == 128) {
                uint32_t u[64];
                tmem_ld64(s_addr, u);
#pragma unroll
                for (int x = 0; x < 64; ++x) s[x] = __uint_as_float(u[x]);
            } else
#endif
#pragma unroll
            for (int c = 0; c < BK / 2; c += 32) {
                uint32_t u[32];
                tmem_ld32(s_addr + c, u);
#pragma unroll
                for (int x = 0; x < 32; ++x) s[c + x] = __uint_as_float(u[x]);
            }
            tmem_wait_ld();
            float mh[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) mh[x] = s[x];
#if !defined(RADIAL_FWD_LD32)
            if constexpr (BK == 128) {
                uint32_t u[64];
                tmem_ld64(s_addr + 64, u);
#pragma unroll
                for (int x = 0; x < 64; ++x) s[64 + x] = __uint_as_float(u[x]);
            } else
#endif
#pragma unroll
            for (int c = BK / 2; c < BK; c += 32) {
                uint32_t u[32];
                tmem_ld32(s_addr + c, u);
#pragma unroll
                for (int x = 0; x < 32; ++x) s[c + x] = __uint_as_float(u[x]);
            }
#pragma unroll
            for (int c = 8; c < BK / 2; c += 8)
#pragma unroll
                for (int x = 0; x < 8; ++x) mh[x] = fmaxf(mh[x], s[c + x]);
            tmem_wait_ld();
            if (warp == 4 && lane == 0) TRACE(14, j);
            if (!full) {
                // rare (tail KV block, a row whose query block skips J, or a token-masked
                // entry): mask in place so a single code path follows; masked entries
                // become -inf -> exp2 = 0
                if constexpr (TOKEN) {
                    // kmask already holds active && c < valid: one bit test (LOP3 -> predicate)
                    // and one select per column
#pragma unroll
                    for (int w = 0; w < BK / 32; ++w) kmask[w] = active ? kmask[w] : 0u;
#pragma unroll
                    for (int c = 0; c < BK; ++c) s[c] = (kmask[c >> 5] & (1u << (c & 31))) ? s[c] : -INFINITY;
                } else {
#pragma unroll
                    for (int c = 0; c < BK; ++c) s[c] = (active && c < valid) ? s[c] : -INFINITY;
                }
            }
            // tree reduction: 8 independent chains instead of one 128-long chain
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
            if (warp == 4 && lane == 0) TRACE(15, j);
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
            // rows that never saw a kept block keep m = -inf; all their entries are -inf
            const float mb = (m == -INFINITY) ? 0.f : m;
            // P is produced in two key halves, each published on its own barrier, so
            // the MMA warp starts the first half of PV while the second half's
            // exponentials are still being computed.
            float2 r2a = make_float2(0.f, 0.f), r2b = make_float2(0.f, 0.f);
            const float2 sl = make_float2(sl2, sl2), nm = make_float2(-mb, -mb);
            auto half = [&](int h, auto POLY) {
                constexpr int NP = decltype(POLY)::value;
                constexpr int CP = BK / kPParts;  // columns per part
                static_assert(CP >= 32 && CP % 32 == 0, "P parts must be whole 32-column groups");
                uint32_t pk[CP / 2];
#pragma unroll
                for (int c = h * CP; c < (h + 1) * CP; c += 2) {
                    // store each 32-column group of P as soon as it is packed, so its
                    // tcgen05.st latency overlaps the next group's exponentials
                    if (c > h * CP && (c - h * CP) % 32 == 0)
                        tmem_st16(s_addr + h * (CP / 2) + (c - h * CP) / 2 - 16, pk + (c - h * CP) / 2 - 16);
                    const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), sl, nm);
                    float2 pr;
                    if (((c >> 1) & 7) < NP) {
                        pr = ex2_poly2(x);  // FA4-style FMA-pipe exp2 for a share of columns
                    } else {
                        pr.x = ex2(x.x);
                        pr.y = ex2(x.y);
                    }
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
                if (lane == 0) mbar_arrive(&bar_pready[kPParts * t + h]);
                if ((warp & 3) == 0 && lane == 0) TRACE(4 * t + 2 + (h * 2) / kPParts, j);
            };
#pragma unroll
            for (int h = 0; h < kPParts; ++h) {
                if (kPolyPairs > 0 && full)
                    half(h, std::integral_constant<int, kPolyPairs>{});
                else
                    half(h, std::integral_constant<int, 0>{});
            }
            l += (r2a.x + r2a.y) + (r2b.x + r2b.y);
        }
        // ------------------------------------------------------------ epilogue
        if (warp == 4 && lane == 0) TRACE(22, 2);  // tile 0 softmax done
        mbar_wait(&bar_ofull[t], 0);
        if (warp == 4 && lane == 0) TRACE(22, 3);  // O final
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
                    for (int x = 0; x < 4; ++x) {
#if RADIAL_FWD_L2HINTS
                        __stcs(dst + x, make_uint4(w[4 * x], w[4 * x + 1], w[4 * x + 2], w[4 * x + 3]));  // streaming
#else
                        dst[x] = make_uint4(w[4 * x], w[4 * x + 1], w[4 * x + 2], w[4 * x + 3]);
#endif
                    }
                } else {
                    // every rank's full O: stores to peer GPUs go straight over NVLink while the
                    // other CTAs are still computing (no all-gather after the kernel)
                    for (uint32_t r = 0; r < p.n_dst; ++r) {
                        uint4* dst = reinterpret_cast<uint4*>(p.dst[r] + frow + c);
#pragma unroll
                        for (int x = 0; x < 4; ++x)
                            dst[x] = make_uint4(w[4 * x], w[4 * x + 1], w[4 * x + 2], w[4 * x + 3]);
                    }
                }
            }
        }
        if (p.lse && grow < p.n)
            p.lse[static_cast<uint64_t>(head) * p.n + grow] =
                l > 0.f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(*tmem_slot, Cfg::kTmemCols);
    }
    if (threadIdx.x == 0) TRACE(22, 1);  // CTA end
}
#undef FWD_WORK_ITEM

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

}  // namespace

namespace radial_detail {

// bf16 [heads][n][D] tensor map with a (64 x rows x 1) box, 128 B swizzle,
// zero fill out of bounds (tail rows / keys beyond n).
int make_tmap_bf16_3d(CUtensorMap* m, const void* base, uint64_t n, uint32_t D, uint32_t heads,
                      uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(RADIAL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (reinterpret_cast<uintptr_t>(base) % 16 != 0)
        return fail(RADIAL_ERR_INVALID, "tensor base must be 16-byte aligned");
    cuuint64_t dims[3] = {D, n, heads};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(D) * 2 * n};
    cuuint32_t box[3] = {64, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
#ifndef RADIAL_TMA_L2_PROMO
#define RADIAL_TMA_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
                    RADIAL_TMA_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(RADIAL_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return RADIAL_OK;
}

template <int D, int BK>
int launch_fwd_t(const void* q, const void* k, const void* v, void* o, float* lse,
                 uint32_t heads, uint64_t n, float scale, const radial_layout* L, uint32_t R,
                 bool token, cudaStream_t st, const FwdScatter* sc) {
    using Cfg = FwdCfg<D, BK>;
    CUtensorMap tq, tk, tv;
    int rc;
    if ((rc = make_tmap_bf16_3d(&tq, q, n, D, heads, kBQ))) return rc;
    if ((rc = make_tmap_bf16_3d(&tk, k, n, D, heads, BK))) return rc;
    if ((rc = make_tmap_bf16_3d(&tv, v, n, D, heads, BK))) return rc;
    FwdParams p{};
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
    p.C = (R + Cfg::G - 1) / Cfg::G;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.dense = L == nullptr;
    if (L) {
        p.uptr = L->uptr;
        p.uidx = (token && !kTokPaired && L->uidx_asc) ? L->uidx_asc : L->uidx;
#ifndef RADIAL_FWD_NATURAL_ORDER
        p.order = L->uorder;
#endif
    }
    if (token) {
        p.rule = radial_rule::MaskParams{L->f, L->s, L->B, n, L->kind, L->sink, L->tw, L->sw};
        p.s_inv = 0xffffffffu / L->s;
        p.ufull = L->ufull;
        if (!p.ufull) return fail(RADIAL_ERR_INVALID, "masked_attention: token-exact mode needs a layout built by radial_cuda_mask_build");
    }
    auto kern = token ? radial_attn_fwd_kernel<D, BK, true> : radial_attn_fwd_kernel<D, BK, false>;
    RADIAL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemAlloc));
    const uint64_t items = static_cast<uint64_t>(p.C) * heads;
    if (items == 0) return RADIAL_OK;
    if (items > 0x7fffffffull) return fail(RADIAL_ERR_INVALID, "too many work items");
    kern<<<static_cast<unsigned>(items), kThreads, Cfg::kSmemAlloc, st>>>(tq, tk, tv, p);
    RADIAL_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    note_use(L, st);
    return RADIAL_OK;
}

#ifdef RADIAL_TRACE
extern "C" int radial_cuda_debug_trace(void* buf) {
    RADIAL_CUDA_TRY(cudaMemcpyToSymbol(g_trace, &buf, sizeof(void*)));
    return RADIAL_OK;
}
#endif

int launch_fwd_pair(const void* q, const void* k, const void* v, void* o, float* lse, uint32_t heads, uint64_t n,
                    float scale, const radial_layout* L, cudaStream_t st, const FwdScatter* sc);

// CTA-pair kernel (attn_fwd2.cu): opt-in with RADIAL_FWD_PAIR=1 (measured slower than the
// one-CTA kernel at every BASELINE shape).
bool use_pair_kernel() {
    static const bool on = [] {
        const char* e = getenv("RADIAL_FWD_PAIR");
        return e && e[0] == '1';
    }();
    return on;
}

int launch_fwd(const void* q, const void* k, const void* v, void* o, float* lse, uint32_t heads,
               uint64_t n, uint32_t D, uint32_t BK, float scale, const radial_layout* L,
               cudaStream_t st, bool token, const FwdScatter* sc) {
    const uint64_t R64 = (n + BK - 1) / BK;
    if (R64 >= (1ull << 28)) return fail(RADIAL_ERR_INVALID, "block grid too large for the kernel");
    const uint32_t R = static_cast<uint32_t>(R64);
    if (sc && (sc->n_dst < 1 || sc->n_dst > static_cast<uint32_t>(kMaxDst)))
        return fail(RADIAL_ERR_INVALID, "attn_fwd_scatter: 1..8 destination buffers");
    if (D == 128 && BK == 128 && !token && use_pair_kernel())
        return launch_fwd_pair(q, k, v, o, lse, heads, n, scale, L, st, sc);
    if (D == 128 && BK == 128) return launch_fwd_t<128, 128>(q, k, v, o, lse, heads, n, scale, L, R, token, st, sc);
    if (D == 128 && BK == 64) return launch_fwd_t<128, 64>(q, k, v, o, lse, heads, n, scale, L, R, token, st, sc);
    if (D == 64 && BK == 128) return launch_fwd_t<64, 128>(q, k, v, o, lse, heads, n, scale, L, R, token, st, sc);
    if (D == 64 && BK == 64) return launch_fwd_t<64, 64>(q, k, v, o, lse, heads, n, scale, L, R, token, st, sc);
    return fail(RADIAL_ERR_INVALID, "masked_attention: head_dim must be 64 or 128 and block_size 64 or 128");
}

}  // namespace radial_detail

// Diagnostic hook: cudaFuncGetAttributes of the <128,128> forward kernel
// (numRegs, maxThreadsPerBlock, sharedSizeBytes, maxDynamicSharedSizeBytes, localSizeBytes).
extern "C" int radial_cuda_debug_fwd_attrs(int* out5) {
    cudaFuncAttributes a{};
    RADIAL_CUDA_TRY(cudaFuncGetAttributes(&a, radial_attn_fwd_kernel<128, 128, false>));
    out5[0] = a.numRegs;
    out5[1] = a.maxThreadsPerBlock;
    out5[2] = static_cast<int>(a.sharedSizeBytes);
    out5[3] = a.maxDynamicSharedSizeBytes;
    out5[4] = static_cast<int>(a.localSizeBytes);
    return RADIAL_OK;
}
