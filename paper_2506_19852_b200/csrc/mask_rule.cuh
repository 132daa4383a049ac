// mask_rule.cuh -- the reference keep rule on the device, shared by K1 (block
// layouts) and the token-exact forward.  Restates detail::kept_span
// (/root/reference/proj/include/radial/mask.hpp:105-154) for every
// frame-structured kind: for query frame i, query positions [k_lo, k_hi] and key
// frame j, the single kept key-position interval of frame j (or none).
#pragma once

#include <cstdint>

#include "../../include/radial_cuda.h"

namespace radial_rule {

struct MaskParams {
    uint32_t f, s, B;
    uint64_t n;
    int kind, sink;
    uint32_t tw, sw;
};

__host__ __device__ __forceinline__ uint32_t floor_log2_u64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return 63u - __clzll(static_cast<long long>(x));
#else
    return 63u - static_cast<uint32_t>(__builtin_clzll(x));
#endif
}

// mask.hpp:105-154 kept_span for every frame-structured kind.
__host__ __device__ __forceinline__ bool kept_span(const MaskParams& p, uint32_t i, uint32_t k_lo,
                                          uint32_t k_hi, uint32_t j, uint32_t& lo, uint32_t& hi) {
    const uint32_t s = p.s;
    const uint64_t d = i < j ? j - i : i - j;
    auto band = [&](uint32_t sigma) {
        lo = k_lo > sigma ? k_lo - sigma : 0;
        uint64_t h = static_cast<uint64_t>(k_hi) + sigma;
        hi = h >= s ? s - 1 : static_cast<uint32_t>(h);
        return true;
    };
    if (p.sink && j == 0) {
        lo = 0;
        hi = s - 1;
        return true;
    }
    switch (p.kind) {
        case RADIAL_KIND_DENSE:
            lo = 0;
            hi = s - 1;
            return true;
        case RADIAL_KIND_RADIAL: {
            // frame distances are < 2^32: the band test in 32-bit arithmetic (the token-exact
            // forward evaluates this per row and block)
            const uint32_t d32 = static_cast<uint32_t>(d);
#ifdef __CUDA_ARCH__
            const uint32_t e = d32 <= 1 ? 0u : 31u - static_cast<uint32_t>(__clz(static_cast<int>(d32)));
#else
            const uint32_t e = d32 <= 1 ? 0u : 31u - static_cast<uint32_t>(__builtin_clz(d32));
#endif
            if ((1u << e) <= s) return band((s >> e) - 1);  // s / 2^e
            const uint64_t pw = 1ull << e;
            const uint64_t period = (pw + s - 1) / s;
            if (d % period == 0) {
                lo = k_lo;
                hi = k_hi;
                return true;
            }
            return false;
        }
        case RADIAL_KIND_SPATIAL:
            if (d <= p.tw) {
                lo = 0;
                hi = s - 1;
                return true;
            }
            return false;
        case RADIAL_KIND_TEMPORAL:
            return band((p.sw < s - 1 ? p.sw : s - 1));
        case RADIAL_KIND_STA:
            if (d <= p.tw) return band((p.sw < s - 1 ? p.sw : s - 1));
            return false;
        case RADIAL_KIND_HARMONIC: {
            const uint64_t dist = d < 1 ? 1 : d;
            const uint64_t width = s / dist;
            if (width >= 1) return band(static_cast<uint32_t>(width) - 1);
            const uint64_t period = (dist + s - 1) / s;
            if (d % period == 0) {
                lo = k_lo;
                hi = k_hi;
                return true;
            }
            return false;
        }
        default:
            return false;
    }
}

// Every query position k in [k_lo, k_hi] of frame i keeps every key position of
// [l_lo, l_hi] in frame j (token level)?  kept_span's case depends on (i, j) only and, for a
// fixed case, its interval ends are nondecreasing in k (band: [max(k - sigma, 0),
// min(k + sigma, s - 1)]), so the extreme positions decide: the band of k_hi must start by
// l_lo and the band of k_lo must reach l_hi.  Power has no per-frame span (never full here).
__host__ __device__ __forceinline__ bool span_covers(const MaskParams& p, uint32_t i, uint32_t k_lo, uint32_t k_hi,
                                                     uint32_t j, uint32_t l_lo, uint32_t l_hi) {
    if (p.kind == RADIAL_KIND_POWER) return false;
    uint32_t lo_a, hi_a, lo_b, hi_b;
    if (!kept_span(p, i, k_hi, k_hi, j, lo_a, hi_a)) return false;
    if (!kept_span(p, i, k_lo, k_lo, j, lo_b, hi_b)) return false;
    return lo_a <= l_lo && hi_a >= l_hi && lo_b <= l_lo && hi_b >= l_hi;
}

}  // namespace radial_rule
