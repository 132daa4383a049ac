// radial/attention.hpp -- drop-in for the reference's attention API
// (/root/reference/proj/include/radial/attention.hpp:23-270).
//
// masked_attention(inst, layout) and dense_attention(inst) keep their names,
// argument meaning and exceptions but run the B200 kernels (K2 / K4) through
// the host-buffer C-ABI: Q/K/V are rounded to bf16 (RNE), O comes back in
// fp32-accumulated bf16 and is widened to double.  Documented narrowing of the
// device path (std::invalid_argument, no CPU fallback): head_dim in {64, 128},
// block_size in {64, 128}, no explicit-logit instances.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "radial/block.hpp"
#include "radial/grid.hpp"

namespace radial {

// Row-major double matrix (attention.hpp:23-43).
struct Matrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<double> data;

    Matrix() = default;
    Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
    double& operator()(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    double operator()(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    double* row(std::size_t r) { return data.data() + r * cols; }
    const double* row(std::size_t r) const { return data.data() + r * cols; }
    bool empty() const { return data.empty(); }
    bool all_finite() const {
        for (double v : data)
            if (!std::isfinite(v)) return false;
        return true;
    }
};

// One head: Q, K, V of shape n x head_dim (attention.hpp:51-86).
struct AttentionInstance {
    GridShape shape;
    std::uint32_t head_dim = 1;
    Matrix query, key, value;
    Matrix logits;  // explicit-logit instances: not supported by the device path

    bool has_explicit_logits() const { return !logits.empty(); }

    void validate() const {
        const std::size_t n = shape.total_tokens();
        if (value.rows != n || value.cols != head_dim)
            throw std::invalid_argument("AttentionInstance: V must be n x head_dim");
        if (has_explicit_logits()) {
            if (logits.rows != n || logits.cols != n)
                throw std::invalid_argument("AttentionInstance: explicit logits must be n x n");
            if (!logits.all_finite()) throw std::invalid_argument("AttentionInstance: non-finite logit");
        } else {
            if (query.rows != n || query.cols != head_dim || key.rows != n || key.cols != head_dim)
                throw std::invalid_argument("AttentionInstance: Q and K must be n x head_dim");
            if (!query.all_finite() || !key.all_finite())
                throw std::invalid_argument("AttentionInstance: non-finite Q/K entry");
        }
        if (!value.all_finite()) throw std::invalid_argument("AttentionInstance: non-finite V entry");
    }
};

// i.i.d. N(0,1) Q, then K, then V from mt19937_64(seed) (attention.hpp:89-104).
inline AttentionInstance random_instance(const GridShape& shape, std::uint32_t head_dim, std::uint64_t seed) {
    const std::size_t n = shape.total_tokens();
    AttentionInstance inst;
    inst.shape = shape;
    inst.head_dim = head_dim;
    inst.query = Matrix(n, head_dim);
    inst.key = Matrix(n, head_dim);
    inst.value = Matrix(n, head_dim);
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    for (Matrix* m : {&inst.query, &inst.key, &inst.value})
        for (double& v : m->data) v = normal(rng);
    return inst;
}

namespace detail {
inline std::uint16_t to_bf16(double x) {
    float f = static_cast<float>(x);
    std::uint32_t b;
    std::memcpy(&b, &f, 4);
    b += 0x7FFFu + ((b >> 16) & 1u);  // round to nearest even (inputs are finite)
    return static_cast<std::uint16_t>(b >> 16);
}
inline double from_bf16(std::uint16_t h) {
    const std::uint32_t b = std::uint32_t{h} << 16;
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}
inline std::vector<std::uint16_t> pack(const Matrix& m) {
    std::vector<std::uint16_t> out(m.data.size());
    for (std::size_t i = 0; i < out.size(); ++i) out[i] = to_bf16(m.data[i]);
    return out;
}
inline void check_device_instance(const AttentionInstance& inst) {
    inst.validate();
    if (inst.has_explicit_logits())
        throw std::invalid_argument("masked_attention: explicit-logit instances are not supported on the device path");
    if (inst.head_dim != 64 && inst.head_dim != 128)
        throw std::invalid_argument("masked_attention: head_dim must be 64 or 128 on the device path");
}
}  // namespace detail

// radial::masked_attention(inst, layout) (attention.hpp:229-270) on the B200 (K2).
// Throws runtime_error "masked_attention: query row u keeps no keys" for empty rows.
inline Matrix masked_attention(const AttentionInstance& inst, const BlockLayout& layout) {
    detail::check_device_instance(inst);
    if (layout.shape != inst.shape) throw std::invalid_argument("masked_attention: layout shape mismatch");
    const std::size_t n = inst.shape.total_tokens();
    auto q = detail::pack(inst.query), k = detail::pack(inst.key), v = detail::pack(inst.value);
    std::vector<std::uint16_t> o(q.size());
    auto dev = upload_cached(layout);  // per-device cache: one upload for all heads of a call
    detail::check_status(radial_cuda_attn_fwd_host(q.data(), k.data(), v.data(), o.data(), nullptr, 1, n,
                                                   inst.head_dim, 0.f, dev.h, nullptr));
    Matrix out(n, inst.head_dim);
    for (std::size_t i = 0; i < o.size(); ++i) out.data[i] = detail::from_bf16(o[i]);
    return out;
}

// radial::masked_attention(inst, PatternSpec) (attention.hpp:184-225): the token-exact
// mask on the B200 (K2 in token mode over the pattern's 128-block layout), every kind.
inline Matrix masked_attention(const AttentionInstance& inst, const PatternSpec& pattern) {
    detail::check_device_instance(inst);
    pattern.validate();
    const std::size_t n = inst.shape.total_tokens();
    radial_layout* h = nullptr;
    detail::check_status(radial_cuda_layout_acquire(inst.shape.frames, inst.shape.tokens_per_frame, 128,
                                                    static_cast<int>(pattern.kind), pattern.sink ? 1 : 0,
                                                    pattern.temporal_window.value_or(RADIAL_WINDOW_NONE),
                                                    pattern.spatial_window.value_or(RADIAL_WINDOW_NONE), nullptr, &h));
    detail::DeviceLayout dev(h);
    auto q = detail::pack(inst.query), k = detail::pack(inst.key), v = detail::pack(inst.value);
    std::vector<std::uint16_t> o(q.size());
    detail::check_status(radial_cuda_attn_fwd_token_host(q.data(), k.data(), v.data(), o.data(), nullptr, 1, n,
                                                         inst.head_dim, 0.f, dev.h, nullptr));
    Matrix out(n, inst.head_dim);
    for (std::size_t i = 0; i < o.size(); ++i) out.data[i] = detail::from_bf16(o[i]);
    return out;
}

// radial::dense_attention (attention.hpp:141-163) on the B200 (K4 comparator).
inline Matrix dense_attention(const AttentionInstance& inst) {
    detail::check_device_instance(inst);
    const std::size_t n = inst.shape.total_tokens();
    auto q = detail::pack(inst.query), k = detail::pack(inst.key), v = detail::pack(inst.value);
    std::vector<std::uint16_t> o(q.size());
    detail::check_status(radial_cuda_attn_fwd_dense_host(q.data(), k.data(), v.data(), o.data(), nullptr, 1, n,
                                                         inst.head_dim, 128, 0.f, nullptr));
    Matrix out(n, inst.head_dim);
    for (std::size_t i = 0; i < o.size(); ++i) out.data[i] = detail::from_bf16(o[i]);
    return out;
}

}  // namespace radial
