// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers that call the UNMODIFIED reference library
// (/root/reference/proj/include/radial/*.hpp, header-only C++20) so the
// Python test harness and bench.py's reference arm can drive the reference's
// own code path.  Built by oracle/Makefile into oracle/_ref/libradial_ref.so
// with the reference's Release flags (-O3 -DNDEBUG -std=c++20 -pthread,
// CMakeLists.txt:3-8).  No reference source is copied into this repository:
// the headers are included from /root/reference at build time only, and the
// built .so is what travels to the GPU box.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "radial/radial.hpp"

namespace {
thread_local std::string g_err;

radial::PatternSpec make_pattern(int kind, int sink, uint32_t tw, uint32_t sw) {
    radial::PatternSpec p;
    p.kind = static_cast<radial::PatternKind>(kind);
    p.sink = sink != 0;
    p.temporal_window = tw;
    p.spatial_window = sw;
    return p;
}

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

radial::BlockLayout make_layout(uint32_t f, uint32_t s, uint32_t B, uint32_t R,
                                const uint64_t* row_ptr, const uint32_t* col_idx) {
    radial::BlockLayout lay;
    lay.shape = radial::GridShape(f, s);
    lay.block_size = B;
    lay.grid_rows = R;
    lay.row_ptr.assign(row_ptr, row_ptr + R + 1);
    lay.col_idx.assign(col_idx, col_idx + row_ptr[R]);
    return lay;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// radial::blockify (block.hpp:59) then radial::serialize (block.hpp:223).
// Returns the byte count (writes when out != nullptr and cap suffices), or
// -1 with ref_last_error() set.
int64_t ref_blockify_serialize(uint32_t f, uint32_t s, uint32_t B, int kind, int sink, uint32_t tw,
                               uint32_t sw, uint8_t* out, uint64_t cap) {
    try {
        auto lay = radial::blockify(radial::GridShape(f, s), make_pattern(kind, sink, tw, sw), B);
        auto bytes = radial::serialize(lay);
        if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
        return static_cast<int64_t>(bytes.size());
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// radial::radial_keep (mask.hpp:165)
int ref_radial_keep(uint32_t f, uint32_t s, uint32_t i, uint32_t j, uint32_t k, uint32_t l, int sink) {
    try {
        return radial::radial_keep(i, j, k, l, radial::GridShape(f, s), sink != 0) ? 1 : 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// radial::count_kept (mask.hpp:434)
int64_t ref_count_kept(uint32_t f, uint32_t s, int kind, int sink, uint32_t tw, uint32_t sw) {
    try {
        return static_cast<int64_t>(
            radial::count_kept(radial::GridShape(f, s), make_pattern(kind, sink, tw, sw)));
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// radial::random_instance (attention.hpp:89): q, k, v are n*d doubles.
int ref_random_instance(uint32_t f, uint32_t s, uint32_t d, uint64_t seed, double* q, double* k,
                        double* v) {
    try {
        auto inst = radial::random_instance(radial::GridShape(f, s), d, seed);
        std::memcpy(q, inst.query.data.data(), inst.query.data.size() * sizeof(double));
        std::memcpy(k, inst.key.data.data(), inst.key.data.size() * sizeof(double));
        std::memcpy(v, inst.value.data.data(), inst.value.data.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// radial::masked_attention(const AttentionInstance&, const BlockLayout&)
// (attention.hpp:229).  Return codes: 0 ok, 1 invalid_argument,
// 2 runtime_error (e.g. "query row u keeps no keys"), 3 other.
int ref_masked_attention(uint32_t f, uint32_t s, uint32_t d, const double* q, const double* k,
                         const double* v, uint32_t B, uint32_t R, const uint64_t* row_ptr,
                         const uint32_t* col_idx, double* out) {
    try {
        radial::GridShape shape(f, s);
        const std::size_t n = shape.total_tokens();
        radial::AttentionInstance inst;
        inst.shape = shape;
        inst.head_dim = d;
        inst.query = radial::Matrix(n, d);
        inst.key = radial::Matrix(n, d);
        inst.value = radial::Matrix(n, d);
        std::memcpy(inst.query.data.data(), q, n * d * sizeof(double));
        std::memcpy(inst.key.data.data(), k, n * d * sizeof(double));
        std::memcpy(inst.value.data.data(), v, n * d * sizeof(double));
        auto lay = make_layout(f, s, B, R, row_ptr, col_idx);
        auto o = radial::masked_attention(inst, lay);
        std::memcpy(out, o.data.data(), n * d * sizeof(double));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::runtime_error& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 3);
    }
}

// radial::dense_attention (attention.hpp:141)
int ref_dense_attention(uint32_t f, uint32_t s, uint32_t d, const double* q, const double* k,
                        const double* v, double* out) {
    try {
        radial::GridShape shape(f, s);
        const std::size_t n = shape.total_tokens();
        radial::AttentionInstance inst;
        inst.shape = shape;
        inst.head_dim = d;
        inst.query = radial::Matrix(n, d);
        inst.key = radial::Matrix(n, d);
        inst.value = radial::Matrix(n, d);
        std::memcpy(inst.query.data.data(), q, n * d * sizeof(double));
        std::memcpy(inst.key.data.data(), k, n * d * sizeof(double));
        std::memcpy(inst.value.data.data(), v, n * d * sizeof(double));
        auto o = radial::dense_attention(inst);
        std::memcpy(out, o.data.data(), n * d * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

// radial::attention_flops (block.hpp:137) on a blockified radial layout.
int ref_attention_flops(uint32_t f, uint32_t s, uint32_t B, int sink, uint32_t head_dim,
                        uint32_t heads, double* dense, double* sparse, double* reduction,
                        double* sparsity) {
    try {
        auto lay = radial::blockify(radial::GridShape(f, s), radial::PatternSpec::radial(sink != 0), B);
        auto r = radial::attention_flops(lay, head_dim, heads);
        *dense = r.dense_flops;
        *sparse = r.sparse_flops;
        *reduction = r.reduction;
        *sparsity = radial::sparsity(lay);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 1);
    }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Persistent instances for timing the reference (bench.py's cpu baseline and
// reference arm): the AttentionInstance is built once, outside the timed call.
// ---------------------------------------------------------------------------
extern "C" {

void* ref_instance_create(uint32_t f, uint32_t s, uint32_t d, uint64_t seed) {
    try {
        return new radial::AttentionInstance(radial::random_instance(radial::GridShape(f, s), d, seed));
    } catch (const std::exception& e) {
        fail(e, -1);
        return nullptr;
    }
}

void ref_instance_free(void* inst) { delete static_cast<radial::AttentionInstance*>(inst); }

// One radial::masked_attention(inst, layout) call (attention.hpp:229) on a
// persistent instance; out may be NULL (result discarded).
int ref_masked_attention_inst(void* inst_p, uint32_t B, uint32_t R, const uint64_t* row_ptr,
                              const uint32_t* col_idx, double* out) {
    try {
        auto* inst = static_cast<radial::AttentionInstance*>(inst_p);
        auto lay = make_layout(inst->shape.frames, inst->shape.tokens_per_frame, B, R, row_ptr, col_idx);
        auto o = radial::masked_attention(*inst, lay);
        if (out) std::memcpy(out, o.data.data(), o.data.size() * sizeof(double));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::runtime_error& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 3);
    }
}

}  // extern "C"

// radial::masked_attention(const AttentionInstance&, const PatternSpec&)
// (attention.hpp:184) -- the token-exact reference.
extern "C" int ref_masked_attention_pattern(uint32_t f, uint32_t s, uint32_t d, const double* q,
                                            const double* k, const double* v, int kind, int sink,
                                            uint32_t tw, uint32_t sw, double* out) {
    try {
        radial::GridShape shape(f, s);
        const std::size_t n = shape.total_tokens();
        radial::AttentionInstance inst;
        inst.shape = shape;
        inst.head_dim = d;
        inst.query = radial::Matrix(n, d);
        inst.key = radial::Matrix(n, d);
        inst.value = radial::Matrix(n, d);
        std::memcpy(inst.query.data.data(), q, n * d * sizeof(double));
        std::memcpy(inst.key.data.data(), k, n * d * sizeof(double));
        std::memcpy(inst.value.data.data(), v, n * d * sizeof(double));
        auto o = radial::masked_attention(inst, make_pattern(kind, sink, tw, sw));
        std::memcpy(out, o.data.data(), n * d * sizeof(double));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}
