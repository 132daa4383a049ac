// C++ drop-in parity program: reference-style callers (radial::blockify,
// radial::masked_attention, ...) compiled against include/radial/*.hpp and linked with
// libradial_cuda.so.  Restates the reference's own test logic
// (tests/test_blocksparse.cpp, tests/test_attention.cpp) with independent oracles
// written here.  Prints "PASS <name>" / "FAIL <name>: why"; exit code = #failures.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "radial/radial.hpp"

using namespace radial;

static int failures = 0;
static void report(bool ok, const std::string& name, const std::string& why = "") {
    std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), ok ? "" : ": ", ok ? "" : why.c_str());
    if (!ok) ++failures;
}

// independent naive block-masked softmax attention in double (test_attention.cpp:19-50 style)
static Matrix naive(const AttentionInstance& inst, const BlockLayout* lay, bool round_bf16) {
    const std::size_t n = inst.shape.total_tokens(), d = inst.head_dim;
    auto rnd = [&](double x) { return round_bf16 ? detail::from_bf16(detail::to_bf16(x)) : x; };
    Matrix out(n, d);
    std::vector<double> lg(n);
    for (std::size_t u = 0; u < n; ++u) {
        double m = -std::numeric_limits<double>::infinity();
        for (std::size_t v = 0; v < n; ++v) {
            const bool keep = !lay || lay->block_at(static_cast<std::uint32_t>(u / lay->block_size),
                                                    static_cast<std::uint32_t>(v / lay->block_size));
            if (!keep) {
                lg[v] = -std::numeric_limits<double>::infinity();
                continue;
            }
            double dot = 0;
            for (std::size_t c = 0; c < d; ++c) dot += rnd(inst.query(u, c)) * rnd(inst.key(v, c));
            lg[v] = dot / std::sqrt(double(d));
            m = std::max(m, lg[v]);
        }
        double den = 0;
        for (std::size_t v = 0; v < n; ++v) {
            if (std::isinf(lg[v])) continue;
            const double w = std::exp(lg[v] - m);
            den += w;
            for (std::size_t c = 0; c < d; ++c) out(u, c) += w * rnd(inst.value(v, c));
        }
        for (std::size_t c = 0; c < d; ++c) out(u, c) /= den;
    }
    return out;
}

static double rel_l2(const Matrix& a, const Matrix& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.data.size(); ++i) {
        num += (a.data[i] - b.data[i]) * (a.data[i] - b.data[i]);
        den += b.data[i] * b.data[i];
    }
    return std::sqrt(num / den);
}

int main() {
    // blockify vs a brute-force token-level painting (test_blocksparse.cpp:18-28 idea)
    {
        bool ok = true;
        for (auto [f, s, B] : {std::tuple{8u, 4u, 4u}, {8u, 4u, 3u}, {5u, 7u, 4u}, {12u, 5u, 8u}, {9u, 3u, 2u},
                               {6u, 6u, 16u}, {16u, 4u, 8u}}) {
            for (bool sink : {true, false}) {
                GridShape shape(f, s);
                auto lay = blockify(shape, PatternSpec::radial(sink), B);
                const std::uint64_t n = shape.total_tokens();
                const std::uint32_t R = grid_rows_for(shape, B);
                std::vector<char> kept(std::size_t{R} * R, 0);
                for (std::uint64_t u = 0; u < n; ++u)
                    for (std::uint64_t v = 0; v < n; ++v) {
                        const std::uint32_t i = u / s, j = v / s, k = u % s, l = v % s;
                        bool keep = sink && j == 0;
                        const std::uint64_t dd = i > j ? i - j : j - i;
                        int e = 0;
                        for (std::uint64_t x = dd > 1 ? dd : 1; x >= 2; x >>= 1) ++e;
                        const double pw = std::ldexp(1.0, e);
                        const std::uint64_t dk = k > l ? k - l : l - k;
                        if (pw <= s && double(dk + 1) <= double(s) / pw) keep = true;
                        const std::uint64_t period = static_cast<std::uint64_t>(std::ceil(pw / s));
                        if (dd % period == 0 && k == l) keep = true;
                        if (keep) kept[(u / B) * R + v / B] = 1;
                    }
                for (std::uint32_t I = 0; I < R; ++I)
                    for (std::uint32_t J = 0; J < R; ++J) ok = ok && (lay.block_at(I, J) == (kept[I * R + J] != 0));
            }
        }
        report(ok, "blockify == brute-force block painting (7 shapes x sink)");
    }
    // pixel KATs at f=256, s=64, B=64 (test_blocksparse.cpp:229-243)
    {
        auto lay = blockify(GridShape(256, 64), PatternSpec::radial(true), 64);
        auto pgm = render_pgm(lay);
        const std::uint8_t* px = pgm.data() + std::string("P5\n256 256\n255\n").size();
        bool ok = px[1 * 256 + 130] == 255 && px[1 * 256 + 129] == 0;
        for (std::uint32_t I = 0; I < 256; ++I) ok = ok && px[I * 256] == 0 && px[I * 256 + I] == 0;
        report(ok, "render_pgm pixel KATs (sink column, diagonal, period-2 drop)");
    }
    // serialization round trip + structured parse errors (test_blocksparse.cpp:142-217)
    {
        auto lay = blockify(GridShape(33, 3600), PatternSpec::radial(true), 128);
        auto bytes = serialize(lay);
        bool ok = bytes.size() == 1565108 && deserialize(bytes) == lay;
        auto bad = bytes;
        bad.push_back(0);
        try {
            deserialize(bad);
            ok = false;
        } catch (const ParseError& e) {
            ok = ok && e.field() == "trailer";
        }
        report(ok, "HunyuanVideo-33 layout: .ramk size 1565108, round trip, trailer error");
        auto rep = attention_flops(lay, 128, 24);
        report(std::abs(rep.sparse_flops / 7.8399e13 - 1) < 1e-4 && std::abs(sparsity(lay) - 0.54879) < 1e-4,
               "attention_flops / sparsity at HunyuanVideo-33");
    }
    // masked_attention over a block layout vs the naive masked oracle on bf16-rounded inputs
    for (auto [f, s, B, d] : {std::tuple{8u, 256u, 64u, 64u}, {3u, 300u, 128u, 128u}}) {
        auto inst = random_instance(GridShape(f, s), d, 42);
        auto lay = blockify(inst.shape, PatternSpec::radial(true), B);
        auto got = masked_attention(inst, lay);
        auto want = naive(inst, &lay, true);
        const double rel = rel_l2(got, want);
        report(rel < 1e-2, "masked_attention f" + std::to_string(f) + " s" + std::to_string(s) + " B" +
                               std::to_string(B) + " d" + std::to_string(d) + " rel-L2 " + std::to_string(rel));
    }
    // token-exact masked_attention(inst, PatternSpec) vs a naive token-masked softmax
    {
        GridShape shape(6, 300);
        auto inst = random_instance(shape, 128, 9);
        auto got = masked_attention(inst, PatternSpec::radial(true));
        // B = 1 layout == the token mask (test_blocksparse.cpp:78-90), built on the GPU
        auto tok = blockify(shape, PatternSpec::radial(true), 1);
        auto want = naive(inst, &tok, true);
        const double rel = rel_l2(got, want);
        report(rel < 1e-2, "masked_attention(inst, PatternSpec) token-exact rel-L2 " + std::to_string(rel));
    }
    // power kind, token-exact (mask.hpp:246-270): the B = 1 power layout is its token mask
    for (bool sink : {false, true}) {
        GridShape shape(5, 60);
        auto inst = random_instance(shape, 64, 17);
        auto got = masked_attention(inst, PatternSpec::power(sink));
        auto tok = blockify(shape, PatternSpec::power(sink), 1);
        const double rel = rel_l2(got, naive(inst, &tok, true));
        report(rel < 1e-2, std::string("masked_attention(inst, power") + (sink ? "+sink" : "") +
                               ") token-exact rel-L2 " + std::to_string(rel));
    }
    // the reference's per-head call pattern (one masked_attention per head, same layout): the
    // device layout cache uploads the layout once, later heads skip the upload and work lists
    {
        GridShape shape(9, 360);
        auto lay = blockify(shape, PatternSpec::radial(true), 128);
        double first_ms = 0, rest_ms = 0, worst = 0;
        for (int h = 0; h < 6; ++h) {
            auto inst = random_instance(shape, 128, 100 + h);
            auto t0 = std::chrono::steady_clock::now();
            auto got = masked_attention(inst, lay);
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            (h == 0 ? first_ms : rest_ms) += ms;
            if (h < 2) worst = std::max(worst, rel_l2(got, naive(inst, &lay, true)));
        }
        std::printf("per-head loop: first call %.2f ms, later calls %.2f ms each\n", first_ms, rest_ms / 5);
        report(worst < 1e-2, "per-head masked_attention loop (cached layout) rel-L2 " + std::to_string(worst));
    }
    // dense_attention vs naive dense (test_attention.cpp:80-83 style)
    {
        auto inst = random_instance(GridShape(4, 100), 128, 123);
        auto rel = rel_l2(dense_attention(inst), naive(inst, nullptr, true));
        report(rel < 1e-2, "dense_attention rel-L2 " + std::to_string(rel));
    }
    // error semantics (test_attention.cpp:143-154, narrowing)
    {
        auto inst = random_instance(GridShape(2, 64), 64, 1);
        BlockLayout empty;
        empty.shape = inst.shape;
        empty.block_size = 64;
        empty.grid_rows = 2;
        empty.row_ptr.assign(3, 0);
        bool ok = false;
        try {
            masked_attention(inst, empty);
        } catch (const std::runtime_error& e) {
            ok = std::string(e.what()).find("row 0") != std::string::npos;
        }
        report(ok, "fully masked rows throw runtime_error naming row 0");
        auto odd = random_instance(GridShape(2, 64), 32, 1);
        ok = false;
        try {
            masked_attention(odd, blockify(odd.shape, PatternSpec::radial(), 64));
        } catch (const std::invalid_argument&) {
            ok = true;
        }
        report(ok, "unsupported head_dim throws invalid_argument");
    }
    std::printf("%d failure(s)\n", failures);
    return failures;
}
