// radial_cli -- the reference command-line front end's `mask`, `stats` and `bench`
// subcommands (/root/reference/proj/tools/radial_cli.cpp) as native C++ over the drop-in
// headers (include/radial/*.hpp) and the C-ABI library: K1 builds the masks, K2 / K4 run the
// bench on the B200.  Same flags (radial_cli.cpp:40-96), JSON keys (:122-133, :143, :400-417)
// and exit codes (0 success, 2 usage or input error, :487-514).  `verify`, `compare` and `fit`
// are the reference's analysis tooling and stay out of scope.
//
//   radial_cli [--pretty] stats --preset hunyuan-509 --head-dim 128
//   radial_cli mask --frames 256 --tokens 64 --block 64 --out m.ramk --pgm m.pgm
//   radial_cli bench --frames 16 --tokens 256 --head-dim 64 --block 64
//
// Device-path narrowing (as in radial/attention.hpp): bench needs head_dim 64 or 128
// (default 64; the reference's CPU default is 32).
#include <charconv>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <iterator>
#include <optional>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "radial/radial.hpp"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ minimal ordered JSON
using JsonValue = std::variant<std::uint64_t, double, std::string>;
using JsonObject = std::vector<std::pair<std::string, JsonValue>>;

std::string json_number(double v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);  // shortest round-trip form
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

bool g_pretty = false;

void emit(const JsonObject& obj) {
    std::string out = "{";
    for (std::size_t i = 0; i < obj.size(); ++i) {
        out += i ? (g_pretty ? ",\n  " : ", ") : (g_pretty ? "\n  " : "");
        out += json_string(obj[i].first) + ": ";
        const JsonValue& v = obj[i].second;
        if (auto* u = std::get_if<std::uint64_t>(&v)) out += std::to_string(*u);
        else if (auto* d = std::get_if<double>(&v)) out += json_number(*d);
        else out += json_string(std::get<std::string>(v));
    }
    out += g_pretty ? "\n}" : "}";
    std::cout << out << "\n";
}

// ------------------------------------------------------------------ argument parsing
struct Args {
    std::vector<std::string> v;
    std::size_t i = 0;
    bool more() const { return i < v.size(); }
    std::string value(const std::string& flag) {
        if (i >= v.size()) throw UsageError(flag + ": missing value");
        return v[i++];
    }
};

std::uint64_t parse_uint(const std::string& flag, const std::string& s) {
    std::uint64_t x = 0;
    auto r = std::from_chars(s.data(), s.data() + s.size(), x);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size()) throw UsageError(flag + ": not a non-negative integer: " + s);
    return x;
}

std::uint32_t parse_u32(const std::string& flag, const std::string& s) {
    const std::uint64_t x = parse_uint(flag, s);
    if (x > 0xffffffffull) throw UsageError(flag + ": value out of range: " + s);
    return static_cast<std::uint32_t>(x);
}

// presets.hpp:34-43 latent geometries (frames, tokens per frame, block size)
struct Preset {
    const char* name;
    std::uint32_t frames, tokens, block;
};
constexpr Preset kPresets[] = {
    {"hunyuan-117", 30, 3600, 128}, {"hunyuan-253", 64, 3600, 128}, {"hunyuan-509", 128, 3600, 128},
    {"wan-69", 18, 3600, 128},      {"wan-161", 41, 3600, 128},     {"mochi-163", 28, 1590, 128},
    {"mochi-331", 56, 1590, 128},   {"mochi-667", 112, 1590, 128},
};

// radial_cli.cpp:29-96: shape / pattern options shared by the subcommands
struct ShapeArgs {
    std::uint32_t frames = 0, tokens = 0, block = 128;
    std::string pattern = "radial";
    std::optional<bool> sink;
    std::optional<std::uint32_t> temporal_window, spatial_window;
    std::string preset;

    bool take(const std::string& flag, Args& a, bool want_preset) {
        if (flag == "--frames") frames = parse_u32(flag, a.value(flag));
        else if (flag == "--tokens") tokens = parse_u32(flag, a.value(flag));
        else if (flag == "--block") block = parse_u32(flag, a.value(flag));
        else if (flag == "--pattern") pattern = a.value(flag);
        else if (flag == "--sink") sink = true;
        else if (flag == "--no-sink") sink = false;
        else if (flag == "--temporal-window") temporal_window = parse_u32(flag, a.value(flag));
        else if (flag == "--spatial-window") spatial_window = parse_u32(flag, a.value(flag));
        else if (want_preset && flag == "--preset") preset = a.value(flag);
        else return false;
        return true;
    }
    const Preset* find_preset() const {
        for (const Preset& p : kPresets)
            if (preset == p.name) return &p;
        throw UsageError("--preset: unknown preset '" + preset + "'");
    }
    radial::GridShape shape() const {
        if (!preset.empty()) {
            const Preset* p = find_preset();
            return {p->frames, p->tokens};
        }
        if (frames == 0 || tokens == 0) throw UsageError("--frames/--tokens: shape required (or use --preset)");
        return {frames, tokens};
    }
    std::uint32_t block_size() const { return preset.empty() ? block : find_preset()->block; }
    radial::PatternSpec spec() const {
        auto kind = radial::parse_kind(pattern);
        if (!kind) throw UsageError("--pattern: unknown pattern '" + pattern + "'");
        radial::PatternSpec s;
        s.kind = *kind;
        s.sink = sink.value_or(*kind == radial::PatternKind::radial);
        s.temporal_window = temporal_window;
        s.spatial_window = spatial_window;
        if (s.reads_temporal_window() && !s.temporal_window)
            throw UsageError("--temporal-window: required for pattern '" + pattern + "'");
        if (s.reads_spatial_window() && !s.spatial_window)
            throw UsageError("--spatial-window: required for pattern '" + pattern + "'");
        return s;
    }
};

void write_file(const std::string& path, const std::vector<std::uint8_t>& bytes) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
    out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw std::runtime_error("failed writing '" + path + "'");
}

std::vector<std::uint8_t> read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open '" + path + "'");
    return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

// radial_cli.cpp:122-133
JsonObject stats_json(const radial::BlockLayout& layout, std::uint32_t head_dim, std::uint32_t heads) {
    const auto fl = radial::attention_flops(layout, head_dim, heads);
    return {{"f", std::uint64_t{layout.shape.frames}},
            {"s", std::uint64_t{layout.shape.tokens_per_frame}},
            {"B", std::uint64_t{layout.block_size}},
            {"kept_blocks", layout.kept_blocks()},
            {"sparsity", radial::sparsity(layout)},
            {"dense_flops", fl.dense_flops},
            {"sparse_flops", fl.sparse_flops},
            {"reduction", fl.reduction}};
}

// ------------------------------------------------------------------ subcommands
int run_mask(Args& a) {  // radial_cli.cpp:137-151
    ShapeArgs sh;
    std::string out, pgm;
    while (a.more()) {
        const std::string f = a.v[a.i++];
        if (sh.take(f, a, true)) continue;
        if (f == "--out") out = a.value(f);
        else if (f == "--pgm") pgm = a.value(f);
        else throw UsageError("mask: unknown option " + f);
    }
    if (out.empty()) throw UsageError("--out is required");
    const auto layout = radial::blockify(sh.shape(), sh.spec(), sh.block_size());  // K1 on the GPU
    write_file(out, radial::serialize(layout));
    if (!pgm.empty()) write_file(pgm, radial::render_pgm(layout));
    emit({{"kept_blocks", layout.kept_blocks()}, {"sparsity", radial::sparsity(layout)}});
    return 0;
}

int run_stats(Args& a) {  // radial_cli.cpp:155-171
    ShapeArgs sh;
    std::string in;
    std::uint32_t head_dim = 64, heads = 1;
    while (a.more()) {
        const std::string f = a.v[a.i++];
        if (sh.take(f, a, true)) continue;
        if (f == "--in") in = a.value(f);
        else if (f == "--head-dim") head_dim = parse_u32(f, a.value(f));
        else if (f == "--heads") heads = parse_u32(f, a.value(f));
        else throw UsageError("stats: unknown option " + f);
    }
    const auto layout =
        in.empty() ? radial::blockify(sh.shape(), sh.spec(), sh.block_size()) : radial::deserialize(read_file(in));
    emit(stats_json(layout, head_dim, heads));
    return 0;
}

int run_bench(Args& a) {  // radial_cli.cpp:382-418: dense vs token-exact masked attention, one head
    ShapeArgs sh;
    std::uint32_t head_dim = 64;
    std::uint64_t seed = 0;
    while (a.more()) {
        const std::string f = a.v[a.i++];
        if (sh.take(f, a, false)) continue;
        if (f == "--head-dim") head_dim = parse_u32(f, a.value(f));
        else if (f == "--seed") seed = parse_uint(f, a.value(f));
        else throw UsageError("bench: unknown option " + f);
    }
    const auto shape = sh.shape();
    const auto pattern = sh.spec();
    const auto inst = radial::random_instance(shape, head_dim, seed);
    using clock = std::chrono::steady_clock;
    (void)radial::masked_attention(inst, pattern);  // warm: context, layout build, kernel load
    const auto t0 = clock::now();
    const auto dense_out = radial::dense_attention(inst);
    const auto t1 = clock::now();
    const auto masked_out = radial::masked_attention(inst, pattern);
    const auto t2 = clock::now();
    const double dense_s = std::chrono::duration<double>(t1 - t0).count();
    const double masked_s = std::chrono::duration<double>(t2 - t1).count();
    const auto fl = radial::attention_flops(radial::blockify(shape, pattern, sh.block), head_dim, 1);
    volatile double keep = dense_out.data[0] + masked_out.data[0];
    (void)keep;
    emit({{"dense_seconds", dense_s},
          {"masked_seconds", masked_s},
          {"speedup", dense_s / masked_s},
          {"flops_reduction", fl.reduction}});
    return 0;
}

const char* kUsage =
    "usage: radial_cli [--pretty] <mask|stats|bench> [options]\n"
    "  shape:   --frames F --tokens S [--block B] [--pattern radial|dense|spatial|temporal|sta|power|harmonic]\n"
    "           [--sink|--no-sink] [--temporal-window W] [--spatial-window W] [--preset NAME]\n"
    "  mask:    shape --out FILE.ramk [--pgm FILE.pgm]\n"
    "  stats:   shape | --in FILE.ramk  [--head-dim D] [--heads H]\n"
    "  bench:   shape [--head-dim 64|128] [--seed N]\n";

}  // namespace

int main(int argc, char** argv) {
    Args a{std::vector<std::string>(argv + 1, argv + argc)};
    try {
        while (a.more() && a.v[a.i].rfind("--", 0) == 0) {
            const std::string f = a.v[a.i++];
            if (f == "--pretty") g_pretty = true;
            else if (f == "--help" || f == "-h") {
                std::cout << kUsage;
                return 0;
            } else throw UsageError("unknown option " + f);
        }
        if (!a.more()) throw UsageError("a subcommand is required");
        const std::string cmd = a.v[a.i++];
        if (cmd == "mask") return run_mask(a);
        if (cmd == "stats") return run_stats(a);
        if (cmd == "bench") return run_bench(a);
        throw UsageError("unknown subcommand '" + cmd + "'");
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n" << kUsage;
        return 2;
    } catch (const std::exception& e) {  // ParseError, invalid_argument, runtime_error: input errors
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
