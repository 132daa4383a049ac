// radial_cuda.cu -- the C-ABI (include/radial_cuda.h): layout handles,
// argument validation with the reference's error semantics, launches.
#include <atomic>
#include <cstring>
#include <new>
#include <mutex>
#include <string>
#include <thread>
#include <algorithm>
#include <vector>

#include "radial_internal.h"

namespace radial_detail {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

void count_launches(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

void note_use(const radial_layout* Lc, cudaStream_t st) {
    if (!Lc) return;
    auto* L = const_cast<radial_layout*>(Lc);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return;
    }
    std::lock_guard<std::mutex> g(L->use_mu);
    for (auto& u : L->uses)
        if (u.first == st) {
            // a destroyed stream's handle can be reused by a new one: order the new stream after
            // the old event before replacing it, so no earlier use is lost (no-op on one stream)
            cudaStreamWaitEvent(st, u.second, 0);
            cudaEventRecord(u.second, st);
            return;
        }
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return;
    cudaEventRecord(e, st);
    L->uses.emplace_back(st, e);
}

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* where) {
    g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                   ") at " + where;
    return e == cudaErrorMemoryAllocation ? RADIAL_ERR_OOM : RADIAL_ERR_CUDA;
}

int launch_fwd(const void* q, const void* k, const void* v, void* o, float* lse, uint32_t heads,
               uint64_t n, uint32_t D, uint32_t BK, float scale, const radial_layout* L,
               cudaStream_t st, bool token = false, const FwdScatter* sc = nullptr);
int launch_bwd(const void* q, const void* k, const void* v, const void* o, const float* lse,
               const void* dout, void* dq, void* dk, void* dv, uint32_t heads, uint64_t n,
               uint32_t D, float scale, const radial_layout* L, void* workspace, cudaStream_t st);
size_t bwd_workspace_bytes(uint32_t heads, uint64_t n, uint32_t D);

}  // namespace radial_detail

using namespace radial_detail;

namespace {

// Per-device stream on which layouts are freed (stream-ordered, after their last uses).
cudaStream_t free_stream(int dev) {
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        streams[dev] = nullptr;
    }
    return streams[dev];
}

// Drops one reference; the last one frees the device buffers stream-ordered: a private
// stream waits for the layout's recorded uses (one event per stream that launched work on
// it) and releases the buffers with cudaFreeAsync -- no device-wide synchronisation, and
// correct whichever device is current.
void free_layout(radial_layout* L) {
    if (!L) return;
    if (L->refs.fetch_sub(1, std::memory_order_acq_rel) != 1) return;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != L->device) cudaSetDevice(L->device);
    cudaStream_t fs = free_stream(L->device);
    {
        std::lock_guard<std::mutex> g(L->use_mu);
        for (auto& u : L->uses) {
            if (fs) cudaStreamWaitEvent(fs, u.second, 0);
            else cudaEventSynchronize(u.second);
            cudaEventDestroy(u.second);
        }
        L->uses.clear();
    }
    void* ptrs[] = {L->row_ptr, L->col_idx, L->col_ptr, L->row_idx, L->uptr,
                    L->uidx,    L->uorder,  L->rorder,  L->corder,  L->uidx_asc, L->ufull,
                    L->u4ptr,   L->u4idx,   L->u4order};
    for (void* p : ptrs)
        if (p) cudaFreeAsync(p, fs);
    cudaGetLastError();  // teardown at process exit may find the context gone
    if (cur >= 0 && cur != L->device) cudaSetDevice(cur);
    delete L;
}

// A failed build frees what it allocated after the work it queued on `st`.
int bail_layout(radial_layout* L, cudaStream_t st, int rc) {
    note_use(L, st);
    free_layout(L);
    return rc;
}

int check_shape(uint32_t f, uint32_t s, uint32_t B) {
    if (f < 1 || s < 1)
        return fail(RADIAL_ERR_INVALID, "GridShape: frames and tokens_per_frame must be >= 1");
    if (static_cast<uint64_t>(f) * s > (1ull << 32))
        return fail(RADIAL_ERR_INVALID, "GridShape: total tokens exceeds 2^32");
    if (B < 1) return fail(RADIAL_ERR_INVALID, "blockify: block_size must be >= 1");
    const uint64_t rows = (static_cast<uint64_t>(f) * s + B - 1) / B;
    if (rows > 0xffffffffull) return fail(RADIAL_ERR_LENGTH, "block grid exceeds 2^32 rows");
    return RADIAL_OK;
}

// PatternSpec::validate (grid.hpp:118-139): a kind that reads a window must be given one
// (RADIAL_WINDOW_NONE = absent).
int check_pattern(int kind, uint32_t tw, uint32_t sw) {
    static const char* names[] = {"radial", "dense", "spatial", "temporal", "sta", "power", "harmonic"};
    if (kind < 0 || kind > RADIAL_KIND_HARMONIC) return fail(RADIAL_ERR_INVALID, "unknown pattern kind");
    const bool reads_tw = kind == RADIAL_KIND_SPATIAL || kind == RADIAL_KIND_STA;
    const bool reads_sw = kind == RADIAL_KIND_TEMPORAL || kind == RADIAL_KIND_STA;
    if (reads_tw && tw == RADIAL_WINDOW_NONE)
        return fail(RADIAL_ERR_INVALID, std::string(names[kind]) + " pattern requires temporal_window");
    if (reads_sw && sw == RADIAL_WINDOW_NONE)
        return fail(RADIAL_ERR_INVALID, std::string(names[kind]) + " pattern requires spatial_window");
    return RADIAL_OK;
}

int check_attn(const void* q, const void* k, const void* v, const void* o, uint32_t heads,
               uint64_t n, uint32_t D) {
    if (!q || !k || !v || !o) return fail(RADIAL_ERR_INVALID, "masked_attention: null tensor");
    if (heads < 1 || n < 1) return fail(RADIAL_ERR_INVALID, "masked_attention: heads and n must be >= 1");
    if (D != 64 && D != 128)
        return fail(RADIAL_ERR_INVALID, "masked_attention: head_dim must be 64 or 128 on the device path");
    return RADIAL_OK;
}

int check_layout_for_attn(const radial_layout* L, uint64_t n) {
    if (!L) return fail(RADIAL_ERR_INVALID, "masked_attention: null layout");
    if (static_cast<uint64_t>(L->f) * L->s != n)
        return fail(RADIAL_ERR_INVALID, "masked_attention: layout shape mismatch");
    if (L->B != 64 && L->B != 128)
        return fail(RADIAL_ERR_INVALID, "masked_attention: block_size must be 64 or 128 on the device path");
    if (L->first_empty_row >= 0)
        return fail(RADIAL_ERR_EMPTY_ROW,
                    "masked_attention: query row " +
                        std::to_string(static_cast<uint64_t>(L->first_empty_row) * L->B) +
                        " keeps no keys");
    return RADIAL_OK;
}

float resolve_scale(float scale, uint32_t D) {
    return scale > 0.f ? scale : static_cast<float>(1.0 / std::sqrt(static_cast<double>(D)));
}

// Host-buffer forward: H2D q/k/v, kernel (sparse when L != nullptr, else dense),
// D2H o (+ lse), synchronise.  Heads are processed in groups on a three-stage stream
// pipeline -- copy-in of group g+1 and copy-out of group g-1 overlap the kernel of
// group g (H2D and D2H use separate copy engines) -- so end-to-end time approaches
// the kernel time plus one group's transfers.  Heads are independent, so the result
// is identical to one monolithic call.  Device workspace and helper streams are cached
// per thread and device.
struct HostPipe {
    int dev = -1;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    cudaStream_t in = nullptr, out = nullptr, comp[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev;
    ~HostPipe() {
        if (ws) cudaFree(ws);
        for (cudaStream_t s : {in, out, comp[0], comp[1]})
            if (s) cudaStreamDestroy(s);
        for (auto e : ev) cudaEventDestroy(e);
    }
};

thread_local HostPipe t_hp;

int host_fwd_impl(HostPipe& hp, const void* q, const void* k, const void* v, void* o, float* lse, uint32_t heads,
                  uint64_t n, uint32_t head_dim, uint32_t BK, float scale, const radial_layout* L,
                  cudaStream_t st, bool token) {
    int dev = 0;
    RADIAL_CUDA_TRY(cudaGetDevice(&dev));
    const size_t hbytes = static_cast<size_t>(n) * head_dim * 2;  // one head of one tensor
    const size_t tbytes = hbytes * heads;
    const size_t lbytes = static_cast<size_t>(heads) * n * 4;
    const size_t need = 4 * tbytes + lbytes + 4096;
    if (hp.dev != dev) {
        hp.~HostPipe();
        new (&hp) HostPipe();
        hp.dev = dev;
        for (cudaStream_t* s : {&hp.in, &hp.out, &hp.comp[0], &hp.comp[1]})
            RADIAL_CUDA_TRY(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
    }
    if (hp.ws_bytes < need) {
        if (hp.ws) cudaFree(hp.ws);
        hp.ws = nullptr;
        hp.ws_bytes = 0;
        RADIAL_CUDA_TRY(cudaMalloc(&hp.ws, need));
        hp.ws_bytes = need;
    }
    auto* base = static_cast<uint8_t*>(hp.ws);
    auto* dq = base;
    auto* dk = base + tbytes;
    auto* dv = base + 2 * tbytes;
    auto* dO = base + 3 * tbytes;
    float* dl = reinterpret_cast<float*>(base + 4 * tbytes);
    // head groups: a single head first and last (only their copy-in / copy-out is exposed),
    // groups of up to RADIAL_HOST_GROUP_MAX heads in between; consecutive kernels alternate
    // between two streams so one group's tail overlaps the next group's start
    std::vector<uint32_t> gstart;
    {
        const uint32_t mid = heads > 2 ? heads - 2 : 0;
#ifndef RADIAL_HOST_GROUP_MAX  // measured at H33: 1 head per group 70.0 ms, 2: 70.1, 4: 72.4
#define RADIAL_HOST_GROUP_MAX 1
#endif
        const uint32_t gm = std::max<uint32_t>(1, std::min<uint32_t>(RADIAL_HOST_GROUP_MAX, (mid + 4) / 5));
        uint32_t h = 0;
        gstart.push_back(h);
        if (heads > 1) gstart.push_back(h += 1);
        while (h + gm < heads - (heads > 2 ? 1u : 0u)) gstart.push_back(h += gm);
        if (heads > 2 && gstart.back() != heads - 1) gstart.push_back(heads - 1);
        if (gstart.back() >= heads) gstart.pop_back();
    }
    const uint32_t groups = static_cast<uint32_t>(gstart.size());
    while (hp.ev.size() < 3 * static_cast<size_t>(groups) + 1) {
        cudaEvent_t e;
        RADIAL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        hp.ev.push_back(e);
    }
    cudaEvent_t start = hp.ev[3 * groups];
    RADIAL_CUDA_TRY(cudaEventRecord(start, st));  // order after prior work on the caller's stream
    RADIAL_CUDA_TRY(cudaStreamWaitEvent(hp.in, start, 0));
    const float sc = resolve_scale(scale, head_dim);
    for (uint32_t g = 0; g < groups; ++g) {
        const uint32_t h0 = gstart[g], hn = (g + 1 < groups ? gstart[g + 1] : heads) - h0;
        const size_t off = hbytes * h0, len = hbytes * hn;
        cudaEvent_t e_in = hp.ev[3 * g], e_k = hp.ev[3 * g + 1], e_out = hp.ev[3 * g + 2];
        const auto* hq = static_cast<const uint8_t*>(q) + off;
        const auto* hk = static_cast<const uint8_t*>(k) + off;
        const auto* hv = static_cast<const uint8_t*>(v) + off;
        RADIAL_CUDA_TRY(cudaMemcpyAsync(dq + off, hq, len, cudaMemcpyHostToDevice, hp.in));
        RADIAL_CUDA_TRY(cudaMemcpyAsync(dk + off, hk, len, cudaMemcpyHostToDevice, hp.in));
        RADIAL_CUDA_TRY(cudaMemcpyAsync(dv + off, hv, len, cudaMemcpyHostToDevice, hp.in));
        RADIAL_CUDA_TRY(cudaEventRecord(e_in, hp.in));
        cudaStream_t cs = hp.comp[g & 1];  // alternate so one group's tail overlaps the next
        RADIAL_CUDA_TRY(cudaStreamWaitEvent(cs, e_in, 0));
        int rc = launch_fwd(dq + off, dk + off, dv + off, dO + off,
                            lse ? dl + static_cast<size_t>(h0) * n : nullptr, hn, n, head_dim, BK, sc, L, cs,
                            token);
        if (rc) return rc;
        RADIAL_CUDA_TRY(cudaEventRecord(e_k, cs));
        RADIAL_CUDA_TRY(cudaStreamWaitEvent(hp.out, e_k, 0));
        RADIAL_CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(o) + off, dO + off, len, cudaMemcpyDeviceToHost,
                                        hp.out));
        if (lse)
            RADIAL_CUDA_TRY(cudaMemcpyAsync(lse + static_cast<size_t>(h0) * n, dl + static_cast<size_t>(h0) * n,
                                            static_cast<size_t>(hn) * n * 4, cudaMemcpyDeviceToHost, hp.out));
        RADIAL_CUDA_TRY(cudaEventRecord(e_out, hp.out));
    }
    // the caller's stream sees the whole call complete (events timed on it bracket it)
    RADIAL_CUDA_TRY(cudaStreamWaitEvent(st, hp.ev[3 * (groups - 1) + 2], 0));
    (void)lbytes;
    RADIAL_CUDA_TRY(cudaStreamSynchronize(st));
    return RADIAL_OK;
}

// On a mid-pipeline failure the copies already queued still read the caller's q/k/v and write
// o/lse: drain every pipeline stream before returning, so the caller may free its buffers.
int host_fwd(const void* q, const void* k, const void* v, void* o, float* lse, uint32_t heads,
             uint64_t n, uint32_t head_dim, uint32_t BK, float scale, const radial_layout* L,
             cudaStream_t st, bool token = false) {
    const int rc = host_fwd_impl(t_hp, q, k, v, o, lse, heads, n, head_dim, BK, scale, L, st, token);
    if (rc != RADIAL_OK) {
        const std::string msg = g_last_error;
        for (cudaStream_t s : {t_hp.in, t_hp.out, t_hp.comp[0], t_hp.comp[1]})
            if (s) cudaStreamSynchronize(s);
        cudaStreamSynchronize(st);
        cudaGetLastError();
        g_last_error = msg;
    }
    return rc;
}

}  // namespace

extern "C" {

int radial_cuda_abi_version(void) { return RADIAL_CUDA_ABI_VERSION; }
const char* radial_cuda_last_error(void) { return g_last_error.c_str(); }

int radial_cuda_mask_build(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size, int kind,
                           int sink, uint32_t temporal_window, uint32_t spatial_window, void* stream,
                           radial_layout** out) {
    RADIAL_NVTX("radial_cuda_mask_build");
    if (!out) return fail(RADIAL_ERR_INVALID, "null output handle");
    *out = nullptr;
    int rc = check_shape(frames, tokens_per_frame, block_size);
    if (rc) return rc;
    if ((rc = check_pattern(kind, temporal_window, spatial_window))) return rc;
    auto* L = new radial_layout();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaGetDevice(&L->device) != cudaSuccess) {
        delete L;
        return cuda_fail(cudaGetLastError(), "cudaGetDevice");
    }
    L->f = frames;
    L->s = tokens_per_frame;
    L->B = block_size;
    L->R = static_cast<uint32_t>((static_cast<uint64_t>(frames) * tokens_per_frame + block_size - 1) / block_size);
    L->kind = static_cast<uint8_t>(kind);
    L->sink = sink ? 1 : 0;
    L->tw = temporal_window;
    L->sw = spatial_window;
    L->from_pattern = 1;
    if ((rc = build_layout_device(L, st)) || (rc = build_worklists(L, st))) return bail_layout(L, st, rc);
    *out = L;
    return RADIAL_OK;
}

int radial_cuda_layout_from_csr(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size,
                                int kind, int sink, uint32_t grid_rows, const uint64_t* row_ptr,
                                const uint32_t* col_idx, void* stream, radial_layout** out) {
    RADIAL_NVTX("radial_cuda_layout_from_csr");
    if (!out || !row_ptr) return fail(RADIAL_ERR_INVALID, "null argument");
    *out = nullptr;
    int rc = check_shape(frames, tokens_per_frame, block_size);
    if (rc) return rc;
    if (kind < 0 || kind > RADIAL_KIND_HARMONIC) return fail(RADIAL_ERR_INVALID, "unknown pattern kind");
    const uint64_t R = (static_cast<uint64_t>(frames) * tokens_per_frame + block_size - 1) / block_size;
    if (grid_rows != R)
        return fail(RADIAL_ERR_INVALID, "grid_rows: expected " + std::to_string(R) + " for this shape, got " +
                                            std::to_string(grid_rows));
    // validation as in deserialize (block.hpp:274-302), which accepts a nonzero row_ptr[0]:
    // entries before it belong to no row and the uploaded layout drops them
    uint32_t mx = 0, mn = 0xffffffffu;
    int64_t first_empty = -1;
    for (uint64_t I = 0; I < R; ++I) {
        if (row_ptr[I + 1] < row_ptr[I])
            return fail(RADIAL_ERR_INVALID, "row_ptr: not nondecreasing at row " + std::to_string(I + 1));
        const uint64_t len = row_ptr[I + 1] - row_ptr[I];
        mx = std::max<uint32_t>(mx, static_cast<uint32_t>(std::min<uint64_t>(len, 0xffffffffu)));
        mn = std::min<uint32_t>(mn, static_cast<uint32_t>(std::min<uint64_t>(len, 0xffffffffu)));
        if (len == 0 && first_empty < 0) first_empty = static_cast<int64_t>(I);
    }
    if (row_ptr[R] > R * R) return fail(RADIAL_ERR_INVALID, "row_ptr: kept-block count exceeds grid capacity");
    if (row_ptr[R] && !col_idx) return fail(RADIAL_ERR_INVALID, "null col_idx");
    for (uint64_t e = 0; e < row_ptr[R]; ++e)
        if (col_idx[e] >= R)
            return fail(RADIAL_ERR_INVALID, "col_idx: column " + std::to_string(col_idx[e]) +
                                                " out of range at entry " + std::to_string(e));
    for (uint64_t I = 0; I < R; ++I)
        for (uint64_t e = row_ptr[I] + 1; e < row_ptr[I + 1]; ++e)
            if (col_idx[e] <= col_idx[e - 1])
                return fail(RADIAL_ERR_INVALID, "col_idx: not strictly increasing in row " + std::to_string(I));
    const uint64_t base = row_ptr[0], nnz = row_ptr[R] - base;
    std::vector<uint64_t> rp_norm;
    const uint64_t* rp = row_ptr;
    if (base) {
        rp_norm.assign(row_ptr, row_ptr + R + 1);
        for (auto& x : rp_norm) x -= base;
        rp = rp_norm.data();
    }
    auto* L = new radial_layout();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (cudaGetDevice(&L->device) != cudaSuccess) {
        delete L;
        return cuda_fail(cudaGetLastError(), "cudaGetDevice");
    }
    L->f = frames;
    L->s = tokens_per_frame;
    L->B = block_size;
    L->R = static_cast<uint32_t>(R);
    L->kind = static_cast<uint8_t>(kind);
    L->sink = sink ? 1 : 0;
    L->nnz = nnz;
    L->first_empty_row = first_empty;
    L->max_row_len = R ? mx : 0;
    L->min_row_len = R ? mn : 0;
    cudaError_t e;
    if ((e = cudaMallocAsync(&L->row_ptr, sizeof(uint64_t) * (R + 1), st)) != cudaSuccess ||
        (e = cudaMallocAsync(&L->col_idx, sizeof(uint32_t) * std::max<uint64_t>(nnz, 1), st)) != cudaSuccess)
        return bail_layout(L, st, cuda_fail(e, "cudaMallocAsync"));
    if ((e = cudaMemcpyAsync(L->row_ptr, rp, sizeof(uint64_t) * (R + 1), cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return bail_layout(L, st, cuda_fail(e, "cudaMemcpyAsync"));
    if (nnz && (e = cudaMemcpyAsync(L->col_idx, col_idx + base, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice, st)) !=
                   cudaSuccess)
        return bail_layout(L, st, cuda_fail(e, "cudaMemcpyAsync"));
    if ((rc = build_worklists(L, st))) return bail_layout(L, st, rc);
    *out = L;
    return RADIAL_OK;
}

// ---- device layout cache: reference callers pass the same layout once
// per head, so uploads / builds are kept per device and handed out with shared ownership.
namespace {
struct CacheEntry {
    int dev;
    uint32_t f, s, B, tw, sw;
    int kind, sink;
    bool csr;  // uploaded CSR (content compared) vs pattern-built
    std::vector<uint64_t> rp;
    std::vector<uint32_t> ci;
    radial_layout* L;
    uint64_t tick;
};
std::mutex g_cache_mu;
std::vector<CacheEntry> g_cache;
uint64_t g_cache_tick = 0;
constexpr size_t kCacheMax = 16;

bool same_key(const CacheEntry& c, const CacheEntry& k) {
    if (c.dev != k.dev || c.f != k.f || c.s != k.s || c.B != k.B || c.kind != k.kind || c.sink != k.sink ||
        c.csr != k.csr)
        return false;
    if (!k.csr) return c.tw == k.tw && c.sw == k.sw;
    return c.rp.size() == k.rp.size() && c.ci.size() == k.ci.size() &&
           std::memcmp(c.rp.data(), k.rp.data(), c.rp.size() * 8) == 0 &&
           (c.ci.empty() || std::memcmp(c.ci.data(), k.ci.data(), c.ci.size() * 4) == 0);
}

radial_layout* cache_find(const CacheEntry& key) {
    std::lock_guard<std::mutex> g(g_cache_mu);
    for (auto& c : g_cache)
        if (same_key(c, key)) {
            c.tick = ++g_cache_tick;
            c.L->refs.fetch_add(1, std::memory_order_acq_rel);
            return c.L;
        }
    return nullptr;
}

// Inserts a freshly built layout (its one reference becomes the cache's) and returns it with
// an extra reference for the caller; a concurrent insert of the same key wins.
radial_layout* cache_insert(CacheEntry&& key, radial_layout* L) {
    std::vector<radial_layout*> drop;
    radial_layout* ret = nullptr;
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        for (auto& c : g_cache)
            if (same_key(c, key)) {
                ret = c.L;
                drop.push_back(L);
                break;
            }
        if (!ret) {
            key.L = L;
            key.tick = ++g_cache_tick;
            g_cache.push_back(std::move(key));
            ret = L;
            if (g_cache.size() > kCacheMax) {
                auto old = std::min_element(g_cache.begin(), g_cache.end(),
                                            [](const CacheEntry& a, const CacheEntry& b) { return a.tick < b.tick; });
                drop.push_back(old->L);
                g_cache.erase(old);
            }
        }
        ret->refs.fetch_add(1, std::memory_order_acq_rel);
    }
    for (auto* d : drop) free_layout(d);
    return ret;
}
}  // namespace

int radial_cuda_layout_acquire(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size, int kind, int sink,
                               uint32_t temporal_window, uint32_t spatial_window, void* stream, radial_layout** out) {
    if (!out) return fail(RADIAL_ERR_INVALID, "null output handle");
    *out = nullptr;
    CacheEntry key{};
    RADIAL_CUDA_TRY(cudaGetDevice(&key.dev));
    key.f = frames;
    key.s = tokens_per_frame;
    key.B = block_size;
    key.kind = kind;
    key.sink = sink ? 1 : 0;
    key.tw = temporal_window;
    key.sw = spatial_window;
    key.csr = false;
    if ((*out = cache_find(key))) return RADIAL_OK;
    radial_layout* L = nullptr;
    int rc = radial_cuda_mask_build(frames, tokens_per_frame, block_size, kind, sink, temporal_window, spatial_window,
                                    stream, &L);
    if (rc) return rc;
    *out = cache_insert(std::move(key), L);
    return RADIAL_OK;
}

int radial_cuda_layout_acquire_csr(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size, int kind,
                                   int sink, uint32_t grid_rows, const uint64_t* row_ptr, const uint32_t* col_idx,
                                   void* stream, radial_layout** out) {
    if (!out || !row_ptr) return fail(RADIAL_ERR_INVALID, "null argument");
    *out = nullptr;
    int rc = check_shape(frames, tokens_per_frame, block_size);
    if (rc) return rc;
    const uint64_t R = (static_cast<uint64_t>(frames) * tokens_per_frame + block_size - 1) / block_size;
    if (grid_rows != R)
        return radial_cuda_layout_from_csr(frames, tokens_per_frame, block_size, kind, sink, grid_rows, row_ptr,
                                           col_idx, stream, out);  // reports the mismatch
    CacheEntry key{};
    RADIAL_CUDA_TRY(cudaGetDevice(&key.dev));
    key.f = frames;
    key.s = tokens_per_frame;
    key.B = block_size;
    key.kind = kind;
    key.sink = sink ? 1 : 0;
    key.csr = true;
    key.rp.assign(row_ptr, row_ptr + R + 1);
    if (row_ptr[R] && col_idx) key.ci.assign(col_idx, col_idx + row_ptr[R]);
    if ((*out = cache_find(key))) return RADIAL_OK;
    radial_layout* L = nullptr;
    if ((rc = radial_cuda_layout_from_csr(frames, tokens_per_frame, block_size, kind, sink, grid_rows, row_ptr,
                                          col_idx, stream, &L)))
        return rc;
    *out = cache_insert(std::move(key), L);
    return RADIAL_OK;
}

void radial_cuda_layout_cache_clear(void) {
    std::vector<radial_layout*> drop;
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        for (auto& c : g_cache) drop.push_back(c.L);
        g_cache.clear();
    }
    for (auto* d : drop) free_layout(d);
}

uint64_t radial_cuda_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int radial_cuda_layout_info(const radial_layout* L, radial_layout_info* info) {
    if (!L || !info) return fail(RADIAL_ERR_INVALID, "null argument");
    info->frames = L->f;
    info->tokens_per_frame = L->s;
    info->block_size = L->B;
    info->grid_rows = L->R;
    info->kind = L->kind;
    info->sink = L->sink;
    info->kept_blocks = L->nnz;
    info->first_empty_row = L->first_empty_row;
    info->max_row_len = L->max_row_len;
    info->min_row_len = L->min_row_len;
    return RADIAL_OK;
}

int radial_cuda_layout_copy_csr(const radial_layout* L, uint64_t* row_ptr, uint32_t* col_idx) {
    if (!L || !row_ptr) return fail(RADIAL_ERR_INVALID, "null argument");
    RADIAL_CUDA_TRY(cudaMemcpy(row_ptr, L->row_ptr, sizeof(uint64_t) * (static_cast<size_t>(L->R) + 1),
                               cudaMemcpyDeviceToHost));
    if (L->nnz && col_idx)
        RADIAL_CUDA_TRY(cudaMemcpy(col_idx, L->col_idx, sizeof(uint32_t) * L->nnz, cudaMemcpyDeviceToHost));
    return RADIAL_OK;
}

int radial_cuda_layout_copy_csc(const radial_layout* L, uint64_t* col_ptr, uint32_t* row_idx) {
    if (!L || !col_ptr) return fail(RADIAL_ERR_INVALID, "null argument");
    RADIAL_CUDA_TRY(cudaMemcpy(col_ptr, L->col_ptr, sizeof(uint64_t) * (static_cast<size_t>(L->R) + 1),
                               cudaMemcpyDeviceToHost));
    if (L->nnz && row_idx)
        RADIAL_CUDA_TRY(cudaMemcpy(row_idx, L->row_idx, sizeof(uint32_t) * L->nnz, cudaMemcpyDeviceToHost));
    return RADIAL_OK;
}

int radial_cuda_layout_device_csr(const radial_layout* L, const uint64_t** row_ptr,
                                  const uint32_t** col_idx) {
    if (!L) return fail(RADIAL_ERR_INVALID, "null layout");
    if (row_ptr) *row_ptr = L->row_ptr;
    if (col_idx) *col_idx = L->col_idx;
    return RADIAL_OK;
}

void radial_cuda_layout_free(radial_layout* L) { free_layout(L); }

int radial_cuda_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                         uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                         const radial_layout* layout, void* stream) {
    RADIAL_NVTX("radial_cuda_attn_fwd");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if ((rc = check_layout_for_attn(layout, n))) return rc;
    return launch_fwd(q, k, v, o, lse, heads, n, head_dim, layout->B, resolve_scale(scale, head_dim), layout,
                      static_cast<cudaStream_t>(stream));
}

int radial_cuda_attn_fwd_scatter(const void* q, const void* k, const void* v, void* const* o_dst,
                                 uint32_t n_dst, uint32_t head_base, uint32_t heads_full, float* lse,
                                 uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                                 const radial_layout* layout, void* stream) {
    RADIAL_NVTX("radial_cuda_attn_fwd_scatter");
    if (!o_dst || n_dst < 1 || n_dst > 8)
        return fail(RADIAL_ERR_INVALID, "attn_fwd_scatter: 1..8 destination buffers");
    for (uint32_t r = 0; r < n_dst; ++r)
        if (!o_dst[r]) return fail(RADIAL_ERR_INVALID, "attn_fwd_scatter: null destination buffer");
    if (static_cast<uint64_t>(head_base) + heads > heads_full)
        return fail(RADIAL_ERR_INVALID, "attn_fwd_scatter: head_base + heads exceeds heads_full");
    int rc = check_attn(q, k, v, o_dst[0], heads, n, head_dim);
    if (rc) return rc;
    if ((rc = check_layout_for_attn(layout, n))) return rc;
    FwdScatter sc{};
    for (uint32_t r = 0; r < n_dst; ++r) sc.dst[r] = o_dst[r];
    sc.n_dst = n_dst;
    sc.head_base = head_base;
    sc.heads_full = heads_full;
    return launch_fwd(q, k, v, o_dst[0], lse, heads, n, head_dim, layout->B, resolve_scale(scale, head_dim),
                      layout, static_cast<cudaStream_t>(stream), false, &sc);
}

int radial_cuda_attn_fwd_token(const void* q, const void* k, const void* v, void* o, float* lse,
                               uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                               const radial_layout* layout, void* stream) {
    RADIAL_NVTX("radial_cuda_attn_fwd_token");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if ((rc = check_layout_for_attn(layout, n))) return rc;
    if (!layout->from_pattern)
        return fail(RADIAL_ERR_INVALID, "masked_attention: token-exact mode needs a layout built by radial_cuda_mask_build");
    return launch_fwd(q, k, v, o, lse, heads, n, head_dim, layout->B, resolve_scale(scale, head_dim), layout,
                      static_cast<cudaStream_t>(stream), true);
}

int radial_cuda_attn_fwd_dense(const void* q, const void* k, const void* v, void* o, float* lse,
                               uint32_t heads, uint64_t n, uint32_t head_dim, uint32_t block_size,
                               float scale, void* stream) {
    RADIAL_NVTX("radial_cuda_attn_fwd_dense");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if (block_size != 64 && block_size != 128)
        return fail(RADIAL_ERR_INVALID, "dense_attention: block_size must be 64 or 128");
    return launch_fwd(q, k, v, o, lse, heads, n, head_dim, block_size, resolve_scale(scale, head_dim),
                      nullptr, static_cast<cudaStream_t>(stream));
}

int radial_cuda_attn_fwd_host(const void* q, const void* k, const void* v, void* o, float* lse,
                              uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                              const radial_layout* layout, void* stream) {
    RADIAL_NVTX("radial_cuda_attn_fwd_host");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if ((rc = check_layout_for_attn(layout, n))) return rc;
    return host_fwd(q, k, v, o, lse, heads, n, head_dim, layout->B, scale, layout,
                    static_cast<cudaStream_t>(stream));
}

int radial_cuda_attn_fwd_host_multi(const void* q, const void* k, const void* v, void* o, float* lse,
                                    uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                                    uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size, int kind,
                                    int sink, uint32_t temporal_window, uint32_t spatial_window,
                                    const int* devices, int num_devices) {
    RADIAL_NVTX("radial_cuda_attn_fwd_host_multi");
    if (!devices || num_devices < 1) return fail(RADIAL_ERR_INVALID, "attn_fwd_host_multi: no devices");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if ((rc = check_shape(frames, tokens_per_frame, block_size))) return rc;
    if (static_cast<uint64_t>(frames) * tokens_per_frame != n)
        return fail(RADIAL_ERR_INVALID, "masked_attention: layout shape mismatch");
    // one host thread per device, heads split evenly (the split of heads.head_slice); each
    // thread builds the (shared, static) mask on its device and runs the host-buffer pipeline
    // on its slice of the host tensors -- the head-parallel path without torch / torchrun
    const uint32_t ndev = static_cast<uint32_t>(num_devices);
    std::vector<int> rcs(ndev, RADIAL_OK);
    std::vector<std::string> msgs(ndev);
    auto work = [&](uint32_t r) {
        const uint32_t base = heads / ndev, rem = heads % ndev;
        const uint32_t h0 = r * base + std::min(r, rem), hn = base + (r < rem ? 1u : 0u);
        if (hn == 0) return;
        int e = RADIAL_OK;
        radial_layout* L = nullptr;
        if (cudaSetDevice(devices[r]) != cudaSuccess) {
            rcs[r] = fail(RADIAL_ERR_CUDA, "attn_fwd_host_multi: cudaSetDevice failed");
        } else if ((e = radial_cuda_layout_acquire(frames, tokens_per_frame, block_size, kind, sink, temporal_window,
                                                   spatial_window, nullptr, &L)) != RADIAL_OK) {
            rcs[r] = e;
        } else {
            const size_t hb = static_cast<size_t>(n) * head_dim * 2 * h0;
            e = radial_cuda_attn_fwd_host(static_cast<const uint8_t*>(q) + hb, static_cast<const uint8_t*>(k) + hb,
                                          static_cast<const uint8_t*>(v) + hb, static_cast<uint8_t*>(o) + hb,
                                          lse ? lse + static_cast<size_t>(n) * h0 : nullptr, hn, n, head_dim, scale, L,
                                          nullptr);
            rcs[r] = e;
            radial_cuda_layout_free(L);
        }
        if (rcs[r] != RADIAL_OK) msgs[r] = g_last_error;
    };
    int cur = 0;
    cudaGetDevice(&cur);
    std::vector<std::thread> th;
    for (uint32_t r = 1; r < ndev; ++r) th.emplace_back(work, r);
    work(0);
    for (auto& t : th) t.join();
    cudaSetDevice(cur);
    for (uint32_t r = 0; r < ndev; ++r)
        if (rcs[r] != RADIAL_OK) return fail(rcs[r], msgs[r]);
    return RADIAL_OK;
}

int radial_cuda_attn_fwd_token_host(const void* q, const void* k, const void* v, void* o, float* lse,
                                    uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                                    const radial_layout* layout, void* stream) {
    RADIAL_NVTX("radial_cuda_attn_fwd_token_host");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if ((rc = check_layout_for_attn(layout, n))) return rc;
    if (!layout->from_pattern)
        return fail(RADIAL_ERR_INVALID, "masked_attention: token-exact mode needs a layout built by radial_cuda_mask_build");
    return host_fwd(q, k, v, o, lse, heads, n, head_dim, layout->B, scale, layout,
                    static_cast<cudaStream_t>(stream), true);
}

int radial_cuda_attn_fwd_dense_host(const void* q, const void* k, const void* v, void* o, float* lse,
                                    uint32_t heads, uint64_t n, uint32_t head_dim, uint32_t block_size,
                                    float scale, void* stream) {
    RADIAL_NVTX("radial_cuda_attn_fwd_dense_host");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if (block_size != 64 && block_size != 128)
        return fail(RADIAL_ERR_INVALID, "dense_attention: block_size must be 64 or 128");
    return host_fwd(q, k, v, o, lse, heads, n, head_dim, block_size, scale, nullptr,
                    static_cast<cudaStream_t>(stream));
}

size_t radial_cuda_attn_bwd_workspace_size(uint32_t heads, uint64_t n, uint32_t head_dim) {
    return bwd_workspace_bytes(heads, n, head_dim);
}

int radial_cuda_attn_bwd(const void* q, const void* k, const void* v, const void* o, const float* lse,
                         const void* dout, void* dq, void* dk, void* dv, uint32_t heads, uint64_t n,
                         uint32_t head_dim, float scale, const radial_layout* layout, void* workspace,
                         void* stream) {
    RADIAL_NVTX("radial_cuda_attn_bwd");
    int rc = check_attn(q, k, v, o, heads, n, head_dim);
    if (rc) return rc;
    if (!lse || !dout || !dq || !dk || !dv) return fail(RADIAL_ERR_INVALID, "attn_bwd: null tensor");
    if ((rc = check_layout_for_attn(layout, n))) return rc;
    return launch_bwd(q, k, v, o, lse, dout, dq, dk, dv, heads, n, head_dim, resolve_scale(scale, head_dim),
                      layout, workspace, static_cast<cudaStream_t>(stream));
}

int radial_cuda_attention_flops(const radial_layout* L, uint32_t head_dim, uint32_t heads,
                                double* dense_flops, double* sparse_flops, double* reduction) {
    if (!L) return fail(RADIAL_ERR_INVALID, "null layout");
    if (head_dim < 1) return fail(RADIAL_ERR_INVALID, "attention_flops: head_dim must be >= 1");
    if (heads < 1) return fail(RADIAL_ERR_INVALID, "attention_flops: num_heads must be >= 1");
    const double n = static_cast<double>(L->f) * L->s;
    const double B = L->B;
    const double dense = 4.0 * n * n * head_dim * heads;
    const double sparse = 4.0 * static_cast<double>(L->nnz) * B * B * head_dim * heads;
    if (dense_flops) *dense_flops = dense;
    if (sparse_flops) *sparse_flops = sparse;
    if (reduction) *reduction = dense / sparse;
    return RADIAL_OK;
}

double radial_cuda_sparsity(const radial_layout* L) {
    if (!L) return 0.0;
    return 1.0 - static_cast<double>(L->nnz) / (static_cast<double>(L->R) * static_cast<double>(L->R));
}

}  // extern "C"
