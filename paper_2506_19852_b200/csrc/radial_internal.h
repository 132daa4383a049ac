// radial_internal.h -- host-side internals shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/radial_cuda.h"

// Device-resident block layout.  Everything the kernels need is built once
// per (shape, pattern, block size) and is immutable afterwards.
struct radial_layout {
    int device = 0;
    // shared ownership: radial_cuda_layout_free drops one reference; the device layout cache
    // (radial_cuda_layout_acquire*) holds one of its own
    std::atomic<int> refs{1};
    // streams this layout was last used on (one event each, re-recorded per launch): freeing
    // waits for exactly those uses, stream-ordered, instead of synchronising the device
    std::mutex use_mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
    uint64_t kept_offset = 0;  // row_ptr[0] of an uploaded CSR (deserialize accepts a nonzero start)
    uint32_t f = 1, s = 1, B = 1, R = 0;
    uint8_t kind = 0, sink = 1;
    uint32_t tw = 0, sw = 0;
    int from_pattern = 0;   // built by radial_cuda_mask_build (pattern parameters known)
    uint64_t nnz = 0;
    int64_t first_empty_row = -1;
    uint32_t max_row_len = 0, min_row_len = 0;

    // CSR (BlockLayout::row_ptr / col_idx, bit-exact with the reference)
    uint64_t* row_ptr = nullptr;  // [R+1]
    uint32_t* col_idx = nullptr;  // [nnz]
    // CSC: per-KV-block lists of query blocks (backward)
    uint64_t* col_ptr = nullptr;  // [R+1]
    uint32_t* row_idx = nullptr;  // [nnz]

    // Forward work list: a chunk is 256 query rows = G = 256/B query blocks.
    // uidx entries are J | (mask << 28), mask bit g set iff block chunk*G+g keeps J.
    uint32_t G = 0, C = 0;        // blocks per chunk, number of chunks
    uint64_t* uptr = nullptr;     // [C+1]
    uint32_t* uidx = nullptr;
    uint32_t* uorder = nullptr;   // chunks by descending list length within windows (LPT)
    uint32_t* uidx_asc = nullptr; // the same entries in ascending J (token-exact mode); uidx pairs solo entries
    // CTA-pair forward (block 128): 512-row chunk unions (4 query blocks, mask bits 28-31)
    uint32_t C4 = 0;
    uint64_t* u4ptr = nullptr;    // [C4+1]
    uint32_t* u4idx = nullptr;
    uint32_t* u4order = nullptr;
    uint8_t* ufull = nullptr;     // per uidx_asc entry, bit t: Q tile t keeps every token pair of the
                                  // 128 x B block at token level (token-exact fast path)
    // Backward per-block orders (longest list first): CSR rows (dQ), CSC columns (dK/dV)
    uint32_t* rorder = nullptr;
    uint32_t* corder = nullptr;
};

namespace radial_detail {

// Fused reassembly of O across ranks (radial_cuda_attn_fwd_scatter): destination buffers
// [heads_full][n][D] (one per rank, peer pointers), this call's heads at head_base.
struct FwdScatter {
    void* dst[8];
    uint32_t n_dst, head_base, heads_full;
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

// Records that `L` is read by work queued on `st` (skipped while `st` is capturing a graph:
// layouts used by a captured graph must outlive it).
void note_use(const radial_layout* L, cudaStream_t st);
// Kernel launches issued by this library (radial_cuda_kernel_launches).
void count_launches(uint64_t k);

// mask_build.cu
int build_layout_device(radial_layout* L, cudaStream_t st);
int build_worklists(radial_layout* L, cudaStream_t st);

}  // namespace radial_detail

#define RADIAL_CUDA_TRY(expr)                                                   \
    do {                                                                        \
        cudaError_t e_ = (expr);                                                \
        if (e_ != cudaSuccess) return radial_detail::cuda_fail(e_, #expr);      \
    } while (0)

// NVTX ranges around every C-ABI entry point that launches work (nsys / ncu --nvtx see the
// reference-facing call boundaries); NVTX v3 is header-only and a no-op without a tool.
#ifndef RADIAL_NO_NVTX
#include <nvtx3/nvToolsExt.h>
namespace radial_detail {
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace radial_detail
#define RADIAL_NVTX(name) radial_detail::NvtxRange radial_nvtx_range_(name)
#else
#define RADIAL_NVTX(name) \
    do {                  \
    } while (0)
#endif
