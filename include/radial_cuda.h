/*
 * radial_cuda.h -- C-ABI of the B200-native radial attention hot path.
 *
 * Plain pointers, sizes and an opaque layout handle; no C++ or torch types.
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj/include/radial/...).  The C++ drop-in headers under
 * include/radial/ re-expose the reference's names on top of this ABI, and
 * INTEGRATION.md shows the ctypes / C++ bindings a maintainer would add.
 *
 * Conventions
 *  - Return value: RADIAL_OK (0) or one of the RADIAL_ERR_* codes below;
 *    radial_cuda_last_error() returns the thread-local message of the last
 *    failure on the calling thread (reference exception text where one
 *    exists, e.g. "masked_attention: query row 0 keeps no keys").
 *  - Device tensors are bf16 [heads][n][head_dim], row-major, contiguous;
 *    lse is fp32 [heads][n] (natural log of the softmax partition).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *    Device-pointer calls are asynchronous on that stream; host-pointer calls
 *    synchronise before returning.
 *  - Reentrant per stream.  Layout handles are immutable after build and may
 *    be shared by any number of streams on their device.
 */
#ifndef RADIAL_CUDA_H
#define RADIAL_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RADIAL_CUDA_ABI_VERSION 2

enum radial_status {
    RADIAL_OK = 0,
    RADIAL_ERR_INVALID = 1,   /* std::invalid_argument in the reference */
    RADIAL_ERR_EMPTY_ROW = 2, /* std::runtime_error "query row u keeps no keys" (attention.hpp:255-258) */
    RADIAL_ERR_CUDA = 3,      /* CUDA runtime / driver failure */
    RADIAL_ERR_OOM = 4,       /* device allocation failed */
    RADIAL_ERR_LENGTH = 5     /* std::length_error (block grid > 2^32 rows, block.hpp:50-52) */
};

/* PatternKind u8 values (grid.hpp:44-52). */
enum radial_kind {
    RADIAL_KIND_RADIAL = 0,
    RADIAL_KIND_DENSE = 1,
    RADIAL_KIND_SPATIAL = 2,
    RADIAL_KIND_TEMPORAL = 3,
    RADIAL_KIND_STA = 4,
    RADIAL_KIND_POWER = 5,
    RADIAL_KIND_HARMONIC = 6
};

/* "window absent" (PatternSpec's empty std::optional, grid.hpp:83-139): a kind that reads a
 * window it was not given fails with RADIAL_ERR_INVALID "<kind> pattern requires
 * temporal_window" / "... spatial_window", as PatternSpec::validate throws.  Kinds that do
 * not read a window ignore the argument. */
#define RADIAL_WINDOW_NONE 0xFFFFFFFFu

typedef struct radial_layout radial_layout; /* opaque device-resident block layout */

typedef struct radial_layout_info {
    uint32_t frames, tokens_per_frame, block_size, grid_rows;
    uint8_t kind, sink;
    uint64_t kept_blocks;   /* nnz of the CSR */
    int64_t first_empty_row; /* first block row with no kept block, -1 if none */
    uint32_t max_row_len, min_row_len;
} radial_layout_info;

int radial_cuda_abi_version(void);
const char* radial_cuda_last_error(void);

/* ---- mask construction: replaces radial::blockify(GridShape, PatternSpec, B)
 *      (block.hpp:59-120, keep rule mask.hpp:105-154).  Builds the CSR
 *      (bit-exact with the reference), its transpose and the kernel work lists
 *      on the device.  temporal_window / spatial_window are read only by the
 *      kinds that need them (grid.hpp:83-139); pass RADIAL_WINDOW_NONE when absent. */
int radial_cuda_mask_build(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size,
                           int kind, int sink, uint32_t temporal_window,
                           uint32_t spatial_window, void* stream, radial_layout** out);

/* Uploads a host CSR (e.g. from radial::deserialize, block.hpp:239-307) and
 * builds the device work lists for it.  Validates the CSR like deserialize (which
 * accepts row_ptr[0] != 0: the entries before it belong to no row; the uploaded layout
 * drops them, so its kept_blocks / copy_csr count only the rows' entries). */
int radial_cuda_layout_from_csr(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size,
                                int kind, int sink, uint32_t grid_rows, const uint64_t* row_ptr,
                                const uint32_t* col_idx, void* stream, radial_layout** out);

/* ---- per-device layout cache (reference callers pass the same layout once per head,
 *      attention.hpp:229): like radial_cuda_mask_build / radial_cuda_layout_from_csr, but
 *      the handle is shared with a cache keyed by (device, shape, block size, pattern) --
 *      for a CSR also by its contents -- so repeated calls skip the upload and the work-list
 *      build.  Release the handle with radial_cuda_layout_free as usual (it drops one
 *      reference).  The cache keeps up to 16 layouts (least recently used evicted). */
int radial_cuda_layout_acquire(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size,
                               int kind, int sink, uint32_t temporal_window, uint32_t spatial_window,
                               void* stream, radial_layout** out);
int radial_cuda_layout_acquire_csr(uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size,
                                   int kind, int sink, uint32_t grid_rows, const uint64_t* row_ptr,
                                   const uint32_t* col_idx, void* stream, radial_layout** out);
void radial_cuda_layout_cache_clear(void);

int radial_cuda_layout_info(const radial_layout* layout, radial_layout_info* info);

/* D2H copy of the CSR: row_ptr u64[grid_rows+1], col_idx u32[kept_blocks]
 * (BlockLayout::row_ptr / col_idx, block.hpp:23-45).  Synchronous. */
int radial_cuda_layout_copy_csr(const radial_layout* layout, uint64_t* row_ptr, uint32_t* col_idx);

/* D2H copy of the transpose (per-KV-block query-block lists, used by the
 * backward): col_ptr u64[grid_rows+1], row_idx u32[kept_blocks]. */
int radial_cuda_layout_copy_csc(const radial_layout* layout, uint64_t* col_ptr, uint32_t* row_idx);

/* Device pointers of the CSR (valid for the handle's lifetime). */
int radial_cuda_layout_device_csr(const radial_layout* layout, const uint64_t** row_ptr,
                                  const uint32_t** col_idx);

/* Drops one reference; the last one frees the device buffers stream-ordered after the
 * work already queued on them (every stream that launched a kernel reading the layout),
 * without synchronising the device.  A layout used inside a captured CUDA graph must
 * outlive the graph. */
void radial_cuda_layout_free(radial_layout* layout);

/* Kernels this library has launched in this process (all entry points, mask builder
 * included) -- the count a benchmark reports for its timed region. */
uint64_t radial_cuda_kernel_launches(void);

/* ---- sparse forward: replaces radial::masked_attention(const AttentionInstance&,
 *      const BlockLayout&) (attention.hpp:229-270) for all heads at once.
 *      head_dim in {64,128}, block_size in {64,128}; scale <= 0 means 1/sqrt(head_dim)
 *      (attention.hpp:130).  lse may be NULL. */
int radial_cuda_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                         uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                         const radial_layout* layout, void* stream);

/* ---- fused head-parallel reassembly (SURVEY 8e, C1 without a separate all-gather):
 *      the forward of radial_cuda_attn_fwd for this rank's `heads` heads, with every O row
 *      stored directly into each of the n_dst (1..8) destination buffers bf16
 *      [heads_full][n][head_dim] at head head_base + h -- typically every rank's full-O
 *      buffer mapped as peer memory (NVLink / NVSwitch P2P stores issued from the kernel
 *      epilogue while other CTAs still compute).  The caller synchronises the ranks
 *      afterwards (e.g. a symmetric-memory barrier).  lse (this call's heads) may be NULL. */
int radial_cuda_attn_fwd_scatter(const void* q, const void* k, const void* v, void* const* o_dst,
                                 uint32_t n_dst, uint32_t head_base, uint32_t heads_full, float* lse,
                                 uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                                 const radial_layout* layout, void* stream);

/* ---- token-exact forward: replaces radial::masked_attention(const AttentionInstance&,
 *      const PatternSpec&) (attention.hpp:184-225).  Iterates the blocks of a layout built
 *      by radial_cuda_mask_build (a superset, block.hpp:59) and keeps exactly the token
 *      pairs of the pattern's rule (mask.hpp:105-154, 238-272), every kind (power: the token
 *      distance rule of mask.hpp:246-270). */
int radial_cuda_attn_fwd_token(const void* q, const void* k, const void* v, void* o, float* lse,
                               uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                               const radial_layout* layout, void* stream);

/* Host-buffer variant of radial_cuda_attn_fwd_token (masked_attention(inst, PatternSpec)'s
 * call shape). */
int radial_cuda_attn_fwd_token_host(const void* q, const void* k, const void* v, void* o, float* lse,
                                    uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                                    const radial_layout* layout, void* stream);

/* ---- dense comparator: replaces radial::dense_attention (attention.hpp:141-163),
 *      same kernel over every KV block; block_size picks the KV tile (64/128). */
int radial_cuda_attn_fwd_dense(const void* q, const void* k, const void* v, void* o, float* lse,
                               uint32_t heads, uint64_t n, uint32_t head_dim, uint32_t block_size,
                               float scale, void* stream);

/* ---- host-buffer forward (the reference call shape: host data in, host data
 *      out).  q/k/v/o are bf16 [heads][n][head_dim] in host memory (pinned or
 *      pageable); copies H2D, runs radial_cuda_attn_fwd, copies O (and lse when
 *      non-NULL) back, synchronises.  Uses a per-thread cached device workspace. */
int radial_cuda_attn_fwd_host(const void* q, const void* k, const void* v, void* o, float* lse,
                              uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                              const radial_layout* layout, void* stream);

/* ---- head-parallel host-buffer forward over several GPUs of this node:
 *      builds the pattern's block layout (radial_cuda_mask_build) on each listed device
 *      and runs radial_cuda_attn_fwd_host on an even split of the heads there, one host
 *      thread per device -- the multi-GPU path for C / C++ callers without torchrun.
 *      Host buffers as for radial_cuda_attn_fwd_host (pinned for overlap); synchronous. */
int radial_cuda_attn_fwd_host_multi(const void* q, const void* k, const void* v, void* o, float* lse,
                                    uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                                    uint32_t frames, uint32_t tokens_per_frame, uint32_t block_size, int kind,
                                    int sink, uint32_t temporal_window, uint32_t spatial_window,
                                    const int* devices, int num_devices);

/* ---- host-buffer dense comparator (dense_attention's call shape, attention.hpp:141). */
int radial_cuda_attn_fwd_dense_host(const void* q, const void* k, const void* v, void* o, float* lse,
                                    uint32_t heads, uint64_t n, uint32_t head_dim, uint32_t block_size,
                                    float scale, void* stream);

/* ---- backward (no reference exists; SPEC.md:8 scopes training out): gradients
 *      of radial_cuda_attn_fwd over the same layout.  o / lse are the forward's
 *      outputs; dq/dk/dv are bf16 [heads][n][head_dim].  workspace: device
 *      scratch of radial_cuda_attn_bwd_workspace_size() bytes. */
size_t radial_cuda_attn_bwd_workspace_size(uint32_t heads, uint64_t n, uint32_t head_dim);
int radial_cuda_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                         const float* lse, const void* dout, void* dq, void* dk, void* dv,
                         uint32_t heads, uint64_t n, uint32_t head_dim, float scale,
                         const radial_layout* layout, void* workspace, void* stream);

/* ---- accounting helpers: replace attention_flops / sparsity (block.hpp:123-148). */
int radial_cuda_attention_flops(const radial_layout* layout, uint32_t head_dim, uint32_t heads,
                                double* dense_flops, double* sparse_flops, double* reduction);
double radial_cuda_sparsity(const radial_layout* layout);

#ifdef __cplusplus
}
#endif
#endif /* RADIAL_CUDA_H */
