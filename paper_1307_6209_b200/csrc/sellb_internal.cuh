// sellb_internal.cuh -- shared internals of libsellb200.so (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/sellb.h"

#include <nvtx3/nvToolsExt.h>

namespace sellb {
// NVTX range around a host entry point (visible in nsys / ncu timelines;
// free when no tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace sellb

// ---------------------------------------------------------------------------
// Device-resident SELL-C-sigma matrix.
//
// HBM layout (one cudaMalloc per array, 256-byte aligned by the allocator):
//   cs   int64[n_chunks+1]   chunk start offsets (formats.py:358-360)
//   cl   int32[n_chunks]     chunk widths, align-rounded (formats.py:351-356)
//   col  int32[slots]        column-major chunk storage, padding = 0
//   val  T[slots]            T = double | float, padding = 0.0
//   rl   int32[n_pad]        stored-row lengths (row_lengths)
//   perm int32[n_rows]       original -> stored
//   order int32[n_pad]       stored -> original (>= n_rows for padding rows)
// Element (stored row p, slot j) lives at cs[p / C] + j*C + p % C
// (formats.py:185-193), so for C = 32 one warp reads 32 consecutive values
// (256 B fp64) and 32 consecutive indices (128 B) per slot: fully coalesced.
// ---------------------------------------------------------------------------
struct sellb_mat {
    int64_t n_rows = 0, n_cols = 0, C = 1, sigma = 1, sigma_eff = 1;
    int64_t n_pad = 0, n_chunks = 0, slots = 0, nnz = 0;
    int32_t dtype = SELLB_F64, device = 0, col_permuted = 0;
    int32_t variant = SELLB_VARIANT_PAD_INCL, max_cl = 0;
    int64_t* cs = nullptr;
    int32_t* cl = nullptr;
    int32_t* col = nullptr;
    void* val = nullptr;
    int32_t* rl = nullptr;
    int32_t* perm = nullptr;
    int32_t* order = nullptr;
    // stored rows longer than long_th, longest first: the SpMV kernel's
    // warp-per-row role (lanes over slots) takes them
    int32_t* long_rows = nullptr;
    int64_t n_long = 0;
    // the pipelined long-row kernel splits long_rows[] into 8-row groups
    // (aligned, same chunk, >= 4 long rows: lanes = 8 rows x 4 slots, loads
    // coalesced per row group) and the remaining rows (warp per row)
    int32_t* long_groups = nullptr;   // first stored row of each group
    int64_t n_groups = 0;
    int32_t* long_rest = nullptr;
    int64_t n_rest = 0;
    // long-row side table: the long_rest rows' values / indices stored
    // contiguously row after row (side_off[k] = start of long_rest[k]), so the
    // warp-per-row role reads them coalesced instead of one 8-byte element per
    // 128-byte DRAM line in the padded SELL layout (SELLB_LONG_SIDE=0: off)
    int64_t* side_off = nullptr;
    int32_t* side_col = nullptr;
    void* side_val = nullptr;
    // packed stored-order copy (sellb_build.cu build_packed, kernel
    // k_spmv_rows MODE 1) for pad-heavy C = 32 layouts: every stored row's
    // entries without padding, row after row (a CRS of the stored rows), so
    // a warp streams 32 rows' entries as one dense run.  The SELL arrays stay
    // the exported layout; the copy only changes which bytes the SpMV reads.
    int64_t* prpt = nullptr;          // n_pad + 1 row offsets into pcol / pval
    int32_t* pcol = nullptr;
    void* pval = nullptr;
    int64_t n_packed = 0;
    // shadow execution layout (sellb_build.cu build_shadow): the same rows
    // re-laid as SELL-32-N (globally sorted by length), used for full-range
    // SpMVs of irregular layouts.  sh_ord_st / sh_ord_or map a shadow row to
    // the caller's stored / original output row (0x7fffffff: none), bit 31 =
    // the row was shorter than its chunk in the caller's layout (the
    // reference's 0 * x[0] padding term)
    sellb_mat* shadow = nullptr;
    // cs / cl / perm / row_lengths / order of a device build in one allocation
    void* meta_slab = nullptr;
    int32_t* sh_ord_st = nullptr;
    int32_t* sh_ord_or = nullptr;
    int32_t long_th = 0x7fffffff;     // chunks wider than this may hold long rows
    int32_t* chunk_th = nullptr;      // per chunk: rows longer than this are long
    // long-row kernel on a side stream, forked from / joined into the
    // caller's stream around the bulk launch (fork/join under long_mu)
    bool long_ready = false;
    cudaStream_t s_long = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::mutex long_mu;
    // end-to-end staging (device x / y for sellb_spmv_host)
    void* x_buf = nullptr;
    void* y_buf = nullptr;
    // pinned (mapped) host mirrors of x / y for callers with pageable
    // vectors (sellb_host.cu): x staged piece by piece by a host thread pool,
    // y written by the kernels straight into hy and copied out per row block
    void* hx = nullptr;
    void* hy = nullptr;
    std::mutex mu;
    // host copy of cs (lazily fetched) for the TMA path's tile sizing
    std::vector<int64_t> h_cs;
    std::mutex hcs_mu;
    // pipelined host path: x pieces H2D / row blocks / y pieces D2H overlap
    static constexpr int kPipe = 16;
    bool pipe_ready = false;
    cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_start = nullptr, ev_x[kPipe] = {}, ev_blk[kPipe] = {};
    int n_pieces = 0;
    int64_t x_off[kPipe + 1] = {};        // column boundaries of the x pieces
    int64_t blk_c[kPipe + 1] = {};        // chunk boundaries of the row blocks
    int blk_need[kPipe] = {};             // last x piece a row block reads
};

namespace sellb {

int set_error(int code, const char* fmt, ...);
void clear_error();

inline size_t vsize(int32_t dtype) { return dtype == SELLB_F32 ? 4 : 8; }

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Keep freed stream-ordered allocations in the device's default pool (the
// default release threshold of 0 hands them back to the driver at every
// synchronisation, turning each temporary into a fresh cudaMalloc).
void trim_pool_memory();
void retain_pool_memory();

// RAII device buffer (stream-ordered free)
struct DBuf {
    void* p = nullptr;
    cudaStream_t s = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { if (p) cudaFreeAsync(p, s); }
    cudaError_t alloc(size_t bytes, cudaStream_t st) {
        s = st;
        retain_pool_memory();
        return cudaMallocAsync(&p, bytes ? bytes : 16, st);
    }
    template <typename T> T* as() const { return static_cast<T*>(p); }
    void* release() { void* q = p; p = nullptr; return q; }
};

// Declared before a build's DBufs (so it is destroyed after them): once the
// stream's frees have completed, trim the retained pool (trim_pool_memory).
struct PoolTrim {
    cudaStream_t st;
    explicit PoolTrim(cudaStream_t s) : st(s) {}
    PoolTrim(const PoolTrim&) = delete;
    PoolTrim& operator=(const PoolTrim&) = delete;
    ~PoolTrim() {
        cudaStreamSynchronize(st);
        cudaGetLastError();
        trim_pool_memory();
    }
};

// Large build temporaries (GBs): plain cudaMalloc / cudaFree.  Growing the
// stream-ordered pool by 16 GB cost ~90 ms on the box (cfg5 shadow build)
// against ~1 ms for cudaMalloc of the same size.
struct BigBuf {
    void* p = nullptr;
    BigBuf() = default;
    BigBuf(const BigBuf&) = delete;
    BigBuf& operator=(const BigBuf&) = delete;
    ~BigBuf() { if (p) cudaFree(p); }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 16); }
    template <typename T> T* as() const { return static_cast<T*>(p); }
};

// launch helpers implemented in sellb_spmv.cu
int launch_spmv(const sellb_mat* m, const void* x, void* y, int64_t c0, int64_t c1,
                int accumulate, int out_order, cudaStream_t st);
int launch_spmv_list(const sellb_mat* m, const int32_t* ids, int64_t n_ids, const void* x,
                     void* y, int accumulate, cudaStream_t st);
int launch_spmv_crs(const int64_t* rpt, const int32_t* col, const void* val, int32_t dtype,
                    const void* x, void* y, int64_t r0, int64_t r1, int accumulate,
                    int unrolled, cudaStream_t st);
// sellb_tma.cu: returns 1 if launched, 0 if the layout does not qualify
int launch_spmv_tma(const sellb_mat* m, const void* x, void* y, int64_t c0, int64_t c1,
                    int accumulate, cudaStream_t st, const int64_t* h_cs);


// sellb_host.cu: host staging of pageable vectors
void host_parallel_copy(void* dst, const void* src, size_t n);
bool is_pinned(const void* p);
int ensure_host_mirror(void** slot, size_t bytes);

int build_packed(sellb_mat* m, cudaStream_t st, int force);
int build_shadow(sellb_mat* m, cudaStream_t st, int force);
void free_shadow(sellb_mat* m);
constexpr int kPackedLong = 128;      // packed copy: longer rows -> warp-per-row role
                                      // (cfg3 sigma=1, threshold 64 / 128 / 256 / 512: 515 / 539 / 512 / 486 GF/s)

inline int64_t grid_for(int64_t n, int threads) { return (n + threads - 1) / threads; }

// process-wide count of compute-path kernel launches (sellb_launch_count)
void count_launches(int n = 1);
long long launch_counter();

}  // namespace sellb

#define SELLB_CU(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return sellb::set_error(SELLB_ERESOURCE, "%s failed: %s (%s:%d)", #call,   \
                                    cudaGetErrorString(e_), __FILE__, __LINE__);        \
    } while (0)
