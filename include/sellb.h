/*
 * sellb.h -- C ABI of libsellb200.so, the B200-native SELL-C-sigma build and
 * SpMV library (arXiv 1307.6209).
 *
 * Plain C linkage: pointers, sizes and status codes only.  Every entry point
 * returns 0 on success or a negative status whose class mirrors the
 * reference's exception hierarchy (/root/reference/pkg/src/sellkit/errors.py:4-25);
 * the message is available from sellb_last_error() (thread-local).
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/sellkit):
 *   sellb_build_from_crs      crs_to_sell                  formats.py:295-393
 *   sellb_import              SellMatrix(...) constructor  formats.py:183-251
 *   sellb_info                SellMatrix.nnz/stored_slots  formats.py:253-263
 *   sellb_export              SellMatrix array fields      formats.py:201-206
 *   sellb_spmv                spmv_sell -> spmv_sell_range spmv.py:105-122, _kernels.pyx:65-92
 *   sellb_spmv_host           spmv_sell with host x / y    spmv.py:105-122
 *   sellb_spmv_sell_range_host  kernels-module protocol    _kernels.pyx:65-68 (same arguments)
 *   sellb_spmv_crs_range_host   kernels-module protocol    _kernels.pyx:17-31
 *   sellb_spmv_crs_unrolled_range_host                     _kernels.pyx:34-62
 *   sellb_read_sum / sellb_copy  membench kernels           _kernels.pyx:142-170
 *   sellb_lru_stream_misses   kernels-module protocol    _kernels.pyx:95-139 (cachesim.py:74)
 *   sellb_chunk_occupancy     chunk_occupancy              formats.py:274-282
 *
 * Threading: every entry point is safe to call concurrently from several
 * host threads on disjoint outputs (the reference calls range kernels from a
 * ThreadPoolExecutor, spmv.py:53-73).  Calls that take host buffers
 * synchronise their stream before returning (blocking host-array semantics).
 */
#ifndef SELLB_H
#define SELLB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.py:4-25) */
#define SELLB_OK          0
#define SELLB_EPARAM     -1   /* ParameterError   */
#define SELLB_EDIM       -2   /* DimensionError   */
#define SELLB_ESTRUCT    -3   /* StructuralError  */
#define SELLB_ERESOURCE  -4   /* ResourceError: no device, CUDA error, OOM, NCCL */
#define SELLB_EFORMAT    -5   /* FormatError: text outside the fast parser's grammar */

/* value types */
#define SELLB_F64 0
#define SELLB_F32 1

/* SpMV kernel variants (sellb_set_variant) */
#define SELLB_VARIANT_AUTO      0   /* cost model: skip padding when it saves bytes */
#define SELLB_VARIANT_PAD_SKIP  1   /* one thread per row, stops at its row length   */
#define SELLB_VARIANT_PAD_INCL  2   /* runs every slot up to cl (no row_lengths read) */

/* output order of sellb_spmv / sellb_spmv_host */
#define SELLB_ORDER_STORED   0      /* y[n_rows_padded] in stored (permuted) order */
#define SELLB_ORDER_ORIGINAL 1      /* y[n_rows] in original order: fused unpermute */

typedef struct sellb_mat sellb_mat;   /* opaque, library-owned, device-resident */

typedef struct sellb_info_t {
    int64_t n_rows, n_cols;
    int64_t C, sigma, sigma_eff;
    int64_t n_rows_padded, n_chunks;
    int64_t slots;          /* cs[n_chunks] */
    int64_t nnz;            /* sum(row_lengths) */
    int32_t dtype;          /* SELLB_F64 / SELLB_F32 */
    int32_t device;
    int32_t col_permuted;
    int32_t variant;        /* resolved SELLB_VARIANT_PAD_SKIP / _PAD_INCL */
    int32_t has_row_lengths;
    int32_t max_cl;
    int32_t packed;         /* the SpMV streams the packed chunk copy (C = 32, pad-heavy) */
    int32_t shadow;         /* sigma of the SELL-32 shadow full-range SpMVs run on (0: none) */
} sellb_info_t;

/* How the matrix's long rows are handled (rows the bulk role skips):
 * n_long rows in total, n_groups 8-row groups for the row-group kernel,
 * n_rest rows for the warp-per-row role, side_entries of them copied to the
 * contiguous side table (0 when the side table is off or too large). */
int sellb_long_info(const sellb_mat* m, int64_t* n_long, int64_t* n_groups, int64_t* n_rest,
                    int64_t* side_entries);

/* Bytes of val/col the SpMV streams for this matrix as configured (for the
 * alpha-from-DRAM-bytes model, model.py alpha_from_traffic): every slot of
 * pad-inclusive chunks, the 32-byte (and 64-byte) sectors of bulk rows in
 * chunks read with pad-skip semantics, the long rows' entries (contiguous
 * side table, or one sector per element from the padded layout);
 * extra_bytes = the row_lengths reads.  With the packed copy: (s_v + 4) per
 * nonzero, extra = its row offsets and the chunk widths. */
int sellb_streamed_bytes(const sellb_mat* m, int64_t* matrix_bytes, int64_t* matrix_bytes_64,
                         int64_t* extra_bytes, void* stream);

/* raw device pointers of a matrix (borrowed; valid until sellb_free) */
typedef struct sellb_dev_arrays_t {
    const int64_t* cs;
    const int32_t* cl;
    const int32_t* col;
    const void*    val;
    const int32_t* perm;        /* original -> stored, n_rows          */
    const int32_t* order;       /* stored -> original, n_rows_padded    */
    const int32_t* row_lengths; /* n_rows_padded (NULL if imported without) */
} sellb_dev_arrays_t;

const char* sellb_last_error(void);
int sellb_version(void);
int sellb_device_count(int32_t* n);

/* ---- build / import / export -------------------------------------------- */

/* crs_to_sell (formats.py:295-393) on the device.  rpt[n_rows+1], col[nnz],
 * val[nnz] are host pointers (ptrs_on_device=0) or device pointers on
 * `device` (ptrs_on_device=1).  Bit-exact with the reference's arrays. */
int sellb_build_from_crs(const int64_t* rpt, const int32_t* col, const void* val,
                         int32_t dtype, int64_t n_rows, int64_t n_cols,
                         int32_t C, int64_t sigma, int32_t align_bytes,
                         int32_t permute_cols, int32_t device, void* stream,
                         int32_t ptrs_on_device, sellb_mat** out);

/* Wrap an existing SELL layout (e.g. built by the reference or read from a
 * .sell cache).  perm / row_lengths may be NULL (row_lengths NULL => the
 * pad-inclusive kernel, exactly the reference's loop).  n_slots is the
 * length of the caller's col / val buffers; the reference's SellMatrix
 * invariants (formats.py:210-251) are checked before the matrix is usable:
 * cs[n_chunks] == n_slots, cs[0] == 0, cs[i+1] - cs[i] == C * cl[i],
 * 0 <= col < n_cols, perm a bijection, 0 <= row_lengths <= cl and 0 on
 * padding rows -- SELLB_ESTRUCT otherwise. */
int sellb_import(const int64_t* cs, const int32_t* cl, const int32_t* col,
                 const void* val, const int32_t* perm, const int32_t* row_lengths,
                 int32_t dtype, int64_t n_rows, int64_t n_cols, int32_t C,
                 int64_t sigma, int64_t n_chunks, int64_t n_slots, int32_t col_permuted,
                 int32_t device, void* stream, int32_t ptrs_on_device,
                 sellb_mat** out);

int sellb_info(const sellb_mat* m, sellb_info_t* info);
int sellb_device_arrays(const sellb_mat* m, sellb_dev_arrays_t* out);

/* Copy arrays out (host or device destination); NULL pointers are skipped. */
int sellb_export(const sellb_mat* m, int64_t* cs, int32_t* cl, int32_t* col,
                 void* val, int32_t* perm, int32_t* row_lengths, void* stream,
                 int32_t ptrs_on_device);

/* Copy the arrays of chunks [c0, c1) out (host destination): cs is rebased
 * to start at 0 (c1-c0+1 entries), col/val cover cs[c0]..cs[c1), row_lengths
 * cover stored rows [c0*C, c1*C).  Block-wise parity at sizes the host
 * cannot hold whole (cfg5). */
int sellb_export_range(const sellb_mat* m, int64_t c0, int64_t c1, int64_t* cs, int32_t* cl,
                       int32_t* col, void* val, int32_t* row_lengths);

/* Rebuild row_lengths of an imported matrix on the device the way the
 * reference's .sell cache reader does (io.py:308-321): a stored row's length
 * is its chunk width minus the trailing run of (val == 0.0, col == 0) slots.
 * Enables the pad-skipping kernel and the fused unpermute for the matrix. */
int sellb_infer_row_lengths(sellb_mat* m, void* stream);

int sellb_set_variant(sellb_mat* m, int32_t variant);

/* Packed stored-order copy for pad-heavy C = 32 layouts: 1 builds it (the
 * SpMV then streams every row's entries without padding through the
 * row-run kernel, bit-identical sums), 0 drops it, -1 applies the cost
 * model (packed when the pad-skipping kernel's touched 64-byte sectors
 * exceed the packed bytes by more than SELLB_PACKED_MIN_GAIN, default 1.3).
 * Every build applies the cost model unless SELLB_PACKED=0 / 1 forces it. */
int sellb_set_packed(sellb_mat* m, int32_t mode);

/* Shadow execution layout for irregular or C != 32 layouts: 1 builds it (a device copy
 * of the stored rows re-laid as SELL-32-N -- sorted by length over the
 * whole matrix -- when x is at most SELLB_SHADOW_X_MAX bytes (default
 * 48 MiB, i.e. x stays in L2), else as SELL-32-512, which keeps a chunk's
 * rows neighbours and their x lines shared; every full-range sellb_spmv then
 * runs on it and scatters each row's sum to the caller's stored / original
 * row, bit-identical, including the 0 * x[0] term of the caller's padding),
 * 0 drops it, -1 applies the cost model (chunk occupancy < 0.9 or C != 32,
 * and the caller's layout not already a C = 32 one sorted that widely; for
 * C != 32 a SELL-32-1 re-chunking of the stored order is a second
 * candidate; the fastest timed candidate is kept for a >= 5 % win).  Every
 * build applies the cost model unless SELLB_SHADOW=0 / 1 forces it.
 * Chunk-range calls (c0, c1 not the whole matrix) keep the caller's layout.  sellb_info_t.shadow is
 * the shadow's sigma (0: none).  The cost model times its candidates with
 * whole-matrix SpMVs on scratch vectors (SELLB_SHADOW_TIME=0 skips that);
 * like sellb_set_packed / sellb_set_variant it must not run concurrently
 * with other calls on the same matrix. */
int sellb_set_shadow(sellb_mat* m, int32_t mode);
void sellb_free(sellb_mat* m);

/* ---- SpMV ---------------------------------------------------------------- */

/* y (+)= A x over chunks [c0, c1) on device vectors (async on `stream`).
 * out_order STORED: y has n_rows_padded entries (reference convention,
 * spmv.py:109-112); ORIGINAL: y has n_rows entries, written through the
 * stored->original map (fused unpermute_vector, formats.py:433-441). */
int sellb_spmv(const sellb_mat* m, const void* x, void* y, int64_t c0, int64_t c1,
               int32_t accumulate, int32_t out_order, void* stream);

/* Same product over a device list of chunk ids (interior/boundary split of
 * the row-partitioned multi-GPU path). */
int sellb_spmv_chunk_list(const sellb_mat* m, const int32_t* chunk_ids, int64_t n_ids,
                          const void* x, void* y, int32_t accumulate, void* stream);

/* End-to-end: host x[n_cols] -> device, product, device -> host y.  Blocks
 * until y is on the host.  Pinned host buffers give full PCIe bandwidth. */
int sellb_spmv_host(sellb_mat* m, const void* x_host, void* y_host,
                    int64_t c0, int64_t c1, int32_t accumulate, int32_t out_order,
                    void* stream);

/* Stateless reference signature (_kernels.pyx:65-68) on HOST arrays; the
 * extra sizes are the lengths the Python memoryviews carry implicitly. */
int sellb_spmv_sell_range_host(const int64_t* cs, const int32_t* cl, int32_t C,
                               const int32_t* col, const double* val, int64_t n_slots,
                               int64_t n_chunks, const double* x, int64_t n_x,
                               double* y, int64_t n_y, int64_t c0, int64_t c1,
                               int32_t accumulate, int32_t device);

/* CRS kernels of the same protocol (_kernels.pyx:17-62), HOST arrays. */
int sellb_spmv_crs_range_host(const int64_t* rpt, int64_t n_rows, const int32_t* col,
                              const double* val, int64_t nnz, const double* x,
                              int64_t n_x, double* y, int64_t r0, int64_t r1,
                              int32_t accumulate, int32_t unrolled, int32_t device);

/* Device-resident CRS handle for the same protocol: the arrays are
 * validated (rpt starts at 0, ends at nnz, non-decreasing; 0 <= col <
 * n_cols; formats.py:140-155) and uploaded once; each sellb_crs_spmv_host
 * call moves x in and y[r0:r1) out (host arrays, blocking).  The kernels
 * module caches handles by buffer identity (replaces the per-call upload of
 * sellb_spmv_crs_range_host). */
typedef struct sellb_crs sellb_crs;
int sellb_crs_import(const int64_t* rpt, const int32_t* col, const void* val, int32_t dtype,
                     int64_t n_rows, int64_t n_cols, int64_t nnz, int32_t device,
                     sellb_crs** out);
int sellb_crs_spmv_host(sellb_crs* m, const void* x_host, void* y_host, int64_t r0, int64_t r1,
                        int32_t accumulate, int32_t unrolled);
void sellb_crs_free(sellb_crs* m);

/* CRS kernels on device arrays. */
int sellb_spmv_crs(const int64_t* rpt, const int32_t* col, const void* val,
                   int32_t dtype, const void* x, void* y, int64_t r0, int64_t r1,
                   int32_t accumulate, int32_t unrolled, void* stream);

/* ---- measurement support ------------------------------------------------- */

double sellb_chunk_occupancy(const sellb_mat* m);
/* Sector-effective occupancy: nnz / (val/col elements inside the 32-byte
 * sectors the pad-skipping kernel touches). */
int sellb_sector_occupancy(const sellb_mat* m, double* beta_eff, int64_t* val_sectors,
                           int64_t* col_sectors, void* stream);

/* Device read-reduce / copy bandwidth kernels (membench.py:52-116 analogs). */
int sellb_read_sum(const double* a_dev, int64_t n, double* out_host, void* stream);
int sellb_copy(const double* src_dev, double* dst_dev, int64_t n, void* stream);
/* Overwrite a scratch buffer larger than L2, then read half of it back so the
 * L2 holds clean lines (timing hygiene: the next kernel neither hits its own
 * data nor pays for the flush's write-backs). */
int sellb_l2_flush(void* scratch_dev, int64_t bytes, void* stream);

/* Padding fix-up of the row-partitioned path: the reference adds 0*x[0]
 * for every padded slot, which only matters when x[0] is not finite.  With
 * *x0 (device) not finite, every stored row with padding becomes
 * y[p] + 0*x0 (NaN); with finite *x0 the kernel writes nothing. */
int sellb_pad_fixup(const sellb_mat* m, const void* x0, void* y, void* stream);

/* Boundary classification for the row-partitioned path: chunk_flag[c] = 1
 * iff some stored row p of chunk c has row_flag[order[p]] != 0 (row_flag in
 * ORIGINAL row order, e.g. "reads a non-owned column"), else 0. */
int sellb_chunk_flags(const sellb_mat* m, const uint8_t* row_flag, uint8_t* chunk_flag,
                      void* stream);

/* Halo pack / unpack for the row-partitioned multi-GPU SpMV (dist.py):
 * out[k] = x[idx[k]]  and  x[idx[k]] = in[k]  (k < n), on `stream`. */
int sellb_gather(const void* x, const int32_t* idx, void* out, int64_t n, int32_t dtype,
                 void* stream);
int sellb_scatter(const void* in, const int32_t* idx, void* x, int64_t n, int32_t dtype,
                  void* stream);

/* cfg5 generator (BASELINE configs[4]) straight into device CRS, rows
 * [r0, r1) of the N = n banded-random matrix (generate.py:hamiltonian_rows):
 * first rpt[r1-r0+1] (returns nnz), then col/val into caller buffers. */
int sellb_gen_hamiltonian_rpt(int64_t n, int64_t r0, int64_t r1, const int64_t* offs_dev,
                              int32_t n_off, double keep, uint64_t seed, int64_t* rpt_dev,
                              int64_t* nnz_out, void* stream);
int sellb_gen_hamiltonian_fill(int64_t n, int64_t r0, int64_t r1, const int64_t* offs_dev,
                               int32_t n_off, double keep, uint64_t seed, const int64_t* rpt_dev,
                               int32_t* col_dev, void* val_dev, int32_t dtype, void* stream);

/* cfg3 generator (BASELINE configs[2]) straight into device CRS, rows
 * [r0, r1) of the N = n power-law matrix (generate.py:powerlaw_rows, the
 * same counter-hash definition, bit-identical): rpt first (returns nnz),
 * then col / val into caller buffers. */
int sellb_gen_powerlaw_rpt(int64_t n, int64_t r0, int64_t r1, double base, int64_t lmax,
                           uint64_t seed, int64_t* rpt_dev, int64_t* nnz_out, void* stream);
int sellb_gen_powerlaw_fill(int64_t n, int64_t r0, int64_t r1, double base, int64_t lmax,
                            int64_t band, uint64_t seed, const int64_t* rpt_dev, int32_t* col_dev,
                            void* val_dev, int32_t dtype, void* stream);

/* COO -> canonical CRS on the device: the step before the build
 * (SURVEY.md §8(f)3).  Replaces COOMatrix's bounds check (formats.py:50-70),
 * canonicalize_coo (formats.py:89-108) and coo_to_crs (formats.py:169-175).
 * rows/cols int64[nnz], vals f64[nnz] in any order with duplicates; outputs
 * rpt int64[n_rows+1], col int32[cap nnz], val f64[cap nnz] and *nnz_out =
 * the number of distinct coordinates.  Duplicates are summed exactly as the
 * reference's np.add.reduceat (first entry + NumPy pairwise sum of the rest,
 * in stable (row, col) order): bit-identical output.  Host or device
 * pointers (ptrs_on_device); -3 with the reference's message for an
 * out-of-range index. */
int sellb_coo_to_crs(const int64_t* rows, const int64_t* cols, const double* vals, int64_t nnz,
                     int64_t n_rows, int64_t n_cols, int64_t* rpt, int32_t* col, double* val,
                     int64_t* nnz_out, int32_t device, void* stream, int32_t ptrs_on_device);

/* Matrix Market body (host, multi-threaded; io.py:125-162 / 252-259).
 * parse: the text after the size line -> out[n_entries * width] (row-major,
 * like np.loadtxt(..., comments="%")); capacity max_entries rows.  Returns
 * SELLB_EFORMAT for anything outside plain decimal / inf / nan tokens with
 * exactly `width` tokens per data line, or more than max_entries rows: the
 * caller then re-parses with the reference-compatible path for the exact
 * FormatError.  n_threads <= 0: all hardware threads.
 * format: "%d %d %.17g\n" lines of (rows+1, cols+1, vals) as np.savetxt
 * writes them; cap >= 64 * n suffices. */
int sellb_mm_parse_body(const char* text, int64_t len, int32_t width, int64_t max_entries,
                        double* out, int64_t* n_entries, int32_t n_threads);
int sellb_mm_format_body(const int64_t* rows, const int64_t* cols, const double* vals,
                         int64_t n, char* out, int64_t cap, int64_t* used, int32_t n_threads);

/* Process-wide number of compute-path kernel launches so far (SpMV roles,
 * long-row kernels, halo gather/scatter, pad fix-up, CRS kernels, L2 flush,
 * membench kernels): the bench's gpu_launches is a difference of two reads. */
int64_t sellb_launch_count(void);

/* lru_stream_misses (_kernels.pyx:95-139): misses of a fully-associative LRU
 * cache of cache_lines lines replaying lines[0..n) (ids in [0, n_line_slots)),
 * the RHS-traffic simulator behind cachesim.simulate_rhs_traffic.  Computed
 * on the device from LRU stack distances (sellb_lru.cu); n == 0 -> 0,
 * cache_lines <= 0 -> n as in the reference; an id outside the table ->
 * SELLB_EPARAM.  lines may be host (lines_on_device = 0) or device memory. */
int sellb_lru_stream_misses(const int64_t* lines, int64_t n, int64_t cache_lines,
                            int64_t n_line_slots, int32_t lines_on_device,
                            int64_t* misses, void* stream);

/* The x line ids (col / elems_per_line, elems_per_line a power of two) of
 * the matrix's real entries in kernel traversal order -- chunk by chunk,
 * slot-major then lane, padding dropped (cachesim.py:31-46) -- written to
 * the device buffer lines[nnz]; *n_out = nnz.  Feeds
 * sellb_lru_stream_misses(lines_on_device = 1) without a host pass. */
int sellb_sell_x_lines(const sellb_mat* m, int32_t elems_per_line, int64_t* lines,
                       int64_t* n_out, void* stream);

/* Pinned host buffers for the end-to-end path. */
int sellb_host_alloc(size_t bytes, void** out);
int sellb_host_free(void* p);

/* Page-lock (and map) a caller's existing host buffer in place, so
 * sellb_spmv_host moves it by DMA at pinned speed instead of staging it
 * through the library's mirrors.  The caller must unregister before the
 * memory is released (the Python layer ties this to the array's lifetime).
 * Returns SELLB_ERESOURCE if the range cannot be registered (e.g. it
 * shares pages with an already registered range): callers fall back to
 * the staged path. */
int sellb_host_register(void* p, size_t bytes);
int sellb_host_unregister(void* p);

#ifdef __cplusplus
}
#endif

#endif /* SELLB_H */
