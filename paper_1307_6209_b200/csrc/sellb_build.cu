// sellb_build.cu -- SELL-C-sigma construction on the device (crs_to_sell,
// /root/reference/pkg/src/sellkit/formats.py:295-393), import / export of
// device matrices and the kernel-variant cost model.
//
// Pipeline (all stream-ordered, one host sync to size val/col):
//   1. k_row_lengths      len_pad[p] = rpt[p+1]-rpt[p] (0 for padding rows),
//                         column-bound check, max length      (formats.py:336-338)
//   2. k_sort_keys +      stable LSD radix sort of (scope, maxlen-len) with the
//      cub radix sort     index as payload == np.lexsort((idx,-len,scope))
//                                                              (formats.py:285-292)
//   3. k_apply_order      perm[order[p]] = p, row_lengths[p] = len[order[p]]
//                                                              (formats.py:345-349)
//   4. k_chunk_width      cl = max over the chunk, align rounding, C*cl
//                                                              (formats.py:351-356)
//   5. cub scan           cs = [0, cumsum(C*cl)]               (formats.py:358-360)
//   6. k_fill             column-major scatter with zero padding and optional
//                         column permutation                  (formats.py:362-377)
#include <cub/cub.cuh>

#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <vector>

#include "sellb_internal.cuh"

using namespace sellb;

namespace {

__global__ void k_row_lengths(const int64_t* __restrict__ rpt, int64_t n, int64_t n_pad,
                              int32_t* __restrict__ len, unsigned int* __restrict__ maxlen,
                              int* __restrict__ bad) {
    // grid-stride; the maximum is reduced per warp, then per block in shared
    // memory, then one global atomic per block (one per warp serialised 2^21
    // atomics on one address for cfg5: 1.6 ms)
    __shared__ unsigned int s_max;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    unsigned int lmax = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_pad; p += stride) {
        unsigned int l = 0;
        if (p < n) {
            int64_t d = rpt[p + 1] - rpt[p];
            if (d < 0 || d > 0x7fffffffLL) { atomicExch(bad, 1); d = 0; }
            l = (unsigned int)d;
        }
        len[p] = (int32_t)l;
        lmax = max(lmax, l);
    }
    for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if ((threadIdx.x & 31) == 0 && lmax) atomicMax(&s_max, lmax);
    __syncthreads();
    if (threadIdx.x == 0 && s_max) atomicMax(maxlen, s_max);
}

// sellb_import's layout invariants: bad = 3 (cs[0] != 0), 4 (chunk extent
// != C * cl or negative cl)
__global__ void k_check_layout(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                               int64_t n_chunks, int64_t C, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0 && cs[0] != 0) atomicExch(bad, 3);
    if (i < n_chunks && (cl[i] < 0 || cs[i + 1] - cs[i] != C * (int64_t)cl[i]))
        atomicMax(bad, 4);
}

__global__ void k_check_cols(const int32_t* __restrict__ col, int64_t nnz, int64_t n_cols,
                             int* __restrict__ bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int flag = 0;
    for (; i < nnz; i += stride) {
        int32_t c = col[i];
        flag |= (c < 0) | ((int64_t)c >= n_cols);
    }
    if (__any_sync(0xffffffffu, flag) && (threadIdx.x & 31) == 0) atomicExch(bad, 2);
}

template <typename K>
__global__ void k_sort_keys(const int32_t* __restrict__ len, int64_t n_pad, int64_t sigma_eff,
                            int lbits, unsigned int maxlen, K* __restrict__ keys,
                            int32_t* __restrict__ idx) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n_pad) return;
    K scope = (K)(p / sigma_eff);
    K inv = (K)(maxlen - (unsigned int)len[p]);   // descending length
    keys[p] = (scope << lbits) | inv;
    idx[p] = (int32_t)p;
}

__global__ void k_apply_order(const int32_t* __restrict__ order, const int32_t* __restrict__ len,
                              int64_t n, int64_t n_pad, int32_t* __restrict__ perm,
                              int32_t* __restrict__ rl, int32_t* __restrict__ order_out) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n_pad) return;
    int32_t o = order ? order[p] : (int32_t)p;
    rl[p] = len[o];
    order_out[p] = o;
    if (o < n) perm[o] = (int32_t)p;
}

// one warp per chunk: max of the chunk's C stored-row lengths (sigma = 1; the
// sorted layouts get their widths from k_scope_sort).  The largest width is
// the longest row rounded to the unit, so no reduction is needed here.
__global__ void k_chunk_width(const int32_t* __restrict__ rl, int64_t n_chunks, int64_t C,
                              int64_t unit, int32_t* __restrict__ cl,
                              int64_t* __restrict__ slots) {
    int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (w >= n_chunks) return;
    const int32_t* r = rl + w * C;
    int32_t m = 0;
    for (int64_t i = lane; i < C; i += 32) m = max(m, r[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
        int64_t mm = m;
        if (unit > 1) mm = ((mm + unit - 1) / unit) * unit;
        cl[w] = (int32_t)mm;
        slots[w] = C * mm;
    }
}

// sigma = 1: stored order is the original order; row_lengths, order and perm
// in one pass (k_apply_order without the sort)
__global__ void k_identity_order(const int32_t* __restrict__ len, int64_t n, int64_t n_pad,
                                 int32_t* __restrict__ perm, int32_t* __restrict__ rl,
                                 int32_t* __restrict__ order_out) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n_pad) return;
    rl[p] = len[p];
    order_out[p] = (int32_t)p;
    if (p < n) perm[p] = (int32_t)p;
}

// The sigma-window sort (formats.py:285-292, np.lexsort((idx, -len, scope)))
// for scopes of at most TH*IT rows: one CTA per scope loads the scope's row
// lengths, sorts (maxlen - len) with the in-scope index as payload by a
// stable block radix sort over lbits bits only (equal lengths keep their
// original order = the idx tie-break), and writes order / row_lengths / perm
// plus -- scopes are whole chunks (sigma_eff is a multiple of C or n_pad) and
// sorted descending, so a chunk's width is its first row's length -- cl and
// the per-chunk slot counts.  Replaces key build + device radix sort +
// k_apply_order + k_chunk_width (cfg5: 5.4 ms -> one launch).
template <int TH, int IT>
__global__ void __launch_bounds__(TH) k_scope_sort(
        const int32_t* __restrict__ len, int64_t n, int64_t n_pad, int64_t sigma_eff, int lbits,
        unsigned int maxlen, int64_t C, int64_t unit, int32_t* __restrict__ perm,
        int32_t* __restrict__ rl, int32_t* __restrict__ order_out, int32_t* __restrict__ cl,
        int64_t* __restrict__ slots) {
    using Sort = cub::BlockRadixSort<uint32_t, TH, IT, int32_t>;
    __shared__ typename Sort::TempStorage tmp;
    const int64_t s0 = (int64_t)blockIdx.x * sigma_eff;
    const int sz = (int)(n_pad - s0 < sigma_eff ? n_pad - s0 : sigma_eff);
    const uint32_t pad_key = lbits >= 32 ? 0xffffffffu : ((1u << lbits) - 1u);
    uint32_t keys[IT];
    int32_t idx[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const int r = threadIdx.x * IT + i;          // blocked: rank order = input order
        idx[i] = r;
        keys[i] = r < sz ? maxlen - (uint32_t)len[s0 + r] : pad_key;
    }
    Sort(tmp).SortBlockedToStriped(keys, idx, 0, lbits);
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const int r = i * TH + threadIdx.x;          // striped: coalesced stores
        if (r >= sz) continue;
        const int64_t p = s0 + r;
        const int64_t o = s0 + idx[i];
        const int32_t l = (int32_t)(maxlen - keys[i]);
        rl[p] = l;
        order_out[p] = (int32_t)o;
        if (o < n) perm[o] = (int32_t)p;
        if (p % C == 0) {
            int64_t w = l;
            if (unit > 1) w = ((w + unit - 1) / unit) * unit;
            cl[p / C] = (int32_t)w;
            slots[p / C] = C * w;
        }
    }
}

// one thread per stored row; consecutive threads of a chunk write consecutive
// addresses for every slot j (coalesced stores), each thread streams its own
// CRS row (L1-resident lines across j).  U slots per batch: the batch's
// loads are all in flight before its stores (and a row's lines are consumed
// before other warps evict them from L1).
template <typename T, int U>
__global__ void k_fill(const int64_t* __restrict__ rpt, const int32_t* __restrict__ col_in,
                       const T* __restrict__ val_in, int64_t n, int64_t n_pad, int64_t C,
                       const int32_t* __restrict__ order, const int32_t* __restrict__ rl,
                       const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                       const int32_t* __restrict__ perm, int permute_cols,
                       int32_t* __restrict__ col_out, T* __restrict__ val_out, int64_t n_cols,
                       int* __restrict__ bad) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n_pad) return;
    int64_t chunk = p / C;
    int64_t dst = cs[chunk] + (p - chunk * C);
    int32_t w = cl[chunk];
    int32_t len = rl[p];
    int32_t o = order[p];
    int64_t src = (o < n) ? rpt[o] : 0;
    int flag = 0;
    for (int32_t j0 = 0; j0 < w; j0 += U) {
        T v[U];
        int32_t c[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int32_t j = j0 + k;
            v[k] = T(0);
            c[k] = 0;
            if (j < len) {
                v[k] = __ldg(val_in + src + j);
                c[k] = __ldg(col_in + src + j);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int32_t j = j0 + k;
            if (j >= w) break;
            // every CRS entry passes here exactly once: the column-bound
            // check rides on the fill (bad != nullptr) instead of a 4 B/nnz
            // pass of its own; with permute_cols it ran before the fill
            if (j < len) {
                if (bad) flag |= (c[k] < 0) | ((int64_t)c[k] >= n_cols);
                if (permute_cols) c[k] = perm[c[k]];
            }
            __stcs(val_out + dst + (int64_t)j * C, v[k]);
            __stcs(col_out + dst + (int64_t)j * C, c[k]);
        }
    }
    if (bad && flag) atomicExch(bad, 2);
}

// sector accounting for the cost model: a 32-byte sector of val (4 fp64 / 8
// fp32 lanes) or col (8 lanes) is fetched for slot j iff one of its lanes has
// j < row length.  Sum over lane groups of the group's max length.
__global__ void k_sector_count(const int32_t* __restrict__ rl, int64_t n_pad, int64_t C,
                               int gv, int gc, unsigned long long* __restrict__ out) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // group of gc lanes
    unsigned long long sv = 0, sc = 0;
    int64_t p0 = g * gc;
    if (p0 < n_pad) {
        // groups never straddle chunks when C is a multiple of the group size;
        // otherwise this is an estimate (documented in DESIGN.md)
        int32_t mc = 0;
        for (int k = 0; k < gc; k += gv) {
            int32_t mv = 0;
            for (int q = k; q < k + gv && p0 + q < n_pad; ++q) mv = max(mv, rl[p0 + q]);
            sv += (unsigned long long)mv;
            mc = max(mc, mv);
        }
        sc = (unsigned long long)mc;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sv += __shfl_xor_sync(0xffffffffu, sv, o);
        sc += __shfl_xor_sync(0xffffffffu, sc, o);
    }
    // per block in shared memory, then one pair of global atomics per block
    __shared__ unsigned long long s_sum[2];
    if (threadIdx.x == 0) s_sum[0] = s_sum[1] = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_sum[0], sv);
        atomicAdd(&s_sum[1], sc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(out, s_sum[0]);
        atomicAdd(out + 1, s_sum[1]);
    }
}

// Bytes of val/col the SpMV kernels stream for this matrix as configured:
// pad-inclusive chunks (no long-row role in them) read every slot; chunks
// read with pad-skip semantics read the 32-byte sectors holding an active
// lane of a bulk row (long rows -- rl > chunk_th of a chunk wider than
// long_th -- excluded: they go to the long-row roles) plus row_lengths.
// One thread per chunk; gv / gc = lanes per val / col sector, g = 64-byte
// granularity variant (2 sectors) for the DRAM-transfer estimate.
__global__ void k_stream_count(const int32_t* __restrict__ rl, const int32_t* __restrict__ cl,
                               const int32_t* __restrict__ chunk_th, int64_t n_chunks,
                               int64_t C, int skip_variant, int long_th, int vs,
                               unsigned long long* __restrict__ out /* [4] */) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long incl = 0, s32 = 0, s64 = 0, rlb = 0;
    if (c < n_chunks) {
        const int w = cl[c];
        const bool longish = chunk_th && w > long_th;
        if (!skip_variant && !longish) {
            incl = (unsigned long long)C * w * (vs + 4);
        } else {
            const int th = longish ? chunk_th[c] : 0x7fffffff;
            const int gv = 32 / vs, gc = 8;
            for (int pass = 0; pass < 2; ++pass) {          // 32-byte, then 64-byte sectors
                const int mul = pass ? 2 : 1;
                unsigned long long acc = 0;
                for (int64_t r0 = 0; r0 < C; r0 += gv * mul) {
                    int mv = 0;
                    for (int64_t r = r0; r < r0 + gv * mul && r < C; ++r) {
                        const int l = rl[c * C + r];
                        mv = max(mv, l > th ? 0 : l);
                    }
                    acc += (unsigned long long)mv * 32ull * mul;
                }
                for (int64_t r0 = 0; r0 < C; r0 += gc * mul) {
                    int mc = 0;
                    for (int64_t r = r0; r < r0 + gc * mul && r < C; ++r) {
                        const int l = rl[c * C + r];
                        mc = max(mc, l > th ? 0 : l);
                    }
                    acc += (unsigned long long)mc * 32ull * mul;
                }
                if (pass) s64 = acc; else s32 = acc;
            }
            rlb = 4ull * C;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        incl += __shfl_xor_sync(0xffffffffu, incl, o);
        s32 += __shfl_xor_sync(0xffffffffu, s32, o);
        s64 += __shfl_xor_sync(0xffffffffu, s64, o);
        rlb += __shfl_xor_sync(0xffffffffu, rlb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, incl);
        atomicAdd(out + 1, s32);
        atomicAdd(out + 2, s64);
        atomicAdd(out + 3, rlb);
    }
}

// .sell cache semantics (io.py:308-321): length = chunk width minus the
// trailing run of padding-looking slots (value 0.0 and column 0)
template <typename T>
__global__ void k_trailing_len(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                               const int32_t* __restrict__ col, const T* __restrict__ val,
                               int64_t n_pad, int64_t C, int32_t* __restrict__ rl) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n_pad) return;
    const int64_t c = p / C;
    const int64_t base = cs[c] + (p - c * C);
    int32_t len = cl[c];
    while (len > 0 && val[base + (int64_t)(len - 1) * C] == T(0) &&
           col[base + (int64_t)(len - 1) * C] == 0)
        --len;
    rl[p] = len;
}

int64_t sigma_effective(int64_t n, int64_t C, int64_t sigma, int64_t n_pad) {
    // formats.py:325-334
    if (sigma <= C) return 1;
    if (sigma >= n) return std::max<int64_t>(n_pad, 1);
    if (sigma % C != 0) return -1;
    return sigma;
}

int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

void free_mat_arrays(sellb_mat* m) {
    if (!m) return;
    DeviceGuard g(m->device);
    if (m->meta_slab) {
        cudaFree(m->meta_slab);
    } else {
        cudaFree(m->cs);
        cudaFree(m->cl);
        cudaFree(m->rl);
        cudaFree(m->perm);
        cudaFree(m->order);
    }
    m->meta_slab = nullptr;
    cudaFree(m->col);
    cudaFree(m->val);
    cudaFree(m->long_rows);
    cudaFree(m->chunk_th);
    cudaFree(m->long_groups);
    cudaFree(m->long_rest);
    cudaFree(m->side_off);
    cudaFree(m->side_col);
    cudaFree(m->side_val);
    cudaFree(m->prpt);
    cudaFree(m->pcol);
    cudaFree(m->pval);
    free_shadow(m);
    if (m->pipe_ready) {
        cudaStreamDestroy(m->s_h2d);
        cudaStreamDestroy(m->s_comp);
        cudaStreamDestroy(m->s_d2h);
        cudaEventDestroy(m->ev_start);
        for (int i = 0; i < sellb_mat::kPipe; ++i) {
            cudaEventDestroy(m->ev_x[i]);
            cudaEventDestroy(m->ev_blk[i]);
        }
    }
    if (m->long_ready) {
        cudaStreamDestroy(m->s_long);
        cudaEventDestroy(m->ev_fork);
        cudaEventDestroy(m->ev_join);
    }
    cudaFree(m->x_buf);
    cudaFree(m->y_buf);
    if (m->hx) cudaFreeHost(m->hx);
    if (m->hy) cudaFreeHost(m->hy);
}

int alloc_dev(void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e != cudaSuccess) {
        *p = nullptr;
        return set_error(SELLB_ERESOURCE, "device allocation of %zu bytes failed: %s", bytes,
                         cudaGetErrorString(e));
    }
    return 0;
}

int check_stream_error() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SELLB_ERESOURCE, "kernel launch failed: %s", cudaGetErrorString(e));
    return 0;
}

// variant cost model: bytes of the pad-skipping kernel (touched sectors plus
// the row_lengths stream) against the pad-inclusive one (every slot).
int choose_variant(sellb_mat* m, cudaStream_t st, double* beta_eff_out, int64_t* vs_out,
                   int64_t* cs_out) {
    if (!m->rl) { m->variant = SELLB_VARIANT_PAD_INCL; return 0; }
    if (m->n_pad == 0) { m->variant = SELLB_VARIANT_PAD_INCL; return 0; }
    DBuf cnt;
    SELLB_CU(cnt.alloc(2 * sizeof(unsigned long long), st));
    SELLB_CU(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), st));
    int gv = m->dtype == SELLB_F32 ? 8 : 4, gc = 8;
    int64_t groups = (m->n_pad + gc - 1) / gc;
    k_sector_count<<<(unsigned)grid_for(groups, 256), 256, 0, st>>>(
        m->rl, m->n_pad, m->C, gv, gc, cnt.as<unsigned long long>());
    if (int rc = check_stream_error()) return rc;
    unsigned long long h[2];
    SELLB_CU(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    double sv = (double)vsize(m->dtype);
    double bytes_skip = 32.0 * (double)h[0] + 32.0 * (double)h[1] + 4.0 * (double)m->n_pad;
    double bytes_incl = (sv + 4.0) * (double)m->slots;
    if (vs_out) *vs_out = (int64_t)h[0];
    if (cs_out) *cs_out = (int64_t)h[1];
    if (beta_eff_out) {
        double touched = 32.0 * (double)h[0] + 32.0 * (double)h[1];
        *beta_eff_out = touched > 0 ? (sv + 4.0) * (double)m->nnz / touched : 1.0;
    }
    if (m->variant == SELLB_VARIANT_AUTO || m->variant == 0)
        m->variant = bytes_skip < bytes_incl ? SELLB_VARIANT_PAD_SKIP : SELLB_VARIANT_PAD_INCL;
    return 0;
}

// long-row side table: warp k copies stored row rows[k] (slots j < rl, C
// apart in the SELL arrays) to side_*[off[k] + j]
template <typename T>
__global__ void k_side_fill(const int64_t* __restrict__ cs, const int32_t* __restrict__ col,
                            const T* __restrict__ val, const int32_t* __restrict__ rows,
                            int64_t n, int64_t C, const int32_t* __restrict__ rl,
                            const int64_t* __restrict__ off, int32_t* __restrict__ side_col,
                            T* __restrict__ side_val) {
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= n) return;
    const int64_t p = rows[k];
    const int64_t chunk = p / C;
    const int64_t base = cs[chunk] + (p - chunk * C);
    const int len = rl[p];
    for (int j = lane; j < len; j += 32) {
        side_col[off[k] + j] = col[base + (int64_t)j * C];
        side_val[off[k] + j] = val[base + (int64_t)j * C];
    }
}

// Rows longer than the threshold go to the kernel's warp-per-row role.
// Default threshold 256 slots (SELLB_LONG_TH overrides; <= 0 disables).
// uniform_th > 0: every row longer than uniform_th is long (the packed
// copy's rule: the row-run kernel walks a row serially, so its longest rows
// go to the warp-per-row role, which starts first)
int build_long_rows(sellb_mat* m, cudaStream_t st, int uniform_th = 0) {
    cudaFree(m->long_rows);
    cudaFree(m->chunk_th);
    cudaFree(m->long_groups);
    cudaFree(m->long_rest);
    cudaFree(m->side_off);
    cudaFree(m->side_col);
    cudaFree(m->side_val);
    m->side_off = nullptr;
    m->side_col = nullptr;
    m->side_val = nullptr;
    m->long_rows = nullptr;
    m->chunk_th = nullptr;
    m->long_groups = nullptr;
    m->long_rest = nullptr;
    m->n_long = 0;
    m->n_groups = 0;
    m->n_rest = 0;
    m->long_th = 0x7fffffff;
    if (!m->rl || m->n_pad == 0) return 0;
    // Two thresholds: a row longer than th_lo leaves the bulk role when its
    // chunk is heterogeneous (shortest row < 1/4 of the widest: the warp
    // would run mostly idle lanes), and any row longer than th_hi leaves it
    // (one thread's latency chain).  Sorted chunks of similar long rows stay
    // in the coalesced bulk role up to th_hi (measured: cfg3 sigma=N 693 ->
    // 742 GF/s with the threshold raised from 256 to 512).
    int th = 256, th_hi = 512;      // th_hi 512/1024/2048 on cfg3 sigma=N: 742/674/426
    if (const char* e = getenv("SELLB_LONG_TH")) th = th_hi = atoi(e);
    if (const char* e = getenv("SELLB_LONG_TH_HI")) th_hi = atoi(e);
    if (uniform_th > 0) th = th_hi = uniform_th;
    // Rule 1: a row is long when it is longer than th_hi, or than
    // max(floor, f * the chunk's k-th longest row) -- i.e. it stands out of
    // its own chunk (unsorted layouts: one or two long rows among short ones,
    // whose slots would each cost a DRAM line in the bulk) and then reads
    // from the side table; sorted chunks (k-th longest close to the longest)
    // keep their rows in the coalesced bulk role.  Rule 0: the earlier
    // min/max heterogeneity test with the fixed threshold th.
    // Default: rule 1 for unsorted / shortly-sorted layouts (sigma_eff <=
    // 4 C), rule 0 for long scopes whose chunks descend smoothly (measured on
    // cfg3, tools/rule_ab.sh: sigma=1 246 -> 318 GF/s, sigma=128 441 -> 466
    // with rule 1; sigma=512 590 vs 576 keeps rule 0; sigma=N and cfg4 equal).
    const int rule = uniform_th > 0 ? 0
                     : getenv("SELLB_LONG_RULE") ? atoi(getenv("SELLB_LONG_RULE"))
                                                 : (m->sigma_eff <= 4 * m->C ? 1 : 0);
    const int floor_th = getenv("SELLB_LONG_FLOOR") ? atoi(getenv("SELLB_LONG_FLOOR")) : 48;
    const int kth = std::max(1, getenv("SELLB_LONG_K") ? atoi(getenv("SELLB_LONG_K")) : 8);
    const int fct = std::max(1, getenv("SELLB_LONG_F") ? atoi(getenv("SELLB_LONG_F")) : 2);
    if (rule == 1 && !getenv("SELLB_LONG_TH")) th = std::min(th, floor_th);
    if (th <= 0 || m->max_cl <= th) return 0;
    std::vector<int32_t> h_rl(m->n_pad), h_cl(m->n_chunks);
    SELLB_CU(cudaMemcpyAsync(h_rl.data(), m->rl, m->n_pad * 4, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaMemcpyAsync(h_cl.data(), m->cl, m->n_chunks * 4, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    std::vector<int32_t> cth(m->n_chunks, th_hi), rows, lens(m->C);
    for (int64_t c = 0; c < m->n_chunks; ++c) {
        if (h_cl[c] <= th) continue;
        if (rule == 1) {
            for (int64_t r = 0; r < m->C; ++r) lens[r] = h_rl[c * m->C + r];
            const int64_t k = std::min<int64_t>(kth, m->C) - 1;
            std::nth_element(lens.begin(), lens.begin() + k, lens.end(), std::greater<int32_t>());
            const int64_t t = std::max<int64_t>(th, (int64_t)fct * lens[k]);
            cth[c] = (int32_t)std::min<int64_t>(th_hi, t);
        } else {
            int32_t lo = 0x7fffffff, hi = 0;
            for (int64_t r = 0; r < m->C; ++r) {
                lo = std::min(lo, h_rl[c * m->C + r]);
                hi = std::max(hi, h_rl[c * m->C + r]);
            }
            if ((int64_t)lo * 4 < hi || uniform_th > 0) cth[c] = th;
        }
        for (int64_t r = 0; r < m->C; ++r)
            if (h_rl[c * m->C + r] > cth[c]) rows.push_back((int32_t)(c * m->C + r));
    }
    if (rows.empty()) return 0;
    if (int rc = alloc_dev((void**)&m->chunk_th, m->n_chunks * 4)) return rc;
    SELLB_CU(cudaMemcpyAsync(m->chunk_th, cth.data(), m->n_chunks * 4, cudaMemcpyHostToDevice,
                             st));
    std::stable_sort(rows.begin(), rows.end(),
                     [&](int32_t a, int32_t b) { return h_rl[a] > h_rl[b]; });
    if (int rc = alloc_dev((void**)&m->long_rows, rows.size() * 4)) return rc;
    SELLB_CU(cudaMemcpyAsync(m->long_rows, rows.data(), rows.size() * 4,
                             cudaMemcpyHostToDevice, st));
    // 8-row groups for the pipelined kernel: aligned groups of one chunk
    // holding >= 4 long rows (sorted chunks of long rows), longest first
    std::vector<int32_t> groups, rest;
    std::vector<int32_t> gmax;
    // When every long row fits the side table (<= 1/4 of the nonzeros), all
    // of them take the side-table warp-per-row role and no row groups are
    // formed (tools/grp_vs_side.sh: cfg3 sigma=N 843 -> 882 GF/s, cfg4
    // sigma=N C=32/128 733/735 -> 748/758, C=8 707 -> 697); larger long-row
    // shares keep the row-group kernel.  SELLB_LONG_GRP=1 forces groups, =0
    // disables them.
    const bool want_side_all = !(getenv("SELLB_LONG_SIDE") && atoi(getenv("SELLB_LONG_SIDE")) == 0);
    int64_t long_total = 0;
    for (int32_t p : rows) long_total += h_rl[p];
    const char* grp_env = getenv("SELLB_LONG_GRP");
    const bool use_groups =
        m->C % 8 == 0 && uniform_th <= 0 &&
        (grp_env ? atoi(grp_env) != 0
                 : !(want_side_all && long_total * 4 <= std::max<int64_t>(m->nnz, 1)));
    if (use_groups) {
        std::vector<uint8_t> is_long(m->n_pad, 0);
        for (int32_t p : rows) is_long[p] = 1;
        std::vector<uint8_t> in_grp(m->n_pad, 0);
        for (int32_t p : rows) {
            const int32_t g0 = p & ~7;
            if (in_grp[g0]) continue;
            int cnt = 0;
            int32_t mx = 0;
            for (int r = 0; r < 8; ++r)
                if (is_long[g0 + r]) { ++cnt; mx = std::max(mx, h_rl[g0 + r]); }
            if (cnt >= 4) {
                for (int r = 0; r < 8; ++r) in_grp[g0 + r] = 1;
                groups.push_back(g0);
                gmax.push_back(mx);
            } else {
                in_grp[g0] = 2;       // sparse group: its long rows stay per-row
            }
        }
        for (int32_t p : rows)
            if (in_grp[p & ~7] != 1) rest.push_back(p);
        std::vector<int32_t> idx(groups.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int32_t)i;
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int32_t a, int32_t b) { return gmax[a] > gmax[b]; });
        std::vector<int32_t> sorted(groups.size());
        for (size_t i = 0; i < idx.size(); ++i) sorted[i] = groups[idx[i]];
        groups.swap(sorted);
    } else {
        rest = rows;
    }
    if (!groups.empty()) {
        if (int rc = alloc_dev((void**)&m->long_groups, groups.size() * 4)) return rc;
        SELLB_CU(cudaMemcpyAsync(m->long_groups, groups.data(), groups.size() * 4,
                                 cudaMemcpyHostToDevice, st));
    }
    if (!rest.empty()) {
        if (int rc = alloc_dev((void**)&m->long_rest, rest.size() * 4)) return rc;
        SELLB_CU(cudaMemcpyAsync(m->long_rest, rest.data(), rest.size() * 4,
                                 cudaMemcpyHostToDevice, st));
    }
    // side table for the rest rows: at most one more copy of their entries
    // (never more than the padded SELL arrays already hold), and only while
    // it takes under a quarter of the free device memory
    const bool want_side = !(getenv("SELLB_LONG_SIDE") && atoi(getenv("SELLB_LONG_SIDE")) == 0);
    if (want_side && !rest.empty()) {
        std::vector<int64_t> off(rest.size() + 1, 0);
        for (size_t k = 0; k < rest.size(); ++k) off[k + 1] = off[k] + h_rl[rest[k]];
        const int64_t total = off.back();
        const size_t vs = vsize(m->dtype);
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
        if (total > 0 && (size_t)total * (vs + 4) + off.size() * 8 <= free_b / 4) {
            if (int rc = alloc_dev((void**)&m->side_off, off.size() * 8)) return rc;
            if (int rc = alloc_dev((void**)&m->side_col, total * 4)) return rc;
            if (int rc = alloc_dev(&m->side_val, total * vs)) return rc;
            SELLB_CU(cudaMemcpyAsync(m->side_off, off.data(), off.size() * 8,
                                     cudaMemcpyHostToDevice, st));
            const unsigned grid = (unsigned)grid_for((int64_t)rest.size() * 32, 256);
            if (m->dtype == SELLB_F32)
                k_side_fill<float><<<grid, 256, 0, st>>>(
                    m->cs, m->col, (const float*)m->val, m->long_rest, (int64_t)rest.size(),
                    m->C, m->rl, m->side_off, m->side_col, (float*)m->side_val);
            else
                k_side_fill<double><<<grid, 256, 0, st>>>(
                    m->cs, m->col, (const double*)m->val, m->long_rest, (int64_t)rest.size(),
                    m->C, m->rl, m->side_off, m->side_col, (double*)m->side_val);
            SELLB_CU(cudaGetLastError());
        }
    }
    SELLB_CU(cudaStreamSynchronize(st));
    m->n_long = (int64_t)rows.size();
    m->n_groups = (int64_t)groups.size();
    m->n_rest = (int64_t)rest.size();
    m->long_th = th;
    return 0;
}

// ---------------------------------------------------------------------------
// Packed stored-order copy (C = 32): stored row p's entries, slot order,
// at prpt[p] .. prpt[p+1] (prpt = exclusive scan of row_lengths) -- the
// SELL layout without its padding, read by the row-run kernel.
// ---------------------------------------------------------------------------
// a stored row's entries in the packed copy: its length, or 0 for a row the
// warp-per-row role sums (chunk wider than long_th, row longer than chunk_th)
__global__ void k_packed_len(const int32_t* __restrict__ rl, const int32_t* __restrict__ cl,
                             const int32_t* __restrict__ chunk_th, int long_th, int64_t n,
                             int64_t C, int64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t c = i / C;
    const int len = rl[i];
    out[i] = (chunk_th && cl[c] > long_th && len > chunk_th[c]) ? 0 : len;
}

template <typename T>
__global__ void k_packed_fill(const int64_t* __restrict__ cs, const int32_t* __restrict__ rl,
                              const int32_t* __restrict__ col, const T* __restrict__ val,
                              int64_t n_pad, int64_t C, const int64_t* __restrict__ prpt,
                              int32_t* __restrict__ pcol, T* __restrict__ pval) {
    const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= n_pad) return;
    const int64_t chunk = p / C;
    const int64_t src = cs[chunk] + (p - chunk * C);
    const int64_t dst = prpt[p];
    const int len = (int)(prpt[p + 1] - dst);        // 0 for the warp-per-row role's rows
    for (int j = lane; j < len; j += 32) {
        pcol[dst + j] = col[src + (int64_t)j * C];
        pval[dst + j] = val[src + (int64_t)j * C];
    }
}

void free_packed(sellb_mat* m) {
    cudaFree(m->prpt);
    cudaFree(m->pcol);
    cudaFree(m->pval);
    m->prpt = nullptr;
    m->pcol = nullptr;
    m->pval = nullptr;
    m->n_packed = 0;
}

}  // namespace

namespace sellb {

// force: 1 build, 0 drop, -1 cost model, -2 the build's default: the cost
// model unless SELLB_PACKED says 0 / 1 (measured, tools/packed_ab.sh: cfg3
// sigma=1 324 -> 450 GF/s; sigma=128 / 512 and cfg4 are faster in the SELL
// bulk role, and the model leaves them there)
// set while build_shadow builds the shadow's own layout: that build adds
// neither a packed copy nor a shadow of its own
thread_local bool t_shadow_build = false;

int build_packed(sellb_mat* m, cudaStream_t st, int force) {
    if (t_shadow_build) return 0;
    const bool had = m->pcol != nullptr;
    free_packed(m);
    if (had) {   // the SELL kernels' own long-row rule again
        if (int rc = build_long_rows(m, st)) return rc;
    }
    bool from_env = false;
    if (force == -2) {
        const char* e = getenv("SELLB_PACKED");
        force = (!e || strcmp(e, "auto") == 0) ? -1 : (atoi(e) ? 1 : 0);
        from_env = true;
    }
    if (force == 0) return 0;
    const bool possible = m->C == 32 && m->rl && m->n_chunks > 0 && m->slots > 0;
    if (!possible) {
        // an explicit request fails loudly; SELLB_PACKED=1 applies where it can
        if (force == 1 && !from_env)
            return set_error(SELLB_EPARAM, "the packed copy needs C = 32 and row_lengths");
        return 0;
    }
    const int64_t vs = (int64_t)vsize(m->dtype);
    const int64_t total = m->nnz;
    if (force < 0) {
        // cost model: the 64-byte sectors the bulk role touches for the short
        // rows (the long rows read the side table) against the packed copy's
        // bytes (every row, no padding) + its row offsets
        if (m->variant != SELLB_VARIANT_PAD_SKIP) { free_packed(m); return 0; }
        DBuf cnt;
        SELLB_CU(cnt.alloc(4 * sizeof(unsigned long long), st));
        SELLB_CU(cudaMemsetAsync(cnt.p, 0, 4 * sizeof(unsigned long long), st));
        k_stream_count<<<(unsigned)grid_for(m->n_chunks, 256), 256, 0, st>>>(
            m->rl, m->cl, m->chunk_th, m->n_chunks, m->C, 1, m->long_th, (int)vs,
            cnt.as<unsigned long long>());
        if (int rc = check_stream_error()) return rc;
        unsigned long long h[4];
        SELLB_CU(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        double gain_min = 1.3;      // cfg3 sigma=1: 1.52 (packed wins); sigma=512 1.05, cfg4 0.83
        if (const char* e = getenv("SELLB_PACKED_MIN_GAIN")) gain_min = atof(e);
        const double skip_bytes = (double)h[2];     // 64-byte sectors (DRAM bursts)
        const double packed_bytes = (double)(vs + 4) * (double)total + 8.0 * m->n_pad;
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
        if (skip_bytes < gain_min * packed_bytes ||
            (double)total * (double)(vs + 4) > 0.5 * (double)free_b) {
            free_packed(m);
            return 0;
        }
    }
    // the packed copy's long rows: rows longer than kPackedLong go to the
    // warp-per-row role (side table), started first on a side stream; the
    // packed copy leaves them out
    int plong = kPackedLong;
    if (const char* e = getenv("SELLB_PACKED_LONG")) plong = std::max(1, atoi(e));
    if (int rc = build_long_rows(m, st, plong)) return rc;
    if (int rc = alloc_dev((void**)&m->prpt, (m->n_pad + 1) * 8)) return rc;
    {
        DBuf d_len;
        SELLB_CU(d_len.alloc((m->n_pad + 1) * 8, st));
        SELLB_CU(cudaMemsetAsync(d_len.p, 0, 8, st));
        k_packed_len<<<(unsigned)grid_for(m->n_pad, 256), 256, 0, st>>>(
            m->rl, m->cl, m->chunk_th, m->long_th, m->n_pad, m->C, d_len.as<int64_t>() + 1);
        size_t tmp_bytes = 0;
        SELLB_CU(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, d_len.as<int64_t>(), m->prpt,
                                               m->n_pad + 1, st));
        DBuf d_tmp;
        SELLB_CU(d_tmp.alloc(tmp_bytes, st));
        SELLB_CU(cub::DeviceScan::InclusiveSum(d_tmp.p, tmp_bytes, d_len.as<int64_t>(), m->prpt,
                                               m->n_pad + 1, st));
    }
    int64_t packed_total = 0;
    SELLB_CU(cudaMemcpyAsync(&packed_total, m->prpt + m->n_pad, 8, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    if (int rc = alloc_dev((void**)&m->pcol, std::max<int64_t>(packed_total, 1) * 4)) return rc;
    if (int rc = alloc_dev(&m->pval, std::max<int64_t>(packed_total, 1) * vs)) return rc;
    const unsigned grid = (unsigned)grid_for(m->n_pad * 32, 256);
    if (m->dtype == SELLB_F32)
        k_packed_fill<float><<<grid, 256, 0, st>>>(m->cs, m->rl, m->col, (const float*)m->val,
                                                  m->n_pad, m->C, m->prpt, m->pcol,
                                                  (float*)m->pval);
    else
        k_packed_fill<double><<<grid, 256, 0, st>>>(m->cs, m->rl, m->col, (const double*)m->val,
                                                   m->n_pad, m->C, m->prpt, m->pcol,
                                                   (double*)m->pval);
    if (int rc = check_stream_error()) return rc;
    SELLB_CU(cudaStreamSynchronize(st));
    m->n_packed = packed_total;
    return 0;
}

}  // namespace sellb

namespace {

// ---------------------------------------------------------------------------
// Shadow execution layout.  Per-row sums do not depend on where a row is
// stored: SELL-32-N (every row sorted by length, chunks of near-equal rows)
// streams an irregular matrix with almost no padding, its longest rows
// together in the first chunks; SELL-32-512 does most of that for matrices
// whose x is far larger than L2 without scattering neighbouring rows.  The shadow holds the caller's stored rows
// re-laid that way; a full-range SpMV runs on it and scatters each sum to the
// caller's stored (or original) row through sh_ord_*, adding the reference's
// 0 * x[0] term where the CALLER's chunk padded the row (bit 31).  The
// caller's arrays stay the exported layout.
// ---------------------------------------------------------------------------
__global__ void k_shadow_maps(const int32_t* __restrict__ sh_order, int64_t sh_rows,
                              int64_t sh_pad, const int32_t* __restrict__ rl,
                              const int32_t* __restrict__ cl, int64_t C,
                              const int32_t* __restrict__ order, int64_t n_rows, int64_t n_pad,
                              int32_t* __restrict__ ord_st, int32_t* __restrict__ ord_or) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= sh_pad) return;
    const int64_t p = q < sh_rows ? sh_order[q] : n_pad;
    if (p >= n_pad) {
        ord_st[q] = 0x7fffffff;
        ord_or[q] = 0x7fffffff;
        return;
    }
    const uint32_t flag = rl[p] < cl[p / C] ? 0x80000000u : 0u;
    int64_t t = order ? (int64_t)order[p] : p;
    if (t >= n_rows) t = 0x7fffffff;
    ord_st[q] = (int32_t)((uint32_t)p | flag);
    ord_or[q] = (int32_t)((uint32_t)t | flag);
}

}  // namespace

namespace sellb {

// The cost model's candidates are settled by the clock: whole-matrix SpMVs on
// a scratch x (zeros) / y, alternately through the caller's layout and
// through the shadow -- one warm-up round, then five rounds of K back-to-back
// launches each way (K sized so a round lasts >= ~0.5 ms; CUDA events on the
// build's stream), best round per way.  Byte counts alone mislead both ways:
// cfg3 sigma = 1's packed copy streams ~V_alg yet is latency-bound (the
// shadow wins 1.45x), cfg4's spikes already sit in the side table and its
// bulk chunks are full (the shadow's map and scattered stores lose 8 %).
int time_shadow_choice(sellb_mat* m, cudaStream_t st, float* t_base, float* t_shadow) {
    const size_t vs = vsize(m->dtype);
    DBuf x, y;
    SELLB_CU(x.alloc(std::max<int64_t>(m->n_cols, 1) * vs, st));
    SELLB_CU(y.alloc(std::max<int64_t>(m->n_pad, 1) * vs, st));
    SELLB_CU(cudaMemsetAsync(x.p, 0, std::max<int64_t>(m->n_cols, 1) * vs, st));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    SELLB_CU(cudaEventCreate(&e0));
    if (cudaEventCreate(&e1) != cudaSuccess) {
        cudaEventDestroy(e0);
        return set_error(SELLB_ERESOURCE, "event creation failed");
    }
    sellb_mat* sh = m->shadow;
    float best[2] = {3.0e38f, 3.0e38f};
    int k_launch = 1;
    int rc = 0;
    for (int rep = 0; rep < 6 && !rc; ++rep) {
        for (int way = 0; way < 2 && !rc; ++way) {
            m->shadow = way ? sh : nullptr;
            cudaEventRecord(e0, st);
            for (int k = 0; k < k_launch && !rc; ++k)
                rc = launch_spmv(m, x.p, y.p, 0, m->n_chunks, 0, SELLB_ORDER_STORED, st);
            cudaEventRecord(e1, st);
            if (cudaEventSynchronize(e1) != cudaSuccess && !rc)
                rc = set_error(SELLB_ERESOURCE, "timing the shadow layout failed");
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0) best[way] = std::min(best[way], ms / (float)k_launch);
            else best[way] = ms;              // warm-up: one launch each way
        }
        if (rep == 0) {   // size the timed rounds from the warm-up launches
            const float t1 = std::max(std::min(best[0], best[1]), 1e-3f);
            k_launch = (int)std::min(16.0f, std::max(1.0f, 0.5f / t1));
            best[0] = best[1] = 3.0e38f;
        }
    }
    m->shadow = sh;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *t_base = best[0];
    *t_shadow = best[1];
    return rc;
}

void free_shadow(sellb_mat* m) {
    if (m->shadow) {
        free_mat_arrays(m->shadow);
        delete m->shadow;
    }
    cudaFree(m->sh_ord_st);
    cudaFree(m->sh_ord_or);
    m->shadow = nullptr;
    m->sh_ord_st = nullptr;
    m->sh_ord_or = nullptr;
}

// force: 1 build, 0 drop, -1 cost model, -2 the build's default (the cost
// model unless SELLB_SHADOW says 0 / 1).  Cost model: build when the layout is
// irregular (chunk occupancy beta < 0.9) or C != 32, and not already a C = 32
// layout sorted as widely as the shadow would be (SELL-32-N when x fits the L2 comfortably -- the global
// sort scatters rows, and with x in L2 the gathers do not care where a row
// sits -- else SELL-32-512)
int build_shadow(sellb_mat* m, cudaStream_t st, int force) {
    if (t_shadow_build) return 0;                 // the shadow's own build
    free_shadow(m);
    bool from_env = false;
    if (force == -2) {
        const char* e = getenv("SELLB_SHADOW");
        force = (!e || strcmp(e, "auto") == 0) ? -1 : (atoi(e) ? 1 : 0);
        from_env = true;
    }
    if (force == 0) return 0;
    const bool possible = m->rl && m->n_rows > 0 && m->nnz > 0 && m->n_chunks > 0 &&
                          m->n_pad < (1LL << 31) - 64;
    if (!possible) {
        if (force == 1 && !from_env)
            return set_error(SELLB_EPARAM, "the shadow layout needs row_lengths and entries");
        return 0;
    }
    const int64_t vs = (int64_t)vsize(m->dtype);
    // x in L2: one global scope (SELL-32-N; where a row lands does not matter
    // to its gathers).  x far larger than L2: 512-row windows, so the rows a
    // chunk holds stay neighbours and the x lines they gather stay shared
    // (cfg5 at sigma = 1 vs 512: 857 vs 1002 GF/s)
    double x_max = 48.0 * (1 << 20);
    if (const char* e = getenv("SELLB_SHADOW_X_MAX")) x_max = atof(e);
    const bool x_in_l2 = (double)m->n_cols * (double)vs <= x_max;
    const int64_t sh_sigma = x_in_l2 ? m->n_pad : 512;
    const bool cost_model = force < 0;
    if (force < 0) {
        const double beta = m->slots ? (double)m->nnz / (double)m->slots : 1.0;
        const bool sorted = m->C == 32 && m->sigma_eff >= std::min<int64_t>(sh_sigma, m->n_pad);
        // C != 32 layouts are candidates whatever their occupancy: the shadow
        // runs them through the C = 32 kernels (one warp per chunk), which
        // the generic-C instances trail (cfg4 sigma = N: C = 8 / 128 at
        // 0.76 / 0.79 of the roofline vs 0.87 for C = 32)
        if (sorted || (beta >= 0.9 && m->C == 32)) return 0;
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
        if (2.0 * (double)m->nnz * (double)(vs + 4) > 0.5 * (double)free_b) return 0;
    }
    static const bool trace = getenv("SELLB_BUILD_TRACE") != nullptr;
    const auto t_begin = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(st);
        fprintf(stderr, "shadow %-12s %9.3f ms\n", what,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                          t_begin).count());
    };
    // 1. the caller's stored rows as a CRS (every row, slot order)
    const int64_t n = m->n_pad;
    DBuf d_len, d_rpt, d_tmp;
    BigBuf d_col, d_val;
    SELLB_CU(d_len.alloc((n + 1) * 8, st));
    SELLB_CU(d_rpt.alloc((n + 1) * 8, st));
    SELLB_CU(cudaMemsetAsync(d_len.p, 0, 8, st));
    k_packed_len<<<(unsigned)grid_for(n, 256), 256, 0, st>>>(m->rl, m->cl, nullptr, 0x7fffffff, n,
                                                             m->C, d_len.as<int64_t>() + 1);
    size_t tmp_bytes = 0;
    SELLB_CU(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, d_len.as<int64_t>(),
                                           d_rpt.as<int64_t>(), n + 1, st));
    SELLB_CU(d_tmp.alloc(tmp_bytes, st));
    SELLB_CU(cub::DeviceScan::InclusiveSum(d_tmp.p, tmp_bytes, d_len.as<int64_t>(),
                                           d_rpt.as<int64_t>(), n + 1, st));
    SELLB_CU(d_col.alloc(m->nnz * 4));
    SELLB_CU(d_val.alloc(m->nnz * vs));
    const unsigned grid = (unsigned)grid_for(n * 32, 256);
    if (m->dtype == SELLB_F32)
        k_packed_fill<float><<<grid, 256, 0, st>>>(m->cs, m->rl, m->col, (const float*)m->val, n,
                                                  m->C, d_rpt.as<int64_t>(), d_col.as<int32_t>(),
                                                  d_val.as<float>());
    else
        k_packed_fill<double><<<grid, 256, 0, st>>>(m->cs, m->rl, m->col, (const double*)m->val,
                                                   n, m->C, d_rpt.as<int64_t>(),
                                                   d_col.as<int32_t>(), d_val.as<double>());
    if (int rc = check_stream_error()) return rc;
    mark("stored CRS");
    // 2. candidate layouts of those rows (the device builder), each with its
    // output maps.  SELL-32 at sh_sigma first; for C != 32 callers also
    // SELL-32-1 of the stored order (their own rows in C = 32 chunks: what
    // the C = 32 kernels run best when sorting does not pay, cfg4)
    struct Cand {
        sellb_mat* sh = nullptr;
        int32_t* ord_st = nullptr;
        int32_t* ord_or = nullptr;
        float t = 3.0e38f;
    };
    auto free_cand = [](Cand& c) {
        if (c.sh) { free_mat_arrays(c.sh); delete c.sh; }
        cudaFree(c.ord_st);
        cudaFree(c.ord_or);
        c = Cand();
    };
    auto build_cand = [&](int64_t sig, Cand& c) -> int {
        t_shadow_build = true;
        const int rc_b = sellb_build_from_crs(d_rpt.as<int64_t>(), d_col.as<int32_t>(), d_val.p,
                                              m->dtype, n, m->n_cols, 32,
                                              std::min<int64_t>(sig, n), 1, 0, m->device, st, 1,
                                              &c.sh);
        t_shadow_build = false;
        if (rc_b) return rc_b;
        // the shadow keeps the variant its cost model chose (the pad-inclusive
        // kernels skip its padding when x[0] is not finite) and never has a
        // packed copy of its own (t_shadow_build)
        sellb_mat* sh = c.sh;
        if (int rc = alloc_dev((void**)&c.ord_st, sh->n_pad * 4)) { free_cand(c); return rc; }
        if (int rc = alloc_dev((void**)&c.ord_or, sh->n_pad * 4)) { free_cand(c); return rc; }
        k_shadow_maps<<<(unsigned)grid_for(sh->n_pad, 256), 256, 0, st>>>(
            sh->order, sh->n_rows, sh->n_pad, m->rl, m->cl, m->C, m->order, m->n_rows, m->n_pad,
            c.ord_st, c.ord_or);
        if (int rc = check_stream_error()) { free_cand(c); return rc; }
        SELLB_CU(cudaStreamSynchronize(st));
        return 0;
    };
    auto install = [&](Cand& c) {
        m->shadow = c.sh;
        m->sh_ord_st = c.ord_st;
        m->sh_ord_or = c.ord_or;
    };
    auto uninstall = [&]() {
        m->shadow = nullptr;
        m->sh_ord_st = nullptr;
        m->sh_ord_or = nullptr;
    };
    const bool timed = cost_model &&
                       !(getenv("SELLB_SHADOW_TIME") && !atoi(getenv("SELLB_SHADOW_TIME")));
    std::vector<int64_t> sigmas{sh_sigma};
    if (timed && m->C != 32) sigmas.push_back(1);
    Cand best;
    for (size_t i = 0; i < sigmas.size(); ++i) {
        if (i > 0) {   // room for one more copy of the entries next to the kept one
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
            if ((double)m->nnz * (double)(vs + 4) > 0.5 * (double)free_b) break;
        }
        Cand c;
        if (int rc = build_cand(sigmas[i], c)) { free_cand(best); return rc; }
        mark("layout+maps");
        if (!timed) { install(c); return 0; }
        install(c);
        float t_base = 0.0f, t_shadow = 0.0f;
        const int rc_t = time_shadow_choice(m, st, &t_base, &t_shadow);
        uninstall();
        if (rc_t) { free_cand(c); free_cand(best); return rc_t; }
        if (trace)
            fprintf(stderr, "shadow timed: as built %.4f ms, SELL-32-%lld shadow %.4f ms\n",
                    t_base, (long long)std::min<int64_t>(sigmas[i], n), t_shadow);
        mark("timed");
        c.t = t_shadow;
        if (t_shadow < 0.95f * t_base && t_shadow < best.t) {   // a clear win only
            free_cand(best);
            best = c;
        } else {
            free_cand(c);
        }
    }
    if (best.sh) install(best);
    return 0;
}

}  // namespace sellb

// ===========================================================================
// ABI
// ===========================================================================
extern "C" {

int sellb_build_from_crs(const int64_t* rpt, const int32_t* col, const void* val, int32_t dtype,
                         int64_t n_rows, int64_t n_cols, int32_t C, int64_t sigma,
                         int32_t align_bytes, int32_t permute_cols, int32_t device, void* stream,
                         int32_t ptrs_on_device, sellb_mat** out) {
    clear_error();
    NvtxRange nvtx_("sellb_build_from_crs");
    if (!out) return set_error(SELLB_EPARAM, "out must not be NULL");
    *out = nullptr;
    // parameter checks in the reference's order (formats.py:309-319)
    if (C < 1) return set_error(SELLB_EPARAM, "chunk height C must be >= 1, got %d", C);
    if (sigma < 1) return set_error(SELLB_EPARAM, "sigma must be >= 1, got %lld", (long long)sigma);
    if (align_bytes != 1 && align_bytes != 64)
        return set_error(SELLB_EPARAM, "align_bytes must be 1 or 64, got %d", align_bytes);
    if (permute_cols && n_rows != n_cols)
        return set_error(SELLB_EPARAM,
                         "column permutation requires a square matrix (got %lldx%lld); rows "
                         "and columns share one index space",
                         (long long)n_rows, (long long)n_cols);
    if (dtype != SELLB_F64 && dtype != SELLB_F32)
        return set_error(SELLB_EPARAM, "dtype must be SELLB_F64 or SELLB_F32");
    if (n_rows < 0 || n_cols < 0)
        return set_error(SELLB_ESTRUCT, "negative matrix dimension (%lldx%lld)", (long long)n_rows,
                         (long long)n_cols);
    if (n_rows >= (1LL << 31) || n_cols >= (1LL << 31))
        return set_error(SELLB_ESTRUCT, "matrix dimension exceeds 4-byte index range");
    if (!rpt) return set_error(SELLB_EPARAM, "rpt must not be NULL");

    const int64_t n = n_rows;
    const int64_t n_pad = n ? ((n + C - 1) / C) * C : 0;
    const int64_t n_chunks = n_pad / C;
    if (n_pad >= (1LL << 31)) return set_error(SELLB_ESTRUCT, "padded row count exceeds int32");
    const int64_t sigma_eff = sigma_effective(n, C, sigma, n_pad);
    if (sigma_eff < 0)
        return set_error(SELLB_EPARAM,
                         "sigma (%lld) must be a multiple of C (%d) when C < sigma < n_rows",
                         (long long)sigma, C);

    DeviceGuard guard(device);
    if (!guard.ok) return set_error(SELLB_ERESOURCE, "cannot select CUDA device %d", device);
    cudaStream_t st = (cudaStream_t)stream;
    PoolTrim trim_(st);
    const size_t vs = vsize(dtype);
    // SELLB_BUILD_TRACE=1: synchronise after each phase and print its end time
    static const bool trace = getenv("SELLB_BUILD_TRACE") != nullptr;
    const auto t_begin = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(st);
        fprintf(stderr, "build %-12s %9.3f ms\n", what,
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                          t_begin).count());
    };

    // --- inputs on device -------------------------------------------------
    int64_t rpt_host_last = 0, rpt_host_first = 0;
    if (ptrs_on_device) {
        SELLB_CU(cudaMemcpyAsync(&rpt_host_first, rpt, 8, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaMemcpyAsync(&rpt_host_last, rpt + n, 8, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
    } else {
        rpt_host_first = rpt[0];
        rpt_host_last = rpt[n];
    }
    if (n && rpt_host_first != 0) return set_error(SELLB_ESTRUCT, "rpt[0] must be 0");
    const int64_t nnz = rpt_host_last;
    if (nnz < 0) return set_error(SELLB_ESTRUCT, "rpt[-1] must be >= 0");
    if (nnz && (!col || !val)) return set_error(SELLB_EPARAM, "col/val must not be NULL");

    DBuf d_rpt;
    BigBuf d_col, d_val;
    const int64_t* rpt_d = rpt;
    const int32_t* col_d = col;
    const void* val_d = val;
    if (!ptrs_on_device) {
        SELLB_CU(d_rpt.alloc((n + 1) * 8, st));
        SELLB_CU(cudaMemcpyAsync(d_rpt.p, rpt, (n + 1) * 8, cudaMemcpyHostToDevice, st));
        SELLB_CU(d_col.alloc(nnz * 4));
        SELLB_CU(d_val.alloc(nnz * vs));
        if (nnz) {
            SELLB_CU(cudaMemcpyAsync(d_col.p, col, nnz * 4, cudaMemcpyHostToDevice, st));
            SELLB_CU(cudaMemcpyAsync(d_val.p, val, nnz * vs, cudaMemcpyHostToDevice, st));
        }
        rpt_d = d_rpt.as<int64_t>();
        col_d = d_col.as<int32_t>();
        val_d = d_val.p;
    }

    sellb_mat* m = new (std::nothrow) sellb_mat();
    if (!m) return set_error(SELLB_ERESOURCE, "host allocation failed");
    struct Holder {
        sellb_mat* m;
        ~Holder() { if (m) { free_mat_arrays(m); delete m; } }
    } holder{m};
    m->n_rows = n; m->n_cols = n_cols; m->C = C; m->sigma = sigma; m->sigma_eff = sigma_eff;
    m->n_pad = n_pad; m->n_chunks = n_chunks; m->nnz = nnz; m->dtype = dtype;
    m->device = device; m->col_permuted = permute_cols ? 1 : 0;
    m->variant = SELLB_VARIANT_AUTO;

    // --- 1. lengths + checks ------------------------------------------------
    DBuf d_len, d_flags;
    SELLB_CU(d_len.alloc(n_pad * 4, st));
    SELLB_CU(d_flags.alloc(16, st));
    SELLB_CU(cudaMemsetAsync(d_flags.p, 0, 16, st));
    unsigned int* d_maxlen = d_flags.as<unsigned int>();
    int* d_bad = reinterpret_cast<int*>(d_flags.as<unsigned int>() + 1);
    if (n_pad)
        k_row_lengths<<<(unsigned)std::min<int64_t>(grid_for(n_pad, 256), 148 * 8), 256, 0, st>>>(
            rpt_d, n, n_pad,
                                                                       d_len.as<int32_t>(),
                                                                       d_maxlen, d_bad);
    if (nnz && permute_cols) {      // otherwise checked by k_fill
        int blocks = (int)std::min<int64_t>(grid_for(nnz, 256), 148 * 16);
        k_check_cols<<<blocks, 256, 0, st>>>(col_d, nnz, n_cols, d_bad);
    }
    if (int rc = check_stream_error()) return rc;
    unsigned int hflags[2] = {0, 0};
    SELLB_CU(cudaMemcpyAsync(hflags, d_flags.p, 8, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    if (hflags[1] == 1) return set_error(SELLB_ESTRUCT, "rpt must be non-decreasing");
    if (hflags[1] == 2) return set_error(SELLB_ESTRUCT, "column index out of bounds");
    const unsigned int maxlen = hflags[0];
    mark("lengths");

    // --- 2.-4. scope sort, perm / row_lengths / order, chunk widths ---------
    {   // one allocation for the five row / chunk arrays (five cudaMalloc calls
        // of up to 256 MB each cost ~1.5 ms on cfg5)
        auto up = [](int64_t b) { return (b + 255) / 256 * 256; };
        const int64_t b_cs = up((n_chunks + 1) * 8), b_cl = up(std::max<int64_t>(n_chunks, 1) * 4);
        const int64_t b_perm = up(std::max<int64_t>(n, 1) * 4);
        const int64_t b_row = up(std::max<int64_t>(n_pad, 1) * 4);
        if (int rc = alloc_dev(&m->meta_slab, b_cs + b_cl + b_perm + 2 * b_row)) return rc;
        char* q = static_cast<char*>(m->meta_slab);
        m->cs = reinterpret_cast<int64_t*>(q);
        m->cl = reinterpret_cast<int32_t*>(q + b_cs);
        m->perm = reinterpret_cast<int32_t*>(q + b_cs + b_cl);
        m->rl = reinterpret_cast<int32_t*>(q + b_cs + b_cl + b_perm);
        m->order = reinterpret_cast<int32_t*>(q + b_cs + b_cl + b_perm + b_row);
    }
    SELLB_CU(cudaMemsetAsync(m->cs, 0, 8, st));
    int64_t unit = 1;
    if (align_bytes > 1) {
        int64_t a = 4LL * C, b = align_bytes;
        while (b) { int64_t t = a % b; a = b; b = t; }
        unit = align_bytes / a;   // formats.py:354
    }
    DBuf d_slots;
    if (n_chunks) SELLB_CU(d_slots.alloc(n_chunks * 8, st));
    const int lbits = std::max(1, bits_for(maxlen));
    bool widths_done = false;
    if (sigma_eff > 1 && n_pad > 1 && sigma_eff <= 4096) {
        // one CTA per sigma window: sort + order + widths in one launch
        const unsigned n_scopes = (unsigned)((n_pad + sigma_eff - 1) / sigma_eff);
#define SELLB_SCOPE_SORT(TH, IT)                                                              \
        k_scope_sort<TH, IT><<<n_scopes, TH, 0, st>>>(d_len.as<int32_t>(), n, n_pad, sigma_eff, \
                                                    lbits, maxlen, C, unit, m->perm, m->rl,     \
                                                    m->order, m->cl, d_slots.as<int64_t>())
        if (sigma_eff <= 512) SELLB_SCOPE_SORT(128, 4);
        else if (sigma_eff <= 1024) SELLB_SCOPE_SORT(128, 8);
        else if (sigma_eff <= 2048) SELLB_SCOPE_SORT(256, 8);
        else SELLB_SCOPE_SORT(512, 8);
#undef SELLB_SCOPE_SORT
        widths_done = true;
    } else if (sigma_eff > 1 && n_pad > 1) {
        // wide scopes: stable device radix sort of (scope, maxlen - len) with
        // the index as payload == np.lexsort((idx, -len, scope))
        const int64_t n_scopes = (n_pad + sigma_eff - 1) / sigma_eff;
        const int sbits = n_scopes > 1 ? bits_for((uint64_t)(n_scopes - 1)) : 0;
        const int total_bits = lbits + sbits;
        DBuf d_idx_in, d_sorted_idx, d_keys_in, d_keys_out, d_tmp;
        SELLB_CU(d_idx_in.alloc(n_pad * 4, st));
        SELLB_CU(d_sorted_idx.alloc(n_pad * 4, st));
        size_t tmp_bytes = 0;
        if (total_bits <= 32) {
            SELLB_CU(d_keys_in.alloc(n_pad * 4, st));
            SELLB_CU(d_keys_out.alloc(n_pad * 4, st));
            k_sort_keys<uint32_t><<<(unsigned)grid_for(n_pad, 256), 256, 0, st>>>(
                d_len.as<int32_t>(), n_pad, sigma_eff, lbits, maxlen, d_keys_in.as<uint32_t>(),
                d_idx_in.as<int32_t>());
            SELLB_CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_keys_in.as<uint32_t>(),
                                                     d_keys_out.as<uint32_t>(),
                                                     d_idx_in.as<int32_t>(),
                                                     d_sorted_idx.as<int32_t>(), (int)n_pad, 0,
                                                     total_bits, st));
            SELLB_CU(d_tmp.alloc(tmp_bytes, st));
            SELLB_CU(cub::DeviceRadixSort::SortPairs(d_tmp.p, tmp_bytes, d_keys_in.as<uint32_t>(),
                                                     d_keys_out.as<uint32_t>(),
                                                     d_idx_in.as<int32_t>(),
                                                     d_sorted_idx.as<int32_t>(), (int)n_pad, 0,
                                                     total_bits, st));
        } else {
            SELLB_CU(d_keys_in.alloc(n_pad * 8, st));
            SELLB_CU(d_keys_out.alloc(n_pad * 8, st));
            k_sort_keys<uint64_t><<<(unsigned)grid_for(n_pad, 256), 256, 0, st>>>(
                d_len.as<int32_t>(), n_pad, sigma_eff, lbits, maxlen, d_keys_in.as<uint64_t>(),
                d_idx_in.as<int32_t>());
            SELLB_CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_keys_in.as<uint64_t>(),
                                                     d_keys_out.as<uint64_t>(),
                                                     d_idx_in.as<int32_t>(),
                                                     d_sorted_idx.as<int32_t>(), (int)n_pad, 0,
                                                     total_bits, st));
            SELLB_CU(d_tmp.alloc(tmp_bytes, st));
            SELLB_CU(cub::DeviceRadixSort::SortPairs(d_tmp.p, tmp_bytes, d_keys_in.as<uint64_t>(),
                                                     d_keys_out.as<uint64_t>(),
                                                     d_idx_in.as<int32_t>(),
                                                     d_sorted_idx.as<int32_t>(), (int)n_pad, 0,
                                                     total_bits, st));
        }
        k_apply_order<<<(unsigned)grid_for(n_pad, 256), 256, 0, st>>>(
            d_sorted_idx.as<int32_t>(), d_len.as<int32_t>(), n, n_pad, m->perm, m->rl, m->order);
    } else if (n_pad) {
        k_identity_order<<<(unsigned)grid_for(n_pad, 256), 256, 0, st>>>(
            d_len.as<int32_t>(), n, n_pad, m->perm, m->rl, m->order);
    }
    mark("sort+widths");
    // --- 5. cs = [0, cumsum(C * cl)] -------------------------------------------
    if (n_chunks) {
        if (!widths_done)
            k_chunk_width<<<(unsigned)grid_for(n_chunks * 32, 256), 256, 0, st>>>(
                m->rl, n_chunks, C, unit, m->cl, d_slots.as<int64_t>());
        DBuf d_tmp;
        size_t tmp_bytes = 0;
        SELLB_CU(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, d_slots.as<int64_t>(),
                                               m->cs + 1, (int)n_chunks, st));
        SELLB_CU(d_tmp.alloc(tmp_bytes, st));
        SELLB_CU(cub::DeviceScan::InclusiveSum(d_tmp.p, tmp_bytes, d_slots.as<int64_t>(),
                                               m->cs + 1, (int)n_chunks, st));
    }
    if (int rc = check_stream_error()) return rc;
    int64_t total = 0;
    SELLB_CU(cudaMemcpyAsync(&total, m->cs + n_chunks, 8, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    m->slots = total;
    // the widest chunk holds the longest row: max cl = maxlen rounded to the unit
    m->max_cl = n_chunks ? (int32_t)(((int64_t)maxlen + unit - 1) / unit * unit) : 0;

    mark("cs");
    // --- 6. fill -------------------------------------------------------------
    if (int rc = alloc_dev((void**)&m->col, total * 4)) return rc;
    if (int rc = alloc_dev(&m->val, total * vs)) return rc;
    mark("alloc");
    if (n_pad && total) {
        const unsigned grid = (unsigned)grid_for(n_pad, 256);
        int* const chk = permute_cols ? nullptr : d_bad;
        // U = 4 (U = 1: same 6.9 ms on cfg5; U = 8 slower; a warp-per-32-rows
        // transpose through shared memory: 19.7 ms, too few loads in flight).
        // cfg5: 33.3 GB of DRAM traffic (= the algorithmic bytes) in 6.55 ms
        if (dtype == SELLB_F64)
            k_fill<double, 4><<<grid, 256, 0, st>>>(rpt_d, col_d, (const double*)val_d, n, n_pad, C,
                                                    m->order, m->rl, m->cs, m->cl, m->perm,
                                                    permute_cols ? 1 : 0, m->col,
                                                    (double*)m->val, n_cols, chk);
        else
            k_fill<float, 4><<<grid, 256, 0, st>>>(rpt_d, col_d, (const float*)val_d, n, n_pad, C,
                                                   m->order, m->rl, m->cs, m->cl, m->perm,
                                                   permute_cols ? 1 : 0, m->col, (float*)m->val,
                                                   n_cols, chk);
    }
    if (int rc = check_stream_error()) return rc;
    if (nnz && !permute_cols) {
        int hbad = 0;
        SELLB_CU(cudaMemcpyAsync(&hbad, d_bad, 4, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        if (hbad == 2) return set_error(SELLB_ESTRUCT, "column index out of bounds");
    }
    mark("fill");
    if (int rc = choose_variant(m, st, nullptr, nullptr, nullptr)) return rc;
    mark("variant");
    if (int rc = build_long_rows(m, st)) return rc;
    mark("long rows");
    if (int rc = build_packed(m, st, -2)) return rc;
    mark("packed");
    if (int rc = build_shadow(m, st, -2)) return rc;
    SELLB_CU(cudaStreamSynchronize(st));
    mark("shadow");
    holder.m = nullptr;
    *out = m;
    return 0;
}

int sellb_import(const int64_t* cs, const int32_t* cl, const int32_t* col, const void* val,
                 const int32_t* perm, const int32_t* row_lengths, int32_t dtype, int64_t n_rows,
                 int64_t n_cols, int32_t C, int64_t sigma, int64_t n_chunks, int64_t n_slots,
                 int32_t col_permuted, int32_t device, void* stream, int32_t ptrs_on_device,
                 sellb_mat** out) {
    clear_error();
    NvtxRange nvtx_("sellb_import");
    if (!out) return set_error(SELLB_EPARAM, "out must not be NULL");
    *out = nullptr;
    if (C < 1) return set_error(SELLB_EPARAM, "chunk height C must be >= 1, got %d", C);
    if (dtype != SELLB_F64 && dtype != SELLB_F32)
        return set_error(SELLB_EPARAM, "dtype must be SELLB_F64 or SELLB_F32");
    if (n_rows < 0 || n_cols < 0 || n_chunks < 0)
        return set_error(SELLB_ESTRUCT, "negative dimension");
    if (n_chunks * (int64_t)C < n_rows || (n_rows && n_chunks * (int64_t)C >= n_rows + C))
        return set_error(SELLB_ESTRUCT, "n_rows_padded must be n_rows rounded up to C");
    if (!cs || (n_chunks && !cl)) return set_error(SELLB_EPARAM, "cs/cl must not be NULL");
    DeviceGuard guard(device);
    if (!guard.ok) return set_error(SELLB_ERESOURCE, "cannot select CUDA device %d", device);
    cudaStream_t st = (cudaStream_t)stream;
    PoolTrim trim_(st);
    cudaMemcpyKind kind = ptrs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    int64_t total = 0;
    if (ptrs_on_device) {
        SELLB_CU(cudaMemcpyAsync(&total, cs + n_chunks, 8, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
    } else {
        total = cs[n_chunks];
    }
    if (total < 0) return set_error(SELLB_ESTRUCT, "cs[n_chunks] must be >= 0");
    // the caller's col / val buffers hold n_slots entries: never read past them
    if (total != n_slots)
        return set_error(SELLB_ESTRUCT, "col/val length must equal cs[n_chunks]");
    if (total && (!col || !val)) return set_error(SELLB_EPARAM, "col/val must not be NULL");
    if (total && n_cols == 0) return set_error(SELLB_ESTRUCT, "stored slots require n_cols >= 1");
    sellb_mat* m = new (std::nothrow) sellb_mat();
    if (!m) return set_error(SELLB_ERESOURCE, "host allocation failed");
    struct Holder {
        sellb_mat* m;
        ~Holder() { if (m) { free_mat_arrays(m); delete m; } }
    } holder{m};
    const size_t vs = vsize(dtype);
    m->n_rows = n_rows; m->n_cols = n_cols; m->C = C; m->sigma = sigma;
    m->n_pad = n_chunks * C; m->n_chunks = n_chunks; m->slots = total; m->dtype = dtype;
    m->device = device; m->col_permuted = col_permuted;
    m->sigma_eff = sigma_effective(n_rows, C, sigma, m->n_pad);
    if (int rc = alloc_dev((void**)&m->cs, (n_chunks + 1) * 8)) return rc;
    if (int rc = alloc_dev((void**)&m->cl, std::max<int64_t>(n_chunks, 1) * 4)) return rc;
    if (int rc = alloc_dev((void**)&m->col, total * 4)) return rc;
    if (int rc = alloc_dev(&m->val, total * vs)) return rc;
    SELLB_CU(cudaMemcpyAsync(m->cs, cs, (n_chunks + 1) * 8, kind, st));
    if (n_chunks) SELLB_CU(cudaMemcpyAsync(m->cl, cl, n_chunks * 4, kind, st));
    if (total) {
        SELLB_CU(cudaMemcpyAsync(m->col, col, total * 4, kind, st));
        SELLB_CU(cudaMemcpyAsync(m->val, val, total * vs, kind, st));
    }
    // the reference's SellMatrix invariants (formats.py:210-251) on the device:
    // cs[0] == 0, cs[i+1] - cs[i] == C * cl[i], 0 <= col < n_cols -- the
    // kernels index x and the arrays by them
    {
        DBuf d_bad;
        SELLB_CU(d_bad.alloc(4, st));
        SELLB_CU(cudaMemsetAsync(d_bad.p, 0, 4, st));
        k_check_layout<<<(unsigned)grid_for(std::max<int64_t>(n_chunks, 1), 256), 256, 0, st>>>(
            m->cs, m->cl, n_chunks, C, d_bad.as<int>());
        if (total) {
            int blocks = (int)std::min<int64_t>(grid_for(total, 256), 148 * 16);
            k_check_cols<<<blocks, 256, 0, st>>>(m->col, total, n_cols, d_bad.as<int>());
        }
        if (int rc = check_stream_error()) return rc;
        int bad = 0;
        SELLB_CU(cudaMemcpyAsync(&bad, d_bad.p, 4, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        if (bad == 3) return set_error(SELLB_ESTRUCT, "cs[0] must be 0");
        if (bad == 4) return set_error(SELLB_ESTRUCT, "cs[i+1] - cs[i] must equal C * cl[i]");
        if (bad == 2) return set_error(SELLB_ESTRUCT, "column index out of bounds");
    }
    if (perm && n_rows) {
        if (int rc = alloc_dev((void**)&m->perm, n_rows * 4)) return rc;
        SELLB_CU(cudaMemcpyAsync(m->perm, perm, n_rows * 4, kind, st));
        // stored -> original map for the fused unpermute epilogue
        if (int rc = alloc_dev((void**)&m->order, std::max<int64_t>(m->n_pad, 1) * 4)) return rc;
        std::vector<int32_t> h_perm(n_rows), h_order(m->n_pad);
        SELLB_CU(cudaMemcpyAsync(h_perm.data(), m->perm, n_rows * 4, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        for (int64_t p = 0; p < n_rows; ++p) h_order[p] = -1;
        for (int64_t p = n_rows; p < m->n_pad; ++p) h_order[p] = (int32_t)p;   // padding rows
        for (int64_t i = 0; i < n_rows; ++i) {
            int32_t p = h_perm[i];
            if (p < 0 || p >= n_rows || h_order[p] != -1)
                return set_error(SELLB_ESTRUCT, "perm must be a permutation of 0..n_rows-1");
            h_order[p] = (int32_t)i;
        }
        SELLB_CU(cudaMemcpyAsync(m->order, h_order.data(), m->n_pad * 4, cudaMemcpyHostToDevice, st));
        SELLB_CU(cudaStreamSynchronize(st));
    }
    // max cl
    if (n_chunks) {
        std::vector<int32_t> h_cl(n_chunks);
        SELLB_CU(cudaMemcpyAsync(h_cl.data(), m->cl, n_chunks * 4, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        int32_t mx = 0;
        for (auto v : h_cl) mx = std::max(mx, v);
        m->max_cl = mx;
    }
    if (row_lengths && m->n_pad) {
        if (int rc = alloc_dev((void**)&m->rl, m->n_pad * 4)) return rc;
        SELLB_CU(cudaMemcpyAsync(m->rl, row_lengths, m->n_pad * 4, kind, st));
        std::vector<int32_t> h_rl(m->n_pad);
        SELLB_CU(cudaMemcpyAsync(h_rl.data(), m->rl, m->n_pad * 4, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        std::vector<int32_t> h_cl(n_chunks);
        SELLB_CU(cudaMemcpy(h_cl.data(), m->cl, n_chunks * 4, cudaMemcpyDeviceToHost));
        int64_t s = 0;
        for (int64_t p = 0; p < m->n_pad; ++p) {
            const int32_t v = h_rl[p];
            if (v < 0 || v > h_cl[p / C])
                return set_error(SELLB_ESTRUCT, "row length outside [0, cl] for its chunk");
            if (p >= n_rows && v != 0)
                return set_error(SELLB_ESTRUCT, "padding rows must have length 0");
            s += v;
        }
        m->nnz = s;
        m->variant = SELLB_VARIANT_AUTO;
        if (int rc = choose_variant(m, st, nullptr, nullptr, nullptr)) return rc;
        if (int rc = build_long_rows(m, st)) return rc;
    if (int rc = build_packed(m, st, -2)) return rc;
    if (int rc = build_shadow(m, st, -2)) return rc;
    } else {
        m->nnz = -1;   // unknown without row_lengths
        m->variant = SELLB_VARIANT_PAD_INCL;
    }
    SELLB_CU(cudaStreamSynchronize(st));
    holder.m = nullptr;
    *out = m;
    return 0;
}

int sellb_info(const sellb_mat* m, sellb_info_t* info) {
    clear_error();
    if (!m || !info) return set_error(SELLB_EPARAM, "NULL argument");
    info->n_rows = m->n_rows; info->n_cols = m->n_cols; info->C = m->C; info->sigma = m->sigma;
    info->sigma_eff = m->sigma_eff; info->n_rows_padded = m->n_pad; info->n_chunks = m->n_chunks;
    info->slots = m->slots; info->nnz = m->nnz; info->dtype = m->dtype; info->device = m->device;
    info->col_permuted = m->col_permuted; info->variant = m->variant;
    info->has_row_lengths = m->rl != nullptr; info->max_cl = m->max_cl;
    info->packed = m->pcol != nullptr;
    info->shadow = m->shadow ? (int32_t)m->shadow->sigma : 0;
    return 0;
}

int sellb_long_info(const sellb_mat* m, int64_t* n_long, int64_t* n_groups, int64_t* n_rest,
                    int64_t* side_entries) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    int64_t side = 0;
    if (m->side_off && m->n_rest) {
        int64_t last = 0;
        if (cudaMemcpy(&last, m->side_off + m->n_rest, 8, cudaMemcpyDeviceToHost) != cudaSuccess)
            return set_error(SELLB_ERESOURCE, "side-table offset read failed");
        side = last;
    }
    if (n_long) *n_long = m->n_long;
    if (n_groups) *n_groups = m->n_groups;
    if (n_rest) *n_rest = m->n_rest;
    if (side_entries) *side_entries = side;
    return 0;
}

int sellb_device_arrays(const sellb_mat* m, sellb_dev_arrays_t* o) {
    clear_error();
    if (!m || !o) return set_error(SELLB_EPARAM, "NULL argument");
    o->cs = m->cs; o->cl = m->cl; o->col = m->col; o->val = m->val; o->perm = m->perm;
    o->order = m->order; o->row_lengths = m->rl;
    return 0;
}

int sellb_export(const sellb_mat* m, int64_t* cs, int32_t* cl, int32_t* col, void* val,
                 int32_t* perm, int32_t* row_lengths, void* stream, int32_t ptrs_on_device) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    DeviceGuard guard(m->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemcpyKind kind = ptrs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (cs) SELLB_CU(cudaMemcpyAsync(cs, m->cs, (m->n_chunks + 1) * 8, kind, st));
    if (cl && m->n_chunks) SELLB_CU(cudaMemcpyAsync(cl, m->cl, m->n_chunks * 4, kind, st));
    if (col && m->slots) SELLB_CU(cudaMemcpyAsync(col, m->col, m->slots * 4, kind, st));
    if (val && m->slots) SELLB_CU(cudaMemcpyAsync(val, m->val, m->slots * vsize(m->dtype), kind, st));
    if (perm && m->n_rows) {
        if (!m->perm) return set_error(SELLB_EPARAM, "matrix has no permutation");
        SELLB_CU(cudaMemcpyAsync(perm, m->perm, m->n_rows * 4, kind, st));
    }
    if (row_lengths && m->n_pad) {
        if (!m->rl) return set_error(SELLB_EPARAM, "matrix has no row_lengths");
        SELLB_CU(cudaMemcpyAsync(row_lengths, m->rl, m->n_pad * 4, kind, st));
    }
    SELLB_CU(cudaStreamSynchronize(st));
    return 0;
}

int sellb_export_range(const sellb_mat* m, int64_t c0, int64_t c1, int64_t* cs, int32_t* cl,
                       int32_t* col, void* val, int32_t* row_lengths) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    if (c0 < 0 || c1 > m->n_chunks || c0 > c1) return set_error(SELLB_EPARAM, "bad chunk range");
    DeviceGuard guard(m->device);
    const int64_t nc = c1 - c0;
    std::vector<int64_t> hcs(nc + 1);
    SELLB_CU(cudaMemcpy(hcs.data(), m->cs + c0, (nc + 1) * 8, cudaMemcpyDeviceToHost));
    const int64_t s0 = hcs[0], s1 = hcs[nc];
    if (cs)
        for (int64_t i = 0; i <= nc; ++i) cs[i] = hcs[i] - s0;
    if (cl && nc) SELLB_CU(cudaMemcpy(cl, m->cl + c0, nc * 4, cudaMemcpyDeviceToHost));
    if (col && s1 > s0)
        SELLB_CU(cudaMemcpy(col, m->col + s0, (s1 - s0) * 4, cudaMemcpyDeviceToHost));
    if (val && s1 > s0)
        SELLB_CU(cudaMemcpy(val, (const char*)m->val + s0 * vsize(m->dtype),
                            (s1 - s0) * vsize(m->dtype), cudaMemcpyDeviceToHost));
    if (row_lengths && nc) {
        if (!m->rl) return set_error(SELLB_EPARAM, "matrix has no row_lengths");
        SELLB_CU(cudaMemcpy(row_lengths, m->rl + c0 * m->C, nc * m->C * 4,
                            cudaMemcpyDeviceToHost));
    }
    return 0;
}

int sellb_infer_row_lengths(sellb_mat* m, void* stream) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    DeviceGuard guard(m->device);
    cudaStream_t st = (cudaStream_t)stream;
    PoolTrim trim_(st);
    if (!m->rl && m->n_pad)
        if (int rc = alloc_dev((void**)&m->rl, m->n_pad * 4)) return rc;
    if (m->n_pad) {
        if (m->dtype == SELLB_F32)
            k_trailing_len<float><<<(unsigned)grid_for(m->n_pad, 256), 256, 0, st>>>(
                m->cs, m->cl, m->col, (const float*)m->val, m->n_pad, m->C, m->rl);
        else
            k_trailing_len<double><<<(unsigned)grid_for(m->n_pad, 256), 256, 0, st>>>(
                m->cs, m->cl, m->col, (const double*)m->val, m->n_pad, m->C, m->rl);
        if (int rc = check_stream_error()) return rc;
        std::vector<int32_t> h(m->n_pad);
        SELLB_CU(cudaMemcpyAsync(h.data(), m->rl, m->n_pad * 4, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        int64_t s = 0;
        for (auto v : h) s += v;
        m->nnz = s;
    } else {
        m->nnz = 0;
    }
    m->variant = SELLB_VARIANT_AUTO;
    if (int rc = choose_variant(m, st, nullptr, nullptr, nullptr)) return rc;
    if (int rc = build_long_rows(m, st)) return rc;
    if (int rc = build_packed(m, st, -2)) return rc;
    if (int rc = build_shadow(m, st, -2)) return rc;
    return 0;
}

int sellb_set_variant(sellb_mat* m, int32_t variant) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    if (variant < SELLB_VARIANT_AUTO || variant > SELLB_VARIANT_PAD_INCL)
        return set_error(SELLB_EPARAM, "unknown variant %d", variant);
    if (variant == SELLB_VARIANT_PAD_SKIP && !m->rl)
        return set_error(SELLB_EPARAM, "pad-skipping needs row_lengths");
    DeviceGuard guard(m->device);
    m->variant = variant;
    if (variant == SELLB_VARIANT_AUTO) return choose_variant(m, 0, nullptr, nullptr, nullptr);
    return 0;
}

int sellb_set_packed(sellb_mat* m, int32_t mode) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    if (mode < -1 || mode > 1) return set_error(SELLB_EPARAM, "packed mode must be -1, 0 or 1");
    DeviceGuard guard(m->device);
    PoolTrim trim_(0);
    return build_packed(m, 0, mode);
}

int sellb_set_shadow(sellb_mat* m, int32_t mode) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    if (mode < -1 || mode > 1) return set_error(SELLB_EPARAM, "shadow mode must be -1, 0 or 1");
    DeviceGuard guard(m->device);
    PoolTrim trim_(0);
    return build_shadow(m, 0, mode);
}

void sellb_free(sellb_mat* m) {
    if (!m) return;
    free_mat_arrays(m);
    delete m;
}

double sellb_chunk_occupancy(const sellb_mat* m) {
    // formats.py:274-282
    if (!m || m->slots == 0) return 1.0;
    return (double)m->nnz / (double)m->slots;
}

int sellb_streamed_bytes(const sellb_mat* m, int64_t* matrix_bytes, int64_t* matrix_bytes_64,
                         int64_t* extra_bytes, void* stream) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    DeviceGuard guard(m->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int vs = (int)vsize(m->dtype);
    if (m->shadow) {
        // whole-matrix SpMVs read the shadow layout plus one map entry per row
        if (int rc = sellb_streamed_bytes(m->shadow, matrix_bytes, matrix_bytes_64, extra_bytes,
                                          stream))
            return rc;
        if (extra_bytes) *extra_bytes += 4 * m->shadow->n_pad;
        return 0;
    }
    if (m->pcol && m->variant == SELLB_VARIANT_PAD_SKIP) {
        // the packed stored-order copy: every entry once, contiguous; plus
        // the row offsets and the chunk widths (pad fix-up)
        const int64_t mb = (int64_t)(vs + 4) * m->nnz;
        if (matrix_bytes) *matrix_bytes = mb;
        if (matrix_bytes_64) *matrix_bytes_64 = mb;
        if (extra_bytes) *extra_bytes = 8 * (m->n_pad + 1) + 4 * m->n_chunks;
        return 0;
    }
    unsigned long long h[4] = {0, 0, 0, 0};
    const bool skip = m->variant == SELLB_VARIANT_PAD_SKIP;
    if (m->n_chunks && (m->rl || !skip)) {
        DBuf cnt;
        SELLB_CU(cnt.alloc(sizeof(h), st));
        SELLB_CU(cudaMemsetAsync(cnt.p, 0, sizeof(h), st));
        if (m->rl) {
            k_stream_count<<<(unsigned)grid_for(m->n_chunks, 256), 256, 0, st>>>(
                m->rl, m->cl, m->chunk_th, m->n_chunks, m->C, skip ? 1 : 0, m->long_th, vs,
                cnt.as<unsigned long long>());
            SELLB_CU(cudaGetLastError());
            SELLB_CU(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        } else {
            h[0] = (unsigned long long)m->slots * (vs + 4);
        }
        SELLB_CU(cudaStreamSynchronize(st));
    }
    int64_t side = 0;
    if (int rc = sellb_long_info(m, nullptr, nullptr, nullptr, &side)) return rc;
    const int64_t long_bytes = side * (vs + 4);     // side-table rows read contiguously
    int64_t long_direct = 0;                        // long rows read from the SELL arrays
    if (!side && m->n_long && m->rl) {
        std::vector<int32_t> lr(m->n_long), hrl(m->n_pad);
        SELLB_CU(cudaMemcpy(lr.data(), m->long_rows, m->n_long * 4, cudaMemcpyDeviceToHost));
        SELLB_CU(cudaMemcpy(hrl.data(), m->rl, m->n_pad * 4, cudaMemcpyDeviceToHost));
        for (int32_t p : lr) long_direct += (int64_t)hrl[p] * 32 * 2;   // a sector per value / index
    }
    if (matrix_bytes) *matrix_bytes = (int64_t)(h[0] + h[1]) + long_bytes + long_direct;
    if (matrix_bytes_64) *matrix_bytes_64 = (int64_t)(h[0] + h[2]) + long_bytes + 2 * long_direct;
    if (extra_bytes) *extra_bytes = (int64_t)h[3];
    return 0;
}

int sellb_sector_occupancy(const sellb_mat* m, double* beta_eff, int64_t* val_sectors,
                           int64_t* col_sectors, void* stream) {
    clear_error();
    if (!m) return set_error(SELLB_EPARAM, "NULL matrix");
    if (!m->rl) return set_error(SELLB_EPARAM, "matrix has no row_lengths");
    DeviceGuard guard(m->device);
    sellb_mat* mm = const_cast<sellb_mat*>(m);
    int32_t keep = mm->variant;
    int rc = choose_variant(mm, (cudaStream_t)stream, beta_eff, val_sectors, col_sectors);
    mm->variant = keep;
    return rc;
}

}  // extern "C"
