// sellb_coo.cu -- the step before the hot path on the device (SURVEY.md
// §8(f)3): COO bounds check, canonicalisation (row-major sort, duplicate
// coordinates summed, explicit zeros kept) and CRS row pointers, i.e.
// COOMatrix.__post_init__ (formats.py:50-70) + canonicalize_coo
// (formats.py:89-108) + coo_to_crs (formats.py:169-175).
//
// Bit-exactness of duplicate sums: the reference sums each run of equal
// coordinates with np.add.reduceat over the stable (row, col) order.  NumPy's
// reduceat seeds the run with its first element and adds the rest as ONE
// pairwise sum (NumPy's pairwise_sum: < 8 elements sequentially from -0.0,
// <= 128 elements in eight interleaved partial sums combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail, larger runs split at
// n/2 rounded down to a multiple of 8 and the halves added).  pw_sum below
// evaluates the same expression tree with __dadd_rn, so every summed value
// is the reference's bit for bit (verified against the reference's own
// outputs in tests/golden/coo_*.npz).
//
// Pipeline (one stream, HBM-bound): key = row << cbits | col, stable radix
// sort of (key, index) over rbits+cbits bits (skipped when the input is
// already canonical -- formats.py:97-98's early return), run heads, scan,
// one thread per unique coordinate for the sum, rpt by binary search.
#include <cub/cub.cuh>

#include "sellb_internal.cuh"

using namespace sellb;

namespace {

constexpr int kT = 256;

__global__ void k_coo_check(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                            int64_t nnz, int64_t n_rows, int64_t n_cols,
                            unsigned long long* first_bad /* [2]: row, col */,
                            unsigned int* unsorted, int cbits, uint64_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rows[i], c = cols[i];
        const bool br = r < 0 || r >= n_rows, bc = c < 0 || c >= n_cols;
        if (br) atomicMin(&first_bad[0], (unsigned long long)i);
        if (bc) atomicMin(&first_bad[1], (unsigned long long)i);
        if (br || bc) continue;
        keys[i] = ((uint64_t)r << cbits) | (uint64_t)c;
        if (i) {
            const int64_t rp = rows[i - 1], cp = cols[i - 1];
            // canonical = strictly increasing (row, col) (formats.py:78-86)
            if (!(r > rp || (r == rp && c > cp))) *unsorted = 1u;
        }
    }
}

template <typename IdxT>
__global__ void k_iota(IdxT* idx, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        idx[i] = (IdxT)i;
}

__global__ void k_heads(const uint64_t* __restrict__ keys, int64_t n, int64_t* __restrict__ head) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// scan = inclusive sum of heads: a head at i starts unique entry scan[i]-1
__global__ void k_starts(const uint64_t* __restrict__ keys, const int64_t* __restrict__ scan,
                         int64_t n, int64_t* __restrict__ starts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i == 0 || keys[i] != keys[i - 1]) starts[scan[i] - 1] = i;
        if (i == n - 1) starts[scan[i]] = n;
    }
}

// NumPy's pairwise_sum over vals[idx[off .. off+n)] (see the file header)
template <typename IdxT>
__device__ double pw_sum(const double* __restrict__ vals, const IdxT* __restrict__ idx,
                         int64_t off, int64_t n) {
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, vals[idx[off + i]]);
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = vals[idx[off + j]];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], vals[idx[off + i + j]]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, vals[idx[off + i]]);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const double a = pw_sum(vals, idx, off, n2);
    const double b = pw_sum(vals, idx, off + n2, n - n2);
    return __dadd_rn(a, b);
}

// one thread per unique coordinate: column, summed value (reduceat seed +
// pairwise rest, formats.py:102-105), unique key for the rpt search
template <typename IdxT>
__global__ void k_reduce(const uint64_t* __restrict__ keys, const IdxT* __restrict__ idx,
                         const double* __restrict__ vals, const int64_t* __restrict__ starts,
                         int64_t n_unique, int cbits, int32_t* __restrict__ col_out,
                         double* __restrict__ val_out, uint64_t* __restrict__ ukeys) {
    const uint64_t cmask = (cbits ? (~0ull >> (64 - cbits)) : 0ull);
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n_unique;
         u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = starts[u], e = starts[u + 1];
        const uint64_t k = keys[s];
        double v = vals[idx[s]];
        if (e - s > 1) v = __dadd_rn(v, pw_sum(vals, idx, s + 1, e - s - 1));
        col_out[u] = (int32_t)(k & cmask);
        val_out[u] = v;
        ukeys[u] = k;
    }
}

// rpt[r] = #unique entries with row < r (np.cumsum(np.bincount(rows)),
// formats.py:171-173), by lower_bound on the sorted unique keys
__global__ void k_rpt(const uint64_t* __restrict__ ukeys, int64_t n_unique, int64_t n_rows,
                      int cbits, int64_t* __restrict__ rpt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t kr = (uint64_t)r << cbits;
        int64_t lo = 0, hi = n_unique;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ukeys[mid] < kr) lo = mid + 1; else hi = mid;
        }
        rpt[r] = lo;
    }
}

int bits_for(int64_t n) {  // bits to hold values 0 .. n-1
    int b = 0;
    while (b < 63 && (1ll << b) < n) ++b;
    return b;
}

unsigned grid_of(int64_t n) {
    static int sms = 0;
    if (!sms) {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        if (sms <= 0) sms = 148;
    }
    const int64_t g = grid_for(n, kT);
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 16));
}

template <typename IdxT>
int canonicalize(const double* vals, int64_t nnz,
                 int64_t n_rows, int cbits, int rbits, bool sorted, int64_t* rpt_d,
                 int32_t* col_d, double* val_d, int64_t* nnz_out, DBuf& d_keys,
                 cudaStream_t st) {
    DBuf d_idx, d_keys2, d_idx2, d_tmp, d_head, d_starts, d_ukeys;
    SELLB_CU(d_idx.alloc(nnz * sizeof(IdxT), st));
    k_iota<IdxT><<<grid_of(nnz), kT, 0, st>>>(d_idx.as<IdxT>(), nnz);
    const uint64_t* keys = d_keys.as<uint64_t>();
    const IdxT* idx = d_idx.as<IdxT>();
    if (!sorted) {
        // stable LSD radix sort == np.lexsort((cols, rows)) (formats.py:98)
        SELLB_CU(d_keys2.alloc(nnz * 8, st));
        SELLB_CU(d_idx2.alloc(nnz * sizeof(IdxT), st));
        cub::DoubleBuffer<uint64_t> kb(d_keys.as<uint64_t>(), d_keys2.as<uint64_t>());
        cub::DoubleBuffer<IdxT> vb(d_idx.as<IdxT>(), d_idx2.as<IdxT>());
        size_t tmp_bytes = 0;
        const int end_bit = std::max(1, rbits + cbits);
        SELLB_CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, nnz, 0, end_bit, st));
        SELLB_CU(d_tmp.alloc(tmp_bytes, st));
        SELLB_CU(cub::DeviceRadixSort::SortPairs(d_tmp.p, tmp_bytes, kb, vb, nnz, 0, end_bit, st));
        keys = kb.Current();
        idx = vb.Current();
    }
    SELLB_CU(d_head.alloc(nnz * 8, st));
    k_heads<<<grid_of(nnz), kT, 0, st>>>(keys, nnz, d_head.as<int64_t>());
    {
        size_t tmp_bytes = 0;
        DBuf d_tmp2;
        SELLB_CU(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, d_head.as<int64_t>(),
                                               d_head.as<int64_t>(), nnz, st));
        SELLB_CU(d_tmp2.alloc(tmp_bytes, st));
        SELLB_CU(cub::DeviceScan::InclusiveSum(d_tmp2.p, tmp_bytes, d_head.as<int64_t>(),
                                               d_head.as<int64_t>(), nnz, st));
    }
    int64_t n_unique = 0;
    SELLB_CU(cudaMemcpyAsync(&n_unique, d_head.as<int64_t>() + nnz - 1, 8,
                             cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    SELLB_CU(d_starts.alloc((n_unique + 1) * 8, st));
    k_starts<<<grid_of(nnz), kT, 0, st>>>(keys, d_head.as<int64_t>(), nnz,
                                          d_starts.as<int64_t>());
    SELLB_CU(d_ukeys.alloc(n_unique * 8, st));
    k_reduce<IdxT><<<grid_of(n_unique), kT, 0, st>>>(keys, idx, vals, d_starts.as<int64_t>(),
                                                     n_unique, cbits, col_d, val_d,
                                                     d_ukeys.as<uint64_t>());
    k_rpt<<<grid_of(n_rows + 1), kT, 0, st>>>(d_ukeys.as<uint64_t>(), n_unique, n_rows, cbits,
                                              rpt_d);
    SELLB_CU(cudaGetLastError());
    SELLB_CU(cudaStreamSynchronize(st));
    *nnz_out = n_unique;
    return 0;
}

}  // namespace

extern "C" {

int sellb_coo_to_crs(const int64_t* rows, const int64_t* cols, const double* vals, int64_t nnz,
                     int64_t n_rows, int64_t n_cols, int64_t* rpt, int32_t* col, double* val,
                     int64_t* nnz_out, int32_t device, void* stream, int32_t ptrs_on_device) {
    clear_error();
    if (!nnz_out || !rpt) return set_error(SELLB_EPARAM, "rpt / nnz_out must not be NULL");
    if (nnz < 0) return set_error(SELLB_EPARAM, "nnz must be >= 0");
    if (nnz && (!rows || !cols || !vals || !col || !val))
        return set_error(SELLB_EPARAM, "entry / output arrays must not be NULL");
    // formats.py:26-32
    if (n_rows < 0 || n_cols < 0)
        return set_error(SELLB_ESTRUCT, "negative matrix dimension (%lldx%lld)",
                         (long long)n_rows, (long long)n_cols);
    if (n_rows >= (1LL << 31) || n_cols >= (1LL << 31))
        return set_error(SELLB_ESTRUCT, "matrix dimension %lld exceeds 4-byte index range",
                         (long long)std::max(n_rows, n_cols));
    *nnz_out = 0;
    DeviceGuard guard(device);
    if (!guard.ok) return set_error(SELLB_ERESOURCE, "cannot select CUDA device %d", device);
    cudaStream_t st = (cudaStream_t)stream;

    DBuf d_rows, d_cols, d_vals, d_rpt, d_col, d_val;
    const int64_t* rows_d = rows;
    const int64_t* cols_d = cols;
    const double* vals_d = vals;
    int64_t* rpt_d = rpt;
    int32_t* col_d = col;
    double* val_d = val;
    if (!ptrs_on_device) {
        SELLB_CU(d_rows.alloc(nnz * 8, st));
        SELLB_CU(d_cols.alloc(nnz * 8, st));
        SELLB_CU(d_vals.alloc(nnz * 8, st));
        SELLB_CU(d_rpt.alloc((n_rows + 1) * 8, st));
        SELLB_CU(d_col.alloc(nnz * 4, st));
        SELLB_CU(d_val.alloc(nnz * 8, st));
        if (nnz) {
            SELLB_CU(cudaMemcpyAsync(d_rows.p, rows, nnz * 8, cudaMemcpyHostToDevice, st));
            SELLB_CU(cudaMemcpyAsync(d_cols.p, cols, nnz * 8, cudaMemcpyHostToDevice, st));
            SELLB_CU(cudaMemcpyAsync(d_vals.p, vals, nnz * 8, cudaMemcpyHostToDevice, st));
        }
        rows_d = d_rows.as<int64_t>();
        cols_d = d_cols.as<int64_t>();
        vals_d = d_vals.as<double>();
        rpt_d = d_rpt.as<int64_t>();
        col_d = d_col.as<int32_t>();
        val_d = d_val.as<double>();
    }
    if (nnz == 0) {
        SELLB_CU(cudaMemsetAsync(rpt_d, 0, (n_rows + 1) * 8, st));
    } else {
        const int cbits = bits_for(n_cols), rbits = bits_for(n_rows);
        DBuf d_keys, d_flags;
        SELLB_CU(d_keys.alloc(nnz * 8, st));
        SELLB_CU(d_flags.alloc(24, st));
        // first_bad[2] = UINT64_MAX, unsorted = 0
        SELLB_CU(cudaMemsetAsync(d_flags.p, 0xff, 16, st));
        SELLB_CU(cudaMemsetAsync(d_flags.as<uint8_t>() + 16, 0, 8, st));
        k_coo_check<<<grid_of(nnz), kT, 0, st>>>(
            rows_d, cols_d, nnz, n_rows, n_cols, d_flags.as<unsigned long long>(),
            reinterpret_cast<unsigned int*>(d_flags.as<uint8_t>() + 16), cbits,
            d_keys.as<uint64_t>());
        SELLB_CU(cudaGetLastError());
        unsigned long long hf[3] = {};
        SELLB_CU(cudaMemcpyAsync(hf, d_flags.p, 24, cudaMemcpyDeviceToHost, st));
        SELLB_CU(cudaStreamSynchronize(st));
        // the reference checks rows before columns and names the first bad
        // entry in storage order (formats.py:58-70)
        if (hf[0] != ~0ull || hf[1] != ~0ull) {
            const bool row_bad = hf[0] != ~0ull;
            const unsigned long long at = row_bad ? hf[0] : hf[1];
            int64_t bad = 0;
            const int64_t* src = row_bad ? rows : cols;
            if (ptrs_on_device)
                SELLB_CU(cudaMemcpy(&bad, src + at, 8, cudaMemcpyDeviceToHost));
            else
                bad = src[at];
            if (row_bad)
                return set_error(SELLB_ESTRUCT, "row index %lld out of bounds for %lld rows",
                                 (long long)bad, (long long)n_rows);
            return set_error(SELLB_ESTRUCT, "column index %lld out of bounds for %lld columns",
                             (long long)bad, (long long)n_cols);
        }
        const bool sorted = (uint32_t)hf[2] == 0u;
        const int rc = nnz < (1ll << 32)
            ? canonicalize<uint32_t>(vals_d, nnz, n_rows, cbits, rbits, sorted,
                                     rpt_d, col_d, val_d, nnz_out, d_keys, st)
            : canonicalize<uint64_t>(vals_d, nnz, n_rows, cbits, rbits, sorted,
                                     rpt_d, col_d, val_d, nnz_out, d_keys, st);
        if (rc) return rc;
    }
    if (!ptrs_on_device) {
        SELLB_CU(cudaMemcpyAsync(rpt, rpt_d, (n_rows + 1) * 8, cudaMemcpyDeviceToHost, st));
        if (*nnz_out) {
            SELLB_CU(cudaMemcpyAsync(col, col_d, *nnz_out * 4, cudaMemcpyDeviceToHost, st));
            SELLB_CU(cudaMemcpyAsync(val, val_d, *nnz_out * 8, cudaMemcpyDeviceToHost, st));
        }
    }
    SELLB_CU(cudaStreamSynchronize(st));
    return 0;
}

}  // extern "C"
