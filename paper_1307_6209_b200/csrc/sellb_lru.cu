// sellb_lru.cu -- misses of a fully-associative LRU cache replaying a line-id
// stream (the reference's cachesim kernel, _kernels.pyx:95-139), on the GPU.
//
// The reference walks a doubly-linked MRU list, one access at a time.  The
// same count, in parallel, from the stack-distance characterisation of LRU:
// an access to line l at position k whose previous access was at p hits iff
// fewer than L (= cache_lines) DISTINCT other lines were accessed in (p, k):
// each first-since-p access of another line pushes l one place down the MRU
// stack, and l is evicted exactly when L of them have.  With prev[j] the
// previous position of line[j] (-1 for a first access),
//
//     D(k) = #{ j in (p, k) : prev[j] < p }          (distinct lines in (p,k))
//     miss(k) = (p < 0) || D(k) >= L.
//
//   1. cub radix sort of (line, position)   -> prev[]            (stable)
//   2. k_classify: compulsory misses (p < 0), trivial hits (k-p-1 < L), the
//      rest into a candidate list.  If the stream holds <= L distinct lines
//      every reuse hits (D <= distinct-1) and the count is final.
//   3. per-tile sorted copy of prev[] (tiles of kTile positions; one radix
//      sort of (tile, prev+1) keys), so a whole tile's contribution to D is a
//      binary search.
//   4. k_resolve: one warp per candidate -- direct scan of the partial tiles
//      at both ends, binary searches over the full tiles between, early exit
//      once D >= L.
#include <cub/cub.cuh>

#include "sellb_internal.cuh"

using namespace sellb;

namespace {

constexpr int kTile = 1024;

__global__ void k_lru_check(const int64_t* __restrict__ lines, int64_t n, int64_t n_slots,
                            int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && (lines[i] < 0 || lines[i] >= n_slots)) atomicOr(bad, 1);
}

__global__ void k_lru_iota(int64_t* __restrict__ v, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

// sorted (line, position) pairs -> prev[position]
__global__ void k_lru_prev(const uint64_t* __restrict__ key, const int64_t* __restrict__ pos,
                           int64_t n, int64_t* __restrict__ prev) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    prev[pos[i]] = (i > 0 && key[i - 1] == key[i]) ? pos[i - 1] : -1;
}

// counts[0] += compulsory misses, counts[1] = number of candidates
__global__ void k_lru_classify(const int64_t* __restrict__ prev, int64_t n, int64_t L,
                               unsigned long long* __restrict__ counts,
                               int64_t* __restrict__ cand) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    bool first = false, amb = false;
    if (k < n) {
        const int64_t p = prev[k];
        first = p < 0;
        amb = !first && k - p - 1 >= L;
    }
    const unsigned mf = __ballot_sync(0xffffffffu, first);
    const unsigned ma = __ballot_sync(0xffffffffu, amb);
    unsigned long long base = 0;
    if (lane == 0) {
        if (mf) atomicAdd(&counts[0], (unsigned long long)__popc(mf));
        if (ma) base = atomicAdd(&counts[1], (unsigned long long)__popc(ma));
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (amb) cand[base + __popc(ma & ((1u << lane) - 1u))] = k;
}

__global__ void k_lru_tile_keys(const int64_t* __restrict__ prev, int64_t n, int vbits,
                                uint64_t* __restrict__ keys) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < n) keys[j] = ((uint64_t)(j / kTile) << vbits) | (uint64_t)(prev[j] + 1);
}

// one warp per candidate position k: miss iff D(k) >= L
__global__ void k_lru_resolve(const int64_t* __restrict__ prev,
                              const uint64_t* __restrict__ tsorted, int vbits, int64_t n,
                              const int64_t* __restrict__ cand, int64_t n_cand, int64_t L,
                              unsigned long long* __restrict__ misses) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t vmask = (vbits >= 64) ? ~0ull : ((1ull << vbits) - 1ull);
    unsigned long long mine = 0;
    for (int64_t w = w0; w < n_cand; w += nw) {
        const int64_t k = cand[w];
        const int64_t p = prev[k];
        const int64_t lo = p + 1, hi = k;           // j in [lo, hi)
        const int64_t t_lo = (lo + kTile - 1) / kTile, t_hi = hi / kTile;
        int64_t d = 0;                              // per-lane partial count
        if (t_lo >= t_hi) {
            for (int64_t j = lo + lane; j < hi; j += 32) d += prev[j] < p;
        } else {
            for (int64_t j = lo + lane; j < t_lo * kTile; j += 32) d += prev[j] < p;
            for (int64_t j = t_hi * kTile + lane; j < hi; j += 32) d += prev[j] < p;
        }
        int64_t tot = d;
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        // whole tiles: count of (prev+1) <= p, i.e. lower_bound(p + 1)
        for (int64_t t0 = t_lo; t0 < t_hi && tot < L; t0 += 32) {
            int64_t c = 0;
            const int64_t t = t0 + lane;
            if (t < t_hi) {
                const uint64_t* a = tsorted + t * kTile;
                int lo_i = 0, hi_i = kTile;
                while (lo_i < hi_i) {
                    const int mid = (lo_i + hi_i) >> 1;
                    if ((int64_t)(a[mid] & vmask) < p + 1) lo_i = mid + 1; else hi_i = mid;
                }
                c = lo_i;
            }
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            tot += c;
        }
        if (lane == 0 && tot >= L) ++mine;
    }
    if (lane == 0 && mine) atomicAdd(misses, mine);
}

// real entries per chunk (sum of its row lengths): warp per chunk
__global__ void k_chunk_real(const int32_t* __restrict__ rl, int64_t C, int64_t n_chunks,
                             int64_t* __restrict__ cnt) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_chunks) return;
    int64_t s = 0;
    for (int64_t r = lane; r < C; r += 32) s += rl[w * C + r];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cnt[w] = s;
}

// x line ids of the real entries in kernel traversal order (cachesim.py:31-46:
// per chunk slot-major, then lane; padding slots dropped): warp per chunk,
// ballot-compacted per slot column
__global__ void k_x_lines(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                          const int32_t* __restrict__ col, const int32_t* __restrict__ rl,
                          int64_t C, int64_t n_chunks, const int64_t* __restrict__ base,
                          int shift, int64_t* __restrict__ out) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_chunks) return;
    int64_t o = base[w];
    const int64_t c0 = cs[w];
    const int w_cl = cl[w];
    for (int j = 0; j < w_cl; ++j) {
        for (int64_t r0 = 0; r0 < C; r0 += 32) {
            const int64_t r = r0 + lane;
            const bool act = r < C && rl[w * C + r] > j;
            const unsigned m = __ballot_sync(0xffffffffu, act);
            if (act)
                out[o + __popc(m & ((1u << lane) - 1u))] =
                    (int64_t)((uint32_t)col[c0 + j * C + r] >> shift);
            o += __popc(m);
        }
    }
}

int bits_for(uint64_t v) {           // bits needed to hold values 0..v
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

}  // namespace

extern "C" int sellb_lru_stream_misses(const int64_t* lines, int64_t n, int64_t cache_lines,
                                       int64_t n_line_slots, int32_t lines_on_device,
                                       int64_t* misses_out, void* stream) {
    clear_error();
    if (!misses_out) return set_error(SELLB_EPARAM, "NULL misses");
    if (n < 0 || n_line_slots < 0) return set_error(SELLB_EPARAM, "negative length");
    if (n == 0) { *misses_out = 0; return 0; }                   // _kernels.pyx:105-106
    if (!lines) return set_error(SELLB_EPARAM, "NULL lines");
    if (cache_lines <= 0) { *misses_out = n; return 0; }         // _kernels.pyx:107-108
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned T = 256;
    const unsigned G = (unsigned)grid_for(n, T);

    DBuf d_lines;
    const int64_t* dl = lines;
    if (!lines_on_device) {
        SELLB_CU(d_lines.alloc(n * 8, st));
        SELLB_CU(cudaMemcpyAsync(d_lines.p, lines, n * 8, cudaMemcpyHostToDevice, st));
        dl = d_lines.as<int64_t>();
    }
    DBuf d_small;
    SELLB_CU(d_small.alloc(64, st));
    SELLB_CU(cudaMemsetAsync(d_small.p, 0, 64, st));
    int* d_bad = d_small.as<int>();
    unsigned long long* d_counts = reinterpret_cast<unsigned long long*>(d_small.as<char>() + 8);
    k_lru_check<<<G, T, 0, st>>>(dl, n, n_line_slots, d_bad);
    count_launches();
    int bad = 0;
    SELLB_CU(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    if (bad) return set_error(SELLB_EPARAM, "line id outside [0, n_line_slots)");

    // 1. prev[] from a stable sort of (line, position)
    DBuf d_prev;
    SELLB_CU(d_prev.alloc(n * 8, st));
    {
        DBuf k2, v1, v2, tmp;
        SELLB_CU(k2.alloc(n * 8, st));
        SELLB_CU(v1.alloc(n * 8, st));
        SELLB_CU(v2.alloc(n * 8, st));
        k_lru_iota<<<G, T, 0, st>>>(v1.as<int64_t>(), n);
        count_launches();
        // keys are read through a DoubleBuffer whose first half is the input:
        // copy so the caller's lines stay untouched
        DBuf k1;
        SELLB_CU(k1.alloc(n * 8, st));
        SELLB_CU(cudaMemcpyAsync(k1.p, dl, n * 8, cudaMemcpyDeviceToDevice, st));
        cub::DoubleBuffer<uint64_t> kb(k1.as<uint64_t>(), k2.as<uint64_t>());
        cub::DoubleBuffer<int64_t> vb(v1.as<int64_t>(), v2.as<int64_t>());
        const int end_bit = bits_for((uint64_t)std::max<int64_t>(n_line_slots - 1, 0));
        size_t tb = 0;
        SELLB_CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, n, 0, end_bit, st));
        SELLB_CU(tmp.alloc(tb, st));
        SELLB_CU(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kb, vb, n, 0, end_bit, st));
        k_lru_prev<<<G, T, 0, st>>>(kb.Current(), vb.Current(), n, d_prev.as<int64_t>());
        count_launches();
        SELLB_CU(cudaGetLastError());
    }
    // 2. classify
    DBuf d_cand;
    SELLB_CU(d_cand.alloc(n * 8, st));
    k_lru_classify<<<G, T, 0, st>>>(d_prev.as<int64_t>(), n, cache_lines, d_counts,
                                    d_cand.as<int64_t>());
    count_launches();
    unsigned long long h[2] = {0, 0};
    SELLB_CU(cudaMemcpyAsync(h, d_counts, 16, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    const int64_t compulsory = (int64_t)h[0], n_cand = (int64_t)h[1];
    if (n_cand == 0 || compulsory <= cache_lines) {
        // no far reuse, or the whole stream fits: every reuse hits
        *misses_out = compulsory;
        return 0;
    }
    // 3. per-tile sorted prev+1
    const int vbits = bits_for((uint64_t)n);
    const int tbits = bits_for((uint64_t)(n / kTile));
    if (vbits + tbits > 64) return set_error(SELLB_EPARAM, "stream too long");
    DBuf t1, t2, tmp;
    SELLB_CU(t1.alloc(n * 8, st));
    SELLB_CU(t2.alloc(n * 8, st));
    k_lru_tile_keys<<<G, T, 0, st>>>(d_prev.as<int64_t>(), n, vbits, t1.as<uint64_t>());
    count_launches();
    cub::DoubleBuffer<uint64_t> tkb(t1.as<uint64_t>(), t2.as<uint64_t>());
    size_t tb = 0;
    SELLB_CU(cub::DeviceRadixSort::SortKeys(nullptr, tb, tkb, n, 0, vbits + tbits, st));
    SELLB_CU(tmp.alloc(tb, st));
    SELLB_CU(cub::DeviceRadixSort::SortKeys(tmp.p, tb, tkb, n, 0, vbits + tbits, st));
    // 4. resolve the far reuses
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = grid_for(n_cand * 32, T);
    const unsigned GR = (unsigned)std::min<int64_t>(want, (int64_t)sms * 16);
    unsigned long long* d_far = d_counts + 1;     // reuse the candidate counter slot
    SELLB_CU(cudaMemsetAsync(d_far, 0, 8, st));
    k_lru_resolve<<<GR, T, 0, st>>>(d_prev.as<int64_t>(), tkb.Current(), vbits, n,
                                    d_cand.as<int64_t>(), n_cand, cache_lines, d_far);
    count_launches();
    SELLB_CU(cudaGetLastError());
    unsigned long long far = 0;
    SELLB_CU(cudaMemcpyAsync(&far, d_far, 8, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    *misses_out = compulsory + (int64_t)far;
    return 0;
}

extern "C" int sellb_sell_x_lines(const sellb_mat* m, int32_t elems_per_line, int64_t* lines,
                                  int64_t* n_out, void* stream) {
    clear_error();
    if (!m || !lines || !n_out) return set_error(SELLB_EPARAM, "NULL argument");
    if (elems_per_line < 1 || (elems_per_line & (elems_per_line - 1)))
        return set_error(SELLB_EPARAM, "elems_per_line must be a power of two");
    if (!m->rl) return set_error(SELLB_EPARAM, "matrix has no row_lengths");
    DeviceGuard guard(m->device);
    cudaStream_t st = (cudaStream_t)stream;
    *n_out = m->nnz;
    if (m->n_chunks == 0 || m->nnz == 0) return 0;
    int shift = 0;
    while ((1 << shift) < elems_per_line) ++shift;
    const unsigned T = 256;
    const unsigned G = (unsigned)grid_for(m->n_chunks * 32, T);
    DBuf cnt, base, tmp;
    SELLB_CU(cnt.alloc(m->n_chunks * 8, st));
    SELLB_CU(base.alloc(m->n_chunks * 8, st));
    k_chunk_real<<<G, T, 0, st>>>(m->rl, m->C, m->n_chunks, cnt.as<int64_t>());
    count_launches();
    size_t tb = 0;
    SELLB_CU(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<int64_t>(), base.as<int64_t>(),
                                           m->n_chunks, st));
    SELLB_CU(tmp.alloc(tb, st));
    SELLB_CU(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.as<int64_t>(), base.as<int64_t>(),
                                           m->n_chunks, st));
    k_x_lines<<<G, T, 0, st>>>(m->cs, m->cl, m->col, m->rl, m->C, m->n_chunks,
                               base.as<int64_t>(), shift, lines);
    count_launches();
    SELLB_CU(cudaGetLastError());
    SELLB_CU(cudaStreamSynchronize(st));
    return 0;
}
