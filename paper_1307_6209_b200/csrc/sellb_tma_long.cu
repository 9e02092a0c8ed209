// sellb_tma_long.cu -- long rows that sit alone in a chunk of short rows
// (unsorted layouts: sigma = 1, small sigma), one warp per row, with the
// row's val / col brought in by the Tensor Memory Accelerator.
//
// Such a row's slot j lives at cs + j*C + r: 256 bytes (fp64, C = 32) apart,
// so every warp-wide load of the warp-per-row role touches 32 different lines
// (cfg4 sigma=1: 1024 rows of 2048 slots took ~120 us of a 120 us SpMV while
// the rest of the matrix needs 40 us).  Opt-in (SELLB_LONG_TMA=1): measured
// slower than the fused role -- every 16-byte box row still costs a 128-byte
// DRAM line (554 MB read for 25 MB of data, ncu), so these rows are bound by
// DRAM transactions however they are fetched.  Here val and col are 2-D
// tensors [slots / C][C]; one TMA box of
// {16 bytes of rows} x {SB slots} per array and batch lands the row (and its
// neighbours in the same 16 bytes) in shared memory, completing on an
// mbarrier -- no LSU wavefronts, D batches in flight per warp.  The x values
// are then gathered per lane with cp.async one batch ahead, the rounded
// products formed in place, and every lane adds them in slot order (the
// reference's per-row sequence of roundings, _kernels.pyx:65-92): results are
// bit-identical.
#include <cudaTypedefs.h>

#include <algorithm>

#include "sellb_internal.cuh"

using namespace sellb;

namespace {

constexpr int kWarps = 4;          // rows (warps) per CTA
constexpr int kSB = 64;            // slots per batch
constexpr int kD = 3;              // TMA batches in flight
constexpr int kE = 2;              // x-gather batches in flight
constexpr int kNS = kD + 1;        // ring stages

template <typename T> struct Ar;
template <> struct Ar<double> {
    __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct Ar<float> {
    __device__ static __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

__device__ __forceinline__ uint32_t s_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_addr(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_addr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra W_%=;\n\t}" ::"r"(s_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                       uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(s_addr(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(s_addr(bar))
        : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int B>
__device__ __forceinline__ void cp_async(void* sdst, const void* gsrc, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;" ::"r"(s_addr(sdst)),
                 "l"(gsrc), "n"(B), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint64_t pol_kind(int kind) {
    uint64_t p;
    if (kind == 0) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else if (kind == 1) asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    else asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// per-warp shared memory
template <typename T>
struct WarpRing {
    static constexpr int VI = 16 / sizeof(T);   // rows per 16-byte val box row
    uint64_t full[kNS];
    alignas(128) T val[kNS][kSB][VI];           // TMA box {VI rows, SB slots}
    alignas(128) int32_t col[kNS][kSB][4];      // TMA box {4 rows, SB slots}
    alignas(16) T xs[kNS][kSB];                 // x gathers, then the products
};

template <typename T, bool ACC, int ORD>
__global__ void __launch_bounds__(kWarps * 32)
k_spmv_long_tma(const __grid_constant__ CUtensorMap tmv, const __grid_constant__ CUtensorMap tmc,
                const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                const int32_t* __restrict__ rl, const T* __restrict__ x, T* __restrict__ y,
                const int32_t* __restrict__ order, int64_t C, int64_t p0, int64_t p1,
                int64_t n_rows, const int32_t* __restrict__ rows, int64_t n_list, int l2pol) {
    extern __shared__ __align__(128) uint8_t smem[];
    using R = WarpRing<T>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    R& ring = reinterpret_cast<R*>(smem)[warp];
    const int64_t k = (int64_t)blockIdx.x * kWarps + warp;
    if (k >= n_list) return;
    const int64_t p = rows[k];
    if (p < p0 || p >= p1) return;
    const int64_t chunk = p / C;
    const int r = (int)(p - chunk * C);
    const int rv = r % R::VI, rc = r & 3;
    const int outer0 = (int)(cs[chunk] / C);
    const int w = cl[chunk];
    const int len = rl[p];
    const int nb = (len + kSB - 1) / kSB;
    const uint64_t pol_x = pol_kind((l2pol >> 4) & 0xf);
    if (lane == 0) {
        for (int s = 0; s < kNS; ++s) mbar_init(&ring.full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    constexpr uint32_t kBytes = kSB * 16 + kSB * 16;           // val box + col box
    auto issue = [&](int b) {
        if (lane == 0 && b < nb) {
            const int st = b % kNS;
            mbar_expect_tx(&ring.full[st], kBytes);
            tma_2d(&ring.val[st][0][0], &tmv, r - rv, outer0 + b * kSB, &ring.full[st]);
            tma_2d(&ring.col[st][0][0], &tmc, r - rc, outer0 + b * kSB, &ring.full[st]);
        }
    };
    auto gather = [&](int b) {
        if (b < nb) {
            const int st = b % kNS;
            mbar_wait(&ring.full[st], (uint32_t)((b / kNS) & 1));
#pragma unroll
            for (int s = 0; s < kSB / 32; ++s) {
                const int jj = s * 32 + lane;
                if (b * kSB + jj < len)
                    cp_async<sizeof(T)>(&ring.xs[st][jj], x + ring.col[st][jj][rc], pol_x);
            }
        }
        cp_commit();
    };
#pragma unroll
    for (int b = 0; b < kD; ++b) issue(b);
#pragma unroll
    for (int e = 0; e < kE; ++e) gather(e);
    T sum = T(0);
    for (int b = 0; b < nb; ++b) {
        issue(b + kD);                          // stage of batch b-1: consumed
        gather(b + kE);
        cp_wait<kE>();                          // X(b) landed (this lane's)
        const int st = b % kNS;
#pragma unroll
        for (int s = 0; s < kSB / 32; ++s) {
            const int jj = s * 32 + lane;
            ring.xs[st][jj] = (b * kSB + jj < len) ? Ar<T>::mul(ring.val[st][jj][rv], ring.xs[st][jj])
                                                   : T(0);
        }
        __syncwarp();
        // +0.0 products past the row's end are exact no-ops (the sum starts
        // at +0.0 and is never -0.0)
        const T* q = ring.xs[st];
#pragma unroll 16
        for (int jj = 0; jj < kSB; ++jj) sum = Ar<T>::add(sum, q[jj]);
        __syncwarp();
    }
    cp_wait<0>();
    if (lane == 0) {
        if (len < w) sum = Ar<T>::add(sum, Ar<T>::mul(T(0), __ldg(x)));
        if (ORD == 0) {
            y[p] = ACC ? Ar<T>::add(y[p], sum) : sum;
        } else if (p < n_rows) {
            const int64_t o = order[p];
            y[o] = ACC ? Ar<T>::add(y[o], sum) : sum;
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)f;
    }();
    return fn;
}

// encode val / col as 2-D [slots / C][C] tensors (once per matrix)
bool tensor_maps(sellb_mat* m) {
    std::lock_guard<std::mutex> lk(m->tm_mu);
    if (m->tm_state) return m->tm_state > 0;
    m->tm_state = -1;
    if (m->C % 4 || m->slots == 0 || m->slots / m->C >= (1LL << 31)) return false;
    auto enc = encode_fn();
    if (!enc) return false;
    const size_t vs = vsize(m->dtype);
    const cuuint64_t gdim[2] = {(cuuint64_t)m->C, (cuuint64_t)(m->slots / m->C)};
    const cuuint32_t est[2] = {1, 1};
    const cuuint64_t gstr_v[1] = {(cuuint64_t)(m->C * vs)};
    const cuuint32_t box_v[2] = {(cuuint32_t)(16 / vs), (cuuint32_t)kSB};
    const cuuint64_t gstr_c[1] = {(cuuint64_t)(m->C * 4)};
    const cuuint32_t box_c[2] = {4, (cuuint32_t)kSB};
    if (enc(&m->tm_val,
            m->dtype == SELLB_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
            2, m->val, gdim, gstr_v, box_v, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(&m->tm_col, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, m->col, gdim, gstr_c, box_c, est,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    m->tm_state = 1;
    return true;
}

template <typename T>
size_t ring_bytes() { return sizeof(WarpRing<T>) * kWarps; }

}  // namespace

namespace sellb {

bool long_tma_possible(const sellb_mat* m) {
    return m->C % 4 == 0 && m->slots > 0 && encode_fn() != nullptr;
}

int launch_long_tma(const sellb_mat* m, const void* x, void* y, int64_t p0, int64_t p1,
                    int accumulate, int out_order, const int32_t* rows, int64_t n_list,
                    int l2pol, cudaStream_t st) {
    if (n_list <= 0) return 1;
    sellb_mat* mm = const_cast<sellb_mat*>(m);
    if (!tensor_maps(mm)) return 0;
    const unsigned grid = (unsigned)((n_list + kWarps - 1) / kWarps);
#define SELLB_LT(TT, AA, OO)                                                                    \
    do {                                                                                        \
        const size_t smem_ = ring_bytes<TT>();                                                  \
        static unsigned attr_ = 0;                                                              \
        int dev_ = 0;                                                                           \
        cudaGetDevice(&dev_);                                                                   \
        if (!(attr_ & (1u << (dev_ & 31)))) {                                                   \
            cudaFuncSetAttribute(k_spmv_long_tma<TT, AA, OO>,                                   \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_);      \
            attr_ |= 1u << (dev_ & 31);                                                         \
        }                                                                                       \
        k_spmv_long_tma<TT, AA, OO><<<grid, kWarps * 32, smem_, st>>>(                          \
            m->tm_val, m->tm_col, m->cs, m->cl, m->rl, (const TT*)x, (TT*)y, m->order, m->C,    \
            p0, p1, m->n_rows, rows, n_list, l2pol);                                            \
    } while (0)
#define SELLB_LT_O(TT, AA)                                                                      \
    do {                                                                                        \
        if (out_order) SELLB_LT(TT, AA, 1); else SELLB_LT(TT, AA, 0);                           \
    } while (0)
    if (m->dtype == SELLB_F32) {
        if (accumulate) SELLB_LT_O(float, true); else SELLB_LT_O(float, false);
    } else {
        if (accumulate) SELLB_LT_O(double, true); else SELLB_LT_O(double, false);
    }
#undef SELLB_LT_O
#undef SELLB_LT
    count_launches();
    return 1;
}

}  // namespace sellb
