// sellb_tma.cu -- SELL-32 SpMV with the matrix streamed by the Tensor Memory
// Accelerator's bulk-copy engine (cp.async.bulk + mbarrier), for C = 32,
// pad-inclusive layouts (every slot of a chunk is read).
//
// Chunks are stored back to back, so a tile of kTile consecutive chunks is
// ONE contiguous span of val and ONE of col ([cs[c0], cs[c0+kTile])).  A
// producer warp issues two bulk copies per tile into a kStages-deep shared
// memory ring (completion counted in bytes on the stage's "full" mbarrier);
// kTile consumer warps -- one per chunk, one lane per row -- read their
// chunk's val/col from shared memory, gather x from global (L2), and add the
// rounded products in slot order (same per-row sequence of roundings as
// _kernels.pyx:65-92, so bit-identical), then arrive on the stage's "empty"
// mbarrier.  The copy engine keeps the HBM stream in flight independently of
// the consumer warps' gather latency, with two instructions per tile
// instead of two per slot per warp.
#include "sellb_internal.cuh"

using namespace sellb;

namespace {

constexpr int kTile = 4;                 // chunks (consumer warps) per tile
constexpr int kStages = 2;
constexpr int kTmaThreads = (kTile + 1) * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <typename T> struct ArithT;
template <> struct ArithT<double> {
    __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct ArithT<float> {
    __device__ static __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double gx(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float gx(const float* p, uint64_t pol) {
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// stage_slots: capacity of one stage in slots (val T + col int32 per slot)
template <typename T, bool ACC, int U>
__global__ void __launch_bounds__(kTmaThreads)
k_spmv_tma(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
           const int32_t* __restrict__ col, const T* __restrict__ val, const T* __restrict__ x,
           T* __restrict__ y, int64_t c0, int64_t c1, int64_t stage_slots) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + kStages;
    T* sval = reinterpret_cast<T*>(smem + 128);
    int32_t* scol = reinterpret_cast<int32_t*>(smem + 128 + kStages * stage_slots * sizeof(T));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_tiles = (c1 - c0 + kTile - 1) / kTile;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTile);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (warp == kTile) {                               // producer warp
        if (lane == 0) {
            int64_t k = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
                const int s = (int)(k % kStages);
                if (k >= kStages) mbar_wait(&empty[s], (uint32_t)(((k / kStages) - 1) & 1));
                const int64_t ca = c0 + t * kTile;
                const int64_t cb = ca + kTile < c1 ? ca + kTile : c1;
                const int64_t s0 = cs[ca], n = cs[cb] - s0;
                const uint32_t bv = (uint32_t)(n * sizeof(T)), bc = (uint32_t)(n * 4);
                mbar_expect_tx(&full[s], bv + bc);
                if (n) {
                    bulk_g2s(sval + s * stage_slots, val + s0, bv, &full[s]);
                    bulk_g2s(scol + s * stage_slots, col + s0, bc, &full[s]);
                }
            }
        }
        return;
    }
    const uint64_t pol_x = pol_evict_last();
    int64_t k = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int s = (int)(k % kStages);
        const int64_t ca = c0 + t * kTile;
        const int64_t c = ca + warp;
        mbar_wait(&full[s], (uint32_t)((k / kStages) & 1));
        if (c < c1) {
            const int64_t off = cs[c] - cs[ca];
            const int w = cl[c];
            const T* sv = sval + s * stage_slots + off + lane;
            const int32_t* sc = scol + s * stage_slots + off + lane;
            T sum = T(0);
            int j = 0;
            for (; j + U <= w; j += U) {
                T xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) xv[u] = gx(x + sc[(j + u) * 32], pol_x);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    sum = ArithT<T>::add(sum, ArithT<T>::mul(sv[(j + u) * 32], xv[u]));
            }
            for (; j < w; ++j)
                sum = ArithT<T>::add(sum, ArithT<T>::mul(sv[j * 32], gx(x + sc[j * 32], pol_x)));
            T* yp = y + c * 32 + lane;
            *yp = ACC ? ArithT<T>::add(*yp, sum) : sum;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

}  // namespace

namespace sellb {

// Returns 1 if launched, 0 if the layout does not qualify (caller falls back).
int launch_spmv_tma(const sellb_mat* m, const void* x, void* y, int64_t c0, int64_t c1,
                    int accumulate, cudaStream_t st, const int64_t* h_cs) {
    if (m->C != 32 || !h_cs || c1 <= c0) return 0;
    // largest tile (kTile consecutive chunks) in slots
    int64_t max_tile = 0;
    for (int64_t a = c0; a < c1; a += kTile) {
        const int64_t b = a + kTile < c1 ? a + kTile : c1;
        max_tile = std::max<int64_t>(max_tile, h_cs[b] - h_cs[a]);
    }
    const size_t vs = vsize(m->dtype);
    const size_t smem = 128 + (size_t)kStages * max_tile * (vs + 4);
    if (smem > 200 * 1024) return 0;
    static int sms = 0;
    if (!sms) {
        int d = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    }
    const int per_sm = std::max(1, (int)std::min<size_t>(8, (220 * 1024) / smem));
    const int64_t tiles = (c1 - c0 + kTile - 1) / kTile;
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)sms * per_sm);
    static const int u_env = [] {
        const char* e = getenv("SELLB_TMA_U");
        return e ? atoi(e) : 16;
    }();
#define SELLB_TMA_U(TT, AA, UU)                                                               \
    do {                                                                                      \
        auto kern = k_spmv_tma<TT, AA, UU>;                                                   \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
        kern<<<grid, kTmaThreads, smem, st>>>(m->cs, m->cl, m->col, (const TT*)m->val,       \
                                              (const TT*)x, (TT*)y, c0, c1, max_tile);       \
    } while (0)
#define SELLB_TMA(TT, AA)                                                                     \
    do {                                                                                      \
        if (u_env == 32) SELLB_TMA_U(TT, AA, 32);                                             \
        else if (u_env == 8) SELLB_TMA_U(TT, AA, 8);                                          \
        else SELLB_TMA_U(TT, AA, 16);                                                         \
    } while (0)
    if (m->dtype == SELLB_F32) {
        if (accumulate) SELLB_TMA(float, true); else SELLB_TMA(float, false);
    } else {
        if (accumulate) SELLB_TMA(double, true); else SELLB_TMA(double, false);
    }
#undef SELLB_TMA
#undef SELLB_TMA_U
    count_launches();
    return 1;
}

}  // namespace sellb
