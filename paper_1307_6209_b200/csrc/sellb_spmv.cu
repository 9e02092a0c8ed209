// sellb_spmv.cu -- SELL-C-sigma SpMV kernels for sm_100a.
//
// The reference kernel (/root/reference/pkg/src/sellkit/_kernels.pyx:65-92):
//   for each chunk i: tmp[r] = 0 for r < C
//     for j < cl[i]: for r < C: tmp[r] = tmp[r] + val[cs[i]+j*C+r] * x[col[...]]
//     y[i*C+r] = tmp[r]            (or y = y + tmp when accumulating)
//
// B200 mapping: one thread per stored row (the paper's GPU design,
// PAPER.md:770-779, :995-998).  For C = 32 a warp owns a chunk, so each slot j
// is one fully coalesced 256 B (fp64) value load and one 128 B index load.
// The RHS x is gathered through the read-only path (ld.global.nc), matrix
// streams are marked L1::no_allocate with an L2 evict-first policy so they do
// not push x out of the 126 MB L2.
//
// Bitwise parity with the reference: each row is summed from +0.0, in
// ascending slot order, with separately rounded multiply and add (__dmul_rn /
// __dadd_rn: no FMA contraction; the compiled reference has none either) --
// by one thread in the bulk role, or, for very long rows, by a warp that
// first stages the rounded products and then adds them in order.  Loads are
// batched U slots at a time for memory-level parallelism, but the adds are
// issued in slot order.
//
// Padding: the PAD_SKIP variant stops each thread at its own row length (the
// paper's "Sliced ELLR-T, T=1" optimisation).  The reference adds
// 0.0 * x[0] for every padded slot; for finite x[0] that is an exact no-op
// (the running sum starts at +0.0 and can never become -0.0), and for
// non-finite x[0] it turns the row into NaN.  One fused fix-up
// (sum += 0 * x[0] when the row has padding) reproduces that exactly, so both
// variants are bit-identical to the reference for every input.
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "sellb_internal.cuh"

using namespace sellb;

namespace {

template <typename T> struct Arith;
template <> struct Arith<double> {
    __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct Arith<float> {
    __device__ static __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// kind: 0 evict_first, 1 evict_normal, 2 evict_last
__device__ __forceinline__ uint64_t make_policy(int kind) {
    return kind == 0 ? policy_evict_first() : kind == 1 ? policy_evict_normal()
                                                         : policy_evict_last();
}

// streaming (read-once) loads of the matrix arrays
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
    float v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
// RHS gather: read-only path, keep in L2
// SELLB_XLD selects the gather's cache qualifiers at build time (A/B builds,
// tools/build_variant.sh): 0 read-only path (default), 1 read-only without
// L1 allocation, 2 plain coherent load, 3 read-only with L1 evict_last.
#ifndef SELLB_XLD
#define SELLB_XLD 0
#endif
#if SELLB_XLD == 1
#define SELLB_XLD_Q "ld.global.nc.L1::no_allocate.L2::cache_hint"
#elif SELLB_XLD == 2
#define SELLB_XLD_Q "ld.global.L2::cache_hint"
#elif SELLB_XLD == 3
#define SELLB_XLD_Q "ld.global.nc.L1::evict_last.L2::cache_hint"
#else
#define SELLB_XLD_Q "ld.global.nc.L2::cache_hint"
#endif
__device__ __forceinline__ double ld_x(const double* p, uint64_t pol) {
    double v;
    asm(SELLB_XLD_Q ".f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_x(const float* p, uint64_t pol) {
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

constexpr int kThreads = 256;

template <typename T, bool ACC, int ORD>
__device__ __forceinline__ void store_row(T* __restrict__ y, const int32_t* __restrict__ order,
                                          int64_t p, int64_t n_rows, T sum) {
    if (ORD == 0) {
        T out = ACC ? Arith<T>::add(y[p], sum) : sum;
        __stcs(y + p, out);
    } else if (ORD == 1) {
        if (p < n_rows) {
            const int64_t o = order[p];
            y[o] = ACC ? Arith<T>::add(y[o], sum) : sum;
        }
    } else if (p < n_rows) {     // ORD 2: the shadow layout's flagged map
        const int32_t o = order[p] & 0x7fffffff;
        if (o != 0x7fffffff) y[o] = ACC ? Arith<T>::add(y[o], sum) : sum;
    }
}

// The reference's 0 * x[0] padding term applies to row p: `own` (its chunk
// in this layout is wider than the row) or, for the shadow layout (ORD 2),
// bit 31 of its map entry (its chunk in the caller's layout was wider)
template <int ORD>
__device__ __forceinline__ bool pad_term(const int32_t* __restrict__ order, int64_t p,
                                         int64_t n_rows, bool own) {
    if constexpr (ORD == 2) return p < n_rows && order[p] < 0;
    else return own;
}

#ifndef SELLB_VX256
#define SELLB_VX256 0
#endif
__device__ __forceinline__ void ld_x4(const double* p, uint64_t pol, double* w) {
    asm("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
        : "=d"(w[0]), "=d"(w[1]), "=d"(w[2]), "=d"(w[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ double2 ld_x2(const double* p, uint64_t pol) {
    double2 v;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
        : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

// The U x values of a batch.  When the batch's columns are one consecutive
// run (stencil rows, windowed rows: c[u] == c[0] + u), U = 8 (the 4-slot
// instances have no registers to spare for it) and x is 16-byte
// aligned (vx), they come from U/2 aligned 16-byte loads -- plus one more,
// predicated, when the run starts at an odd column -- instead of U scalar
// gathers: the x loads of a warp touch the same lines with fewer
// instructions, i.e. fewer L1 wavefronts (cfg3 sigma=N is L1-data-pipe bound:
// 89 % of peak, ~10 lines per scalar gather).  Values are the same doubles,
// so the sums are unchanged.  Reads stay inside the 16-byte blocks holding
// x[c[0]] .. x[c[U-1]].
template <typename T, int U>
__device__ __forceinline__ void gather_x(T (&xv)[U], const int32_t (&c)[U],
                                         const T* __restrict__ x, uint64_t pol_x, bool vx) {
    if constexpr (sizeof(T) == 8 && U == 8) {
        bool run = vx;
#pragma unroll
        for (int u = 1; u < U; ++u) run = run && (c[u] == c[0] + u);
        if (run) {
#if SELLB_VX256
            // 32-byte loads: 2 (aligned run) or 3 per 8 slots
            const int off = c[0] & 3;
            const double* px = x + (c[0] & ~3);
            double w[U + 4];
#pragma unroll
            for (int k = 0; k < U / 4; ++k) ld_x4(px + 4 * k, pol_x, w + 4 * k);
#pragma unroll
            for (int k = U; k < U + 4; ++k) w[k] = 0.0;
            if (off) ld_x4(px + U, pol_x, w + U);
#pragma unroll
            for (int u = 0; u < U; ++u)
                xv[u] = off == 0 ? w[u] : off == 1 ? w[u + 1] : off == 2 ? w[u + 2] : w[u + 3];
#else
            const bool odd = c[0] & 1;
            const double* px = x + (c[0] & ~1);
            double w[U + 2];
#pragma unroll
            for (int k = 0; k < U / 2; ++k) {
                const double2 t = ld_x2(px + 2 * k, pol_x);
                w[2 * k] = t.x;
                w[2 * k + 1] = t.y;
            }
            w[U] = 0.0;
            w[U + 1] = 0.0;
            if (odd) {
                const double2 t = ld_x2(px + U, pol_x);
                w[U] = t.x;
                w[U + 1] = t.y;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = odd ? w[u + 1] : w[u];
#endif
            return;
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = ld_x(x + c[u], pol_x);
}

// One row's sum over its first len slots (stride C): U-slot batches -- all
// val/col loads of the batch, then the U x gathers, then the adds in slot
// order; a predicated tail batch finishes rows whose length is not a
// multiple of U.
template <typename T, int U>
__device__ __forceinline__ T row_sum(const T* __restrict__ vp, const int32_t* __restrict__ cp,
                                     int64_t C, int len, const T* __restrict__ x,
                                     uint64_t pol_s, uint64_t pol_x, bool vx = false) {
    T sum = T(0);
    int j = 0;
    for (; j + U <= len; j += U) {
        T v[U];
        int32_t c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u] = ld_stream(vp + (int64_t)(j + u) * C, pol_s);
            c[u] = ld_stream(cp + (int64_t)(j + u) * C, pol_s);
        }
        T xv[U];
        gather_x<T, U>(xv, c, x, pol_x, vx);
#pragma unroll
        for (int u = 0; u < U; ++u) sum = Arith<T>::add(sum, Arith<T>::mul(v[u], xv[u]));
    }
    if (j < len) {   // predicated tail batch
        T v[U];
        int32_t c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (j + u < len) {
                v[u] = ld_stream(vp + (int64_t)(j + u) * C, pol_s);
                c[u] = ld_stream(cp + (int64_t)(j + u) * C, pol_s);
            } else {
                v[u] = T(0);
                c[u] = 0;
            }
        }
        T xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = (j + u < len) ? ld_x(x + c[u], pol_x) : T(0);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (j + u < len) sum = Arith<T>::add(sum, Arith<T>::mul(v[u], xv[u]));
    }
    return sum;
}

// Long-row role: one WARP per stored row longer than long_th, lanes over
// slots (lane l loads slot j0+l; stride C).  The rounded products are formed
// in parallel and staged in shared memory, then every lane sums the staged
// products in slot order (broadcast reads, no shuffles in the add chain) --
// the same sequence of roundings as the reference's per-row loop, so the
// result is bitwise identical.  Slots past the row length stage +0.0, and
// adding +0.0 to a sum that started at +0.0 is an exact no-op (the sum can
// never be -0.0), so the chain needs no predicate.  kSeg*32 slots per batch.
constexpr int kSeg = 4;

// vp / cp: the row's first value / index, `stride` elements apart (C in the
// SELL arrays, 1 in the long-row side table); w: the chunk width (padding
// fix-up)
template <typename T, bool ACC, int ORD>
__device__ __forceinline__ void long_row_at(const T* __restrict__ vp,
                                            const int32_t* __restrict__ cp, int64_t stride,
                                            int len, int w, const T* __restrict__ x,
                                            T* __restrict__ y, const int32_t* __restrict__ order,
                                            int64_t p, int64_t n_rows, int lane, uint64_t pol_s,
                                            uint64_t pol_x, T* __restrict__ stage) {
    const int64_t C = stride;
    T sum = T(0);
    // batch b's products are staged and added while batch b+1's val / col
    // loads and x gathers are already in flight (one round trip per batch
    // hidden behind the 128-step add chain)
    T prod[kSeg];
    {
        T v[kSeg];
        int32_t c[kSeg];
#pragma unroll
        for (int s = 0; s < kSeg; ++s) {
            const int j = s * 32 + lane;
            v[s] = T(0);
            c[s] = 0;
            if (j < len) {
                v[s] = ld_stream(vp + (int64_t)j * C, pol_s);
                c[s] = ld_stream(cp + (int64_t)j * C, pol_s);
            }
        }
#pragma unroll
        for (int s = 0; s < kSeg; ++s)
            prod[s] = (s * 32 + lane < len) ? Arith<T>::mul(v[s], ld_x(x + c[s], pol_x)) : T(0);
    }
    for (int j0 = 0; j0 < len; j0 += 32 * kSeg) {
        const int jn = j0 + 32 * kSeg;
        T vn[kSeg];
        int32_t cn[kSeg];
#pragma unroll
        for (int s = 0; s < kSeg; ++s) {
            const int j = jn + s * 32 + lane;
            vn[s] = T(0);
            cn[s] = 0;
            if (j < len) {
                vn[s] = ld_stream(vp + (int64_t)j * C, pol_s);
                cn[s] = ld_stream(cp + (int64_t)j * C, pol_s);
            }
        }
        __syncwarp();                        // previous batch fully consumed
#pragma unroll
        for (int s = 0; s < kSeg; ++s) stage[s * 32 + lane] = prod[s];
        __syncwarp();
        T xn[kSeg];
#pragma unroll
        for (int s = 0; s < kSeg; ++s)
            xn[s] = (jn + s * 32 + lane < len) ? ld_x(x + cn[s], pol_x) : T(0);
        const int nb = min(len - j0, kSeg * 32);      // warp-uniform
        int i = 0;
        for (; i + 8 <= nb; i += 8) {
            T q[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) q[k] = stage[i + k];
#pragma unroll
            for (int k = 0; k < 8; ++k) sum = Arith<T>::add(sum, q[k]);
        }
        for (; i < nb; ++i) sum = Arith<T>::add(sum, stage[i]);
#pragma unroll
        for (int s = 0; s < kSeg; ++s)
            prod[s] = (jn + s * 32 + lane < len) ? Arith<T>::mul(vn[s], xn[s]) : T(0);
    }
    if (pad_term<ORD>(order, p, n_rows, len < w))
        sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
    if (lane == 0) store_row<T, ACC, ORD>(y, order, p, n_rows, sum);
}

// ---------------------------------------------------------------------------
// cp.async ring helpers (the row-group kernel below)
// ---------------------------------------------------------------------------

template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int B>
__device__ __forceinline__ void cp_async(void* sdst, const void* gsrc, uint64_t pol) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;" ::"r"(s),
                 "l"(gsrc), "n"(B), "l"(pol)
                 : "memory");
}

// Group accounting of the copy ring (one commit group per issue):
// prologue VC(0..D-1), then X(0..E-1) each after cp_wait<D-1>; iteration b
// commits VC(b+D) then X(b+E).  wait_vc(b) leaves VC(b+E) landed, wait_x(b)
// leaves X(b) landed (exact counts in steady state, conservative -- waits
// for more -- in the first iterations).
template <int D, int E>
__device__ __forceinline__ void wait_vc(int b) {
    if (b >= D - 2 * E) cp_wait<2 * (D - E)>();
    else cp_wait<D>();
}
template <int E>
__device__ __forceinline__ void wait_x(int b) {
    if (b >= E - 1) cp_wait<2 * E>();
    else cp_wait<E + 1>();
}

// Row-group variant: one CTA per aligned group of 8 stored rows of one chunk
// (sorted chunks of long rows), warp-specialised.  Producer warps (4) copy
// the group's val/col and gather x into a cp.async ring and form the rounded
// products -- producer thread t takes row t % 8 of slot t / 8, so a
// warp-wide copy covers 4 slots x 8 adjacent rows = 4 contiguous 64-byte
// runs instead of the 32 scattered words of the warp-per-row role (which
// saturates the L1: l1tex 78 % of peak for cfg4's long rows).  The products
// go to a double buffer [row][slot]; in the chain warp lane r (< 8) adds row
// r's products in slot order, 16 at a time from registers loaded one block
// ahead (one 8-cycle DADD per slot; the shared-memory latency stays off the
// chain).  Producers and the chain hand the buffers over through named
// barriers (full / empty per buffer), so the chain of batch b overlaps the
// copies and products of batch b+1.
constexpr int kGP = 4;                  // producer warps
constexpr int kGT = (1 + kGP) * 32;     // + one chain warp

// non-.aligned forms: legal for a warp that is not converged (after the
// predicated copies / stores); the .aligned bar.sync raised "illegal
// instruction" once the group loop made divergence reach it
__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// 16 consecutive T from 16-byte-aligned shared memory
template <typename T>
__device__ __forceinline__ void lds16(const T* p, T (&q)[16]) {
    constexpr int V = 16 / sizeof(T);
#pragma unroll
    for (int k = 0; k < 16 / V; ++k) {
        const uint4 u = *reinterpret_cast<const uint4*>(p + k * V);
        const T* t = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int v = 0; v < V; ++v) q[k * V + v] = t[v];
    }
}

template <typename T, bool ACC, int ORD, int D, int E, int SB>
__global__ void __launch_bounds__(kGT)
k_spmv_long_grp(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                const int32_t* __restrict__ rl, const int32_t* __restrict__ col,
                const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y,
                const int32_t* __restrict__ order, int64_t C, int64_t p0, int64_t p1,
                int64_t n_rows, const int32_t* __restrict__ groups, int64_t n_groups,
                const int32_t* __restrict__ chunk_th, int l2pol) {
    constexpr int NS = D + 1;
    constexpr int NP = kGP * 32;               // producer threads
    constexpr int PER = SB * 8 / NP;           // (slot, row) entries per producer per batch
    constexpr int PS = SB + 16 / sizeof(T) * 2;  // row pitch: 16-byte aligned, rows 32 B apart mod 128
    static_assert(PER * NP == SB * 8, "SB * 8 must be a multiple of the producer count");
    static_assert(SB % 16 == 0, "SB must be a multiple of 16");
    // named barriers 1/2: buffer full, 3/4: buffer empty (0 is __syncthreads)
    extern __shared__ __align__(16) uint8_t lsm[];
    T* prod = reinterpret_cast<T*>(lsm);                          // [2][8][PS]
    T* sv = prod + 2 * 8 * PS;                                    // [NS][SB*8]
    T* sx = sv + NS * SB * 8;                                     // [NS][SB*8]
    int32_t* sc = reinterpret_cast<int32_t*>(sx + NS * SB * 8);   // [NS][SB*8]
    __shared__ int s_len[8];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t g0 = groups[blockIdx.x];
    const int64_t chunk = g0 / C;
    const int w = cl[chunk];
    const int th = chunk_th[chunk];
    if (tid < 8) {
        const int64_t row = g0 + tid;
        const int lr = rl[row];
        s_len[tid] = (lr > th && row >= p0 && row < p1) ? lr : 0;
    }
    __syncthreads();
    int maxlen = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) maxlen = max(maxlen, s_len[i]);
    const int nb = (maxlen + SB - 1) / SB;

    if (warp > 0) {                                    // ---- producers
        const uint64_t pol_s = make_policy(l2pol & 0xf);
        const uint64_t pol_x = make_policy((l2pol >> 4) & 0xf);
        const int pt = tid - 32;
        const int r = pt & 7;                          // fixed row per producer thread
        const int len = s_len[r];
        const int64_t base = cs[chunk] + (g0 - chunk * C) + r;
        const T* vp = val + base;
        const int32_t* cp = col + base;
        auto issue_vc = [&](int b) {
            if (b < nb) {
                const int st = b % NS;
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int e = k * NP + pt;
                    const int j = b * SB + (e >> 3);
                    if (j < len) {
                        cp_async<sizeof(T)>(sv + st * SB * 8 + e, vp + (int64_t)j * C, pol_s);
                        cp_async<4>(sc + st * SB * 8 + e, cp + (int64_t)j * C, pol_s);
                    }
                }
            }
            cp_commit();
        };
        auto issue_x = [&](int b) {
            if (b < nb) {
                const int st = b % NS;
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int e = k * NP + pt;
                    if (b * SB + (e >> 3) < len)
                        cp_async<sizeof(T)>(sx + st * SB * 8 + e, x + sc[st * SB * 8 + e],
                                            pol_x);
                }
            }
            cp_commit();
        };
#pragma unroll
        for (int b = 0; b < D; ++b) issue_vc(b);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            cp_wait<D - 1>();
            issue_x(e);
        }
        for (int b = 0; b < nb; ++b) {
            issue_vc(b + D);
            wait_vc<D, E>(b);
            issue_x(b + E);
            wait_x<E>(b);
            const int st = b % NS;
            if (b >= 2) named_sync(3 + (b & 1), kGT);     // chain done with batch b-2
            T* pb = prod + (b & 1) * 8 * PS;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int e = k * NP + pt;
                const int jj = e >> 3;
                const int i = st * SB * 8 + e;
                pb[r * PS + jj] = (b * SB + jj < len) ? Arith<T>::mul(sv[i], sx[i]) : T(0);
            }
            named_arrive(1 + (b & 1), kGT);
        }
        cp_wait<0>();
        for (int b = max(nb - 2, 0); b < nb; ++b) named_sync(3 + (b & 1), kGT);  // drain
        return;
    }
    // ---- chain warp: lane r sums row g0 + r (lanes 8..31 mirror lanes 0..7)
    const int r = lane & 7;
    T sum = T(0);
    for (int b = 0; b < nb; ++b) {
        named_sync(1 + (b & 1), kGT);
        // +0.0 products past a row's end are exact no-ops (the sum starts at
        // +0.0 and is never -0.0): the chain runs the whole batch
        const T* q = prod + (b & 1) * 8 * PS + r * PS;
        T cur[16], nxt[16];
        lds16(q, cur);
#pragma unroll
        for (int k = 0; k < SB / 16; ++k) {
            if (k + 1 < SB / 16) lds16(q + (k + 1) * 16, nxt);
#pragma unroll
            for (int u = 0; u < 16; ++u) sum = Arith<T>::add(sum, cur[u]);
#pragma unroll
            for (int u = 0; u < 16; ++u) cur[u] = nxt[u];
        }
        named_arrive(3 + (b & 1), kGT);
    }
    if (lane < 8 && s_len[r] > 0) {
        const int64_t row = g0 + r;
        if (pad_term<ORD>(order, row, n_rows, s_len[r] < w))
            sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
        store_row<T, ACC, ORD>(y, order, row, n_rows, sum);
    }
}

template <typename T, int D, int SB>
constexpr size_t grp_smem() {
    return (size_t)(D + 1) * SB * 8 * (2 * sizeof(T) + 4) +
           2 * 8 * (SB + 16 / sizeof(T) * 2) * sizeof(T);
}

// The SpMV kernel.  Blocks [0, n_long_blocks) take the long-row role (one
// warp per row of long_rows[], longest first, so they start early and
// overlap the bulk); the remaining blocks take one thread per stored row p
// in [p0, p1) (the paper's GPU design; for C = 32 a warp owns a chunk).
// CC > 0: compile-time chunk height.  ORD 0: y[p] in stored order; ORD 1:
// y[order[p]] for real rows (fused unpermute).  In chunks wider than
// long_th, rows longer than the chunk's threshold chunk_th[] belong to the
// long-row role (the same rule builds long_rows[], sellb_build.cu) and the
// others stop at their own length (pad-skip semantics).
template <typename T, int CC, bool SKIP, bool ACC, int ORD, int U, bool LONG>
#ifndef SELLB_F64_BLOCKS
#define SELLB_F64_BLOCKS 5
#endif
#ifndef SELLB_F32_BLOCKS
#define SELLB_F32_BLOCKS 6   // fp32 U=8: 40 regs, 48 warps/SM (tools/f32occ_ab.sh: cfg4 f32 881 -> 1050)
#endif
// U = 6: 8 blocks (32 registers) for the plain C = 32 pad-inclusive store
// (no spills; cfg5 919 -> 926 GF/s), 6 for the instances that would spill
__global__ void __launch_bounds__(kThreads, U == 4 ? (LONG ? 6 : 8)
                                             : (U == 6 ? ((CC == 32 && !SKIP && !ACC) ? 8 : 6)
                                                       : (sizeof(T) == 4 ? SELLB_F32_BLOCKS
                                                                         : SELLB_F64_BLOCKS)))
k_spmv_sell(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
            const int32_t* __restrict__ rl, const int32_t* __restrict__ col,
            const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y,
            const int32_t* __restrict__ order, int64_t C_rt, int64_t p0, int64_t p1,
            int64_t n_rows, const int32_t* __restrict__ long_rows, int64_t n_long,
            int long_th, const int32_t* __restrict__ chunk_th, int l2pol,
            const int64_t* __restrict__ side_off, const int32_t* __restrict__ side_col,
            const T* __restrict__ side_val) {
    const int64_t C = CC > 0 ? (int64_t)CC : C_rt;
    const uint64_t pol_s = make_policy(l2pol & 0xf);
    const uint64_t pol_x = make_policy((l2pol >> 4) & 0xf);
    // block size: kThreads, or fewer (SELLB_BULK_BT) -- index math uses blockDim
    const int64_t wpb = blockDim.x >> 5;
    const int64_t n_long_blocks = LONG ? (n_long + wpb - 1) / wpb : 0;
    if constexpr (LONG) {
        if ((int64_t)blockIdx.x < n_long_blocks) {
            __shared__ T stage[kThreads / 32][kSeg * 32];
            const int64_t k = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
            if (k >= n_long) return;
            const int64_t p = long_rows[k];
            if (p < p0 || p >= p1) return;
            const int64_t chunk = p / C;
            if (side_off) {             // the row, contiguous (long-row side table)
                const int64_t o = side_off[k];
                long_row_at<T, ACC, ORD>(side_val + o, side_col + o, 1, rl[p], cl[chunk], x, y,
                                         order, p, n_rows, threadIdx.x & 31, pol_s, pol_x,
                                         stage[threadIdx.x >> 5]);
            } else {
                const int64_t base = cs[chunk] + (p - chunk * C);
                long_row_at<T, ACC, ORD>(val + base, col + base, C, rl[p], cl[chunk], x, y,
                                         order, p, n_rows, threadIdx.x & 31, pol_s, pol_x,
                                         stage[threadIdx.x >> 5]);
            }
            return;
        }
    }
    const int64_t p = p0 + ((int64_t)blockIdx.x - n_long_blocks) * (int64_t)blockDim.x +
                      threadIdx.x;
    if (p >= p1) return;
    const int64_t chunk = p / C;
    const int64_t base = cs[chunk] + (p - chunk * C);
    const int w = cl[chunk];
    int len = SKIP ? rl[p] : w;
    bool skip_pad = SKIP;
    if constexpr (ORD == 2 && !SKIP) {
        // the shadow layout, pad-inclusive: its own padding slots add
        // 0 * x[0], an exact no-op while x[0] is finite (the sum starts at
        // +0.0 and is never -0.0); otherwise they are skipped and only the
        // caller's padding term (the map's bit 31) applies
        if (!isfinite(__ldg(x))) {
            len = rl[p];
            skip_pad = true;
        }
    }
    if (LONG && w > long_th) {           // a chunk that may hold long rows
        if (!SKIP) len = rl[p];
        if (len > chunk_th[chunk]) return;   // owned by the long-row role
        skip_pad = true;
    }
    const T* vp = val + base;
    const int32_t* cp = col + base;
    // the output map entry (the shadow's flagged map, or the stored ->
    // original order of the fused unpermute) is loaded before the row's
    // slots, so its latency hides under them instead of trailing the sum
    // (cfg3 sigma = 1 / 512 through the shadow: 780 / 806 -> 831 / 853 GF/s)
    int32_t map = 0x7fffffff;
    if constexpr (ORD != 0) {
        if (p < n_rows) map = __ldg(order + p);
    }
    // vector x loads only in the C = 32 instances (the generic-C ones have
    // no registers to spare for them)
    T sum = row_sum<T, U>(vp, cp, C, len, x, pol_s, pol_x, CC == 32 && ((l2pol >> 8) & 1));
    if constexpr (ORD == 2) {
        // bit 31: the caller's chunk padded this row (pad_term / store_row)
        if (map < 0) sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
        const int32_t o = map & 0x7fffffff;
        if (o != 0x7fffffff) y[o] = ACC ? Arith<T>::add(y[o], sum) : sum;
    } else if constexpr (ORD == 1) {
        if (skip_pad && len < w) sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
        if (p < n_rows) y[map] = ACC ? Arith<T>::add(y[map], sum) : sum;
    } else {
        if (pad_term<ORD>(order, p, n_rows, skip_pad && len < w))
            sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
        store_row<T, ACC, ORD>(y, order, p, n_rows, sum);
    }
}

// Warp-level variant for very short chunks (C = 32, every chunk at most W
// slots wide: diagonal / tridiagonal-like rows): one warp owns K consecutive
// chunks, lane = row in each, and issues all K chunks' metadata loads, then
// all K*W val/col loads, then all x gathers before the first add -- K times
// the bytes in flight of the one-chunk-per-warp grid, whose rows carry too
// little data to cover three dependent DRAM round trips (16 M rows of width
// 1: 3.7 TB/s).  Each row is still summed in slot order from +0.0.
template <typename T, bool SKIP, bool ACC, int ORD, int K, int W>
__global__ void __launch_bounds__(kThreads)
k_spmv_sell_short(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                  const int32_t* __restrict__ rl, const int32_t* __restrict__ col,
                  const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y,
                  const int32_t* __restrict__ order, int64_t c0, int64_t c1, int64_t n_rows,
                  int l2pol) {
    const uint64_t pol_s = make_policy(l2pol & 0xf);
    const uint64_t pol_x = make_policy((l2pol >> 4) & 0xf);
    const int lane = threadIdx.x & 31;
    const int64_t cb = c0 + ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * K;
    if (cb >= c1) return;
    int64_t base[K];
    int w[K], len[K];
    // shadow layout (ORD 2), pad-inclusive: its own padding is skipped when
    // x[0] is not finite (see k_spmv_sell)
    const bool own_skip = SKIP || (ORD == 2 && !isfinite(__ldg(x)));
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int64_t c = cb + k;
        base[k] = 0;
        w[k] = 0;
        len[k] = 0;
        if (c < c1) {
            base[k] = cs[c];
            w[k] = cl[c];
            len[k] = own_skip ? rl[c * 32 + lane] : w[k];
        }
    }
    T v[K][W];
    int32_t ci[K][W];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int j = 0; j < W; ++j) {
            v[k][j] = T(0);
            ci[k][j] = 0;
            if (j < len[k]) {
                v[k][j] = ld_stream(val + base[k] + j * 32 + lane, pol_s);
                ci[k][j] = ld_stream(col + base[k] + j * 32 + lane, pol_s);
            }
        }
    T xv[K][W];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int j = 0; j < W; ++j) xv[k][j] = j < len[k] ? ld_x(x + ci[k][j], pol_x) : T(0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (cb + k >= c1) break;
        T sum = T(0);
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j < len[k]) sum = Arith<T>::add(sum, Arith<T>::mul(v[k][j], xv[k][j]));
        if (pad_term<ORD>(order, (cb + k) * 32 + lane, n_rows, SKIP && len[k] < w[k]))
            sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
        store_row<T, ACC, ORD>(y, order, (cb + k) * 32 + lane, n_rows, sum);
    }
}

// Chunk-list variant (multi-GPU interior / boundary passes): block b handles
// kThreads consecutive stored rows of chunk ids[...]; generic C.
template <typename T, bool SKIP, bool ACC>
__global__ void __launch_bounds__(kThreads)
k_spmv_sell_list(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
                 const int32_t* __restrict__ rl, const int32_t* __restrict__ col,
                 const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y,
                 const int32_t* __restrict__ ids, int64_t n_ids, int64_t C) {
    const int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (t >= n_ids * C) return;
    const int64_t k = t / C;
    const int64_t r = t - k * C;
    const int64_t chunk = ids[k];
    const int64_t p = chunk * C + r;
    const int64_t base = cs[chunk] + r;
    const int w = cl[chunk];
    const int len = SKIP ? rl[p] : w;
    const uint64_t pol_s = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    T sum = T(0);
    for (int j = 0; j < len; ++j) {
        T v = ld_stream(val + base + (int64_t)j * C, pol_s);
        int32_t c = ld_stream(col + base + (int64_t)j * C, pol_s);
        sum = Arith<T>::add(sum, Arith<T>::mul(v, ld_x(x + c, pol_x)));
    }
    if (SKIP && len < w) sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
    y[p] = ACC ? Arith<T>::add(y[p], sum) : sum;
}

// chunk_flag[c] = OR over the chunk's stored rows of row_flag[original row]
// (one warp per chunk)
__global__ void k_chunk_flags(const int32_t* __restrict__ order, int64_t n_rows, int64_t n_chunks,
                              int64_t C, const uint8_t* __restrict__ row_flag,
                              uint8_t* __restrict__ chunk_flag) {
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= n_chunks) return;
    int f = 0;
    for (int64_t r = lane; r < C; r += 32) {
        const int64_t o = order[c * C + r];
        if (o < n_rows) f |= row_flag[o] != 0;
    }
    f = __any_sync(0xffffffffu, f);
    if (lane == 0) chunk_flag[c] = (uint8_t)f;
}

// Padding fix-up for the row-partitioned path (see sellb_pad_fixup).
template <typename T>
__global__ void __launch_bounds__(kThreads)
k_pad_fixup(const int32_t* __restrict__ cl, const int32_t* __restrict__ rl, int64_t C,
            int64_t n_pad, const T* __restrict__ x0, T* __restrict__ y) {
    const T v = *x0;
    if (isfinite(v)) return;
    const int64_t p = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (p >= n_pad) return;
    if (rl[p] < cl[p / C]) y[p] = Arith<T>::add(y[p], Arith<T>::mul(T(0), v));
}

// CRS kernels (_kernels.pyx:17-62), one thread per row, reference order.
template <typename T, bool ACC>
__global__ void __launch_bounds__(kThreads)
k_spmv_crs(const int64_t* __restrict__ rpt, const int32_t* __restrict__ col,
           const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y, int64_t r0,
           int64_t r1) {
    const int64_t i = r0 + (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (i >= r1) return;
    T tmp = T(0);
    for (int64_t j = rpt[i]; j < rpt[i + 1]; ++j)
        tmp = Arith<T>::add(tmp, Arith<T>::mul(val[j], __ldg(x + col[j])));
    y[i] = ACC ? Arith<T>::add(y[i], tmp) : tmp;
}

template <typename T, bool ACC>
__global__ void __launch_bounds__(kThreads)
k_spmv_crs_unrolled(const int64_t* __restrict__ rpt, const int32_t* __restrict__ col,
                    const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y,
                    int64_t r0, int64_t r1) {
    using A = Arith<T>;
    const int64_t i = r0 + (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (i >= r1) return;
    const int64_t s = rpt[i], e = rpt[i + 1];
    const int64_t m = s + ((e - s) & ~(int64_t)3);
    T t0 = 0, t1 = 0, t2 = 0, t3 = 0, acc;
    int64_t j = s;
    for (; j < m; j += 4) {
        t0 = A::add(t0, A::mul(val[j], __ldg(x + col[j])));
        t1 = A::add(t1, A::mul(val[j + 1], __ldg(x + col[j + 1])));
        t2 = A::add(t2, A::mul(val[j + 2], __ldg(x + col[j + 2])));
        t3 = A::add(t3, A::mul(val[j + 3], __ldg(x + col[j + 3])));
    }
    const T comb = A::add(A::add(A::add(t0, t1), t2), t3);
    acc = ACC ? A::add(y[i], comb) : comb;
    for (; j < e; ++j) acc = A::add(acc, A::mul(val[j], __ldg(x + col[j])));
    y[i] = acc;
}

// Row-run kernel: one warp per 32 consecutive rows whose entries form one
// contiguous run [rpt[rb], rpt[rb+32]) -- the CRS arrays (_kernels.pyx:17-62)
// or the packed stored-order copy of a SELL matrix (build_packed).  The warp
// streams the run through a shared-memory stage of S entries:
//   phase 1 -- sub-batches of 32 U entries: lane t loads entries t, t+32, ...
//              (dense, coalesced val / col loads, every lane busy whatever
//              the row lengths), gathers x, stores the rounded products; the
//              next sub-batch's loads are issued before this one's gathers
//              are consumed;
//   phase 2 -- lane l walks row rb + l's products in the stage, in order.
// Runs longer than S go window by window.  The plain walk adds each row's
// products to one sum from +0.0 (the reference's loop), the unrolled one
// into t[j % 4] over the first 4 floor(len/4) entries, combines
// ((t0 + t1) + t2) + t3, adds y when accumulating, then the tail
// (_kernels.pyx:34-62) -- bitwise the reference either way.
// MODE 0: CRS rows, y[i].  MODE 1: packed SELL rows (stored row p = i): y[p]
// (ORD 0) or y[order[p]] (ORD 1), plus the reference's 0 * x[0] term for
// rows shorter than their chunk (the padding slots it adds).
template <typename T, bool ACC, bool UNR, int MODE, int ORD, int U, int S>
__global__ void __launch_bounds__(kThreads, U >= 8 ? 2 : (S * sizeof(T) <= 6144 && !(MODE == 0 && sizeof(T) == 8 && (ACC || UNR)) ? 4 : 3))
k_spmv_rows(const int64_t* __restrict__ rpt, const int32_t* __restrict__ col,
            const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y,
            int64_t r0, int64_t r1, const int32_t* __restrict__ order,
            const int32_t* __restrict__ cl, const int32_t* __restrict__ rl, int64_t n_rows) {
    constexpr int WPB = kThreads / 32;
    constexpr int B = 32 * U;
    static_assert(S % B == 0, "stage must hold whole sub-batches");
    extern __shared__ __align__(16) uint8_t rows_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* st = reinterpret_cast<T*>(rows_smem) + (size_t)warp * S;
    const uint64_t pol_s = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    // persistent warps: group g = 32 rows; the first sub-batch of the next
    // group (and its offsets) is fetched before this group's in-order walks,
    // so the matrix stream stays in flight while a warp adds
    const int64_t n_groups = (r1 - r0 + 31) / 32;
    const int64_t GW = (int64_t)gridDim.x * WPB;
    int64_t g = (int64_t)blockIdx.x * WPB + warp;
    if (g >= n_groups) return;
    auto group_base = [&](int64_t gg) { return rpt[r0 + gg * 32]; };
    auto group_end = [&](int64_t gg) { return rpt[min(r0 + gg * 32 + 32, r1)]; };
    T v[U];
    int32_t ci[U];
    auto load_first = [&](int64_t b0, int64_t en) {
        const int64_t wn0 = min((int64_t)S, en - b0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int t = u * 32 + lane;
            v[u] = T(0);
            ci[u] = 0;
            if (t < wn0) {
                v[u] = ld_stream(val + b0 + t, pol_s);
                ci[u] = ld_stream(col + b0 + t, pol_s);
            }
        }
    };
    int64_t base = group_base(g), end = group_end(g);
    load_first(base, end);
    while (true) {
        const int64_t rb = r0 + g * 32;
        const int64_t i = rb + lane;
        const bool valid = i < r1;
        const int64_t s = valid ? rpt[i] : 0;
        const int64_t e = valid ? rpt[i + 1] : 0;
        const int64_t gn = g + GW;
        const bool has_next = gn < n_groups;
        const int64_t nbase = has_next ? group_base(gn) : 0;
        const int64_t nend = has_next ? group_end(gn) : 0;
        const int64_t m4 = s + ((e - s) & ~(int64_t)3);
        int64_t pos = s;
        T sum = T(0), t0 = T(0), t1 = T(0), t2 = T(0), t3 = T(0);
        bool tail = !UNR;
        bool prefetched = false;
        for (int64_t wb = base; wb < end; wb += S) {
            const int64_t we = min(wb + (int64_t)S, end);
            const int wn = (int)(we - wb);             // window entries (<= S)
            const T* __restrict__ vw = val + wb;
            const int32_t* __restrict__ cw = col + wb;
            if (wb != base) load_first(wb, end);
            for (int sb = 0; sb < wn; sb += B) {
                T xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    xv[u] = (sb + u * 32 + lane < wn) ? ld_x(x + ci[u], pol_x) : T(0);
                T vn[U];
                int32_t cn[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int t = sb + B + u * 32 + lane;
                    vn[u] = T(0);
                    cn[u] = 0;
                    if (t < wn) {
                        vn[u] = ld_stream(vw + t, pol_s);
                        cn[u] = ld_stream(cw + t, pol_s);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (sb + u * 32 + lane < wn)
                        st[sb + u * 32 + lane] = Arith<T>::mul(v[u], xv[u]);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    v[u] = vn[u];
                    ci[u] = cn[u];
                }
            }
            if (we == end && has_next) {               // the next group's stream
                load_first(nbase, nend);
                prefetched = true;
            }
            __syncwarp();
            // phase 2: this row's products inside the window, in order
            const T* sp = st - wb;
            if (!UNR) {
                const int64_t stop = min(e, we);
                for (; pos + 4 <= stop; pos += 4) {
                    const T a0 = sp[pos], a1 = sp[pos + 1], a2 = sp[pos + 2], a3 = sp[pos + 3];
                    sum = Arith<T>::add(sum, a0);
                    sum = Arith<T>::add(sum, a1);
                    sum = Arith<T>::add(sum, a2);
                    sum = Arith<T>::add(sum, a3);
                }
                for (; pos < stop; ++pos) sum = Arith<T>::add(sum, sp[pos]);
            } else {
                const int64_t stop4 = min(m4, we);
                // whole groups of four (pos - s is a multiple of 4 here unless a
                // window boundary split a group: then one entry at a time)
                while (pos < stop4) {
                    if (((pos - s) & 3) == 0 && pos + 4 <= stop4) {
                        t0 = Arith<T>::add(t0, sp[pos]);
                        t1 = Arith<T>::add(t1, sp[pos + 1]);
                        t2 = Arith<T>::add(t2, sp[pos + 2]);
                        t3 = Arith<T>::add(t3, sp[pos + 3]);
                        pos += 4;
                    } else {
                        const int k = (int)((pos - s) & 3);
                        const T pr = sp[pos];
                        if (k == 0) t0 = Arith<T>::add(t0, pr);
                        else if (k == 1) t1 = Arith<T>::add(t1, pr);
                        else if (k == 2) t2 = Arith<T>::add(t2, pr);
                        else t3 = Arith<T>::add(t3, pr);
                        ++pos;
                    }
                }
                const int64_t stop = min(e, we);
                if (pos >= m4 && pos < stop && !tail) {
                    const T comb = Arith<T>::add(Arith<T>::add(Arith<T>::add(t0, t1), t2), t3);
                    sum = ACC ? Arith<T>::add(y[i], comb) : comb;
                    tail = true;
                }
                for (; pos < stop; ++pos) sum = Arith<T>::add(sum, sp[pos]);
            }
            __syncwarp();
        }
        if (!prefetched && has_next) load_first(nbase, nend);   // an empty group
        if (valid) {
            if (MODE == 0) {
                if (!UNR) {
                    y[i] = ACC ? Arith<T>::add(y[i], sum) : sum;
                } else {
                    if (!tail) {
                        const T comb =
                            Arith<T>::add(Arith<T>::add(Arith<T>::add(t0, t1), t2), t3);
                        sum = ACC ? Arith<T>::add(y[i], comb) : comb;
                    }
                    y[i] = sum;
                }
            } else {
                const int len = rl[i];
                if ((int64_t)(e - s) == len) {        // else a long row: the warp-per-row role's
                    if (len < cl[i >> 5]) sum = Arith<T>::add(sum, Arith<T>::mul(T(0), __ldg(x)));
                    store_row<T, ACC, ORD>(y, order, i, n_rows, sum);
                }
            }
        }
        if (!has_next) break;
        g = gn;
        base = nbase;
        end = nend;
    }
}

constexpr int kRowsU = 4;
#ifndef SELLB_ROWS_S
#define SELLB_ROWS_S 768
#endif
constexpr int kRowsS = SELLB_ROWS_S;

template <typename T, bool ACC, bool UNR, int MODE, int ORD>
void launch_rows(const int64_t* rpt, const int32_t* col, const void* val, const void* x, void* y,
                 int64_t r0, int64_t r1, const int32_t* order, const int32_t* cl,
                 const int32_t* rl, int64_t n_rows, cudaStream_t st) {
    // stage of 768 entries per warp, 4 blocks / SM at 64 registers (A/B of
    // 256 / 512 / 1024 at 3 blocks: cfg2 CRS 544 / 656 / 697, cfg3 411 / 455 /
    // 455 GF/s; 768 at 4 blocks vs 1024 at 3: cfg3 447 -> 480, cfg4 288 ->
    // 323, cfg2 688 -> 656)
    // persistent grid: one wave (the kernel's resident blocks per SM x SMs),
    // each warp walks groups warp, warp + all warps, ...
    static const int sms_ = [] {
        int d = 0, n = 148;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
        return n;
    }();
    const int64_t groups_ = grid_for(grid_for(r1 - r0, 32), kThreads / 32);
#define SELLB_ROWS(UU, SS)                                                                     \
    do {                                                                                       \
        auto kern = k_spmv_rows<T, ACC, UNR, MODE, ORD, UU, SS>;                               \
        constexpr size_t smem_ = (size_t)(kThreads / 32) * SS * sizeof(T);                     \
        static unsigned attr_ = 0;                                                             \
        static int bps_ = 0;                                                                   \
        int dev_ = 0;                                                                          \
        cudaGetDevice(&dev_);                                                                  \
        if (!(attr_ & (1u << (dev_ & 31)))) {                                                  \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_); \
            attr_ |= 1u << (dev_ & 31);                                                        \
            if (!bps_ && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_, kern, kThreads,  \
                                                                       smem_) != cudaSuccess) \
                bps_ = 1;                                                                      \
        }                                                                                      \
        const unsigned grid = (unsigned)std::max<int64_t>(                                     \
            1, std::min<int64_t>(groups_, (int64_t)sms_ * std::max(bps_, 1)));                 \
        kern<<<grid, kThreads, smem_, st>>>(rpt, col, (const T*)val, (const T*)x, (T*)y, r0,   \
                                            r1, order, cl, rl, n_rows);                        \
    } while (0)
    // U = 4 (B = 128-entry sub-batches, 3 blocks / SM): U = 8 measured slower
    // everywhere (cfg2 / cfg3 / cfg4 CRS 698 / 452 / 289 -> 622 / 380 / 239)
    SELLB_ROWS(kRowsU, kRowsS);
#undef SELLB_ROWS
    count_launches();
}

// The warp-per-row role alone (one warp per row of rows[], side table or
// SELL arrays): the long rows next to the packed copy's row-run kernel.
template <typename T, bool ACC, int ORD>
__global__ void __launch_bounds__(kThreads)
k_long_rows(const int64_t* __restrict__ cs, const int32_t* __restrict__ cl,
            const int32_t* __restrict__ rl, const int32_t* __restrict__ col,
            const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y,
            const int32_t* __restrict__ order, int64_t C, int64_t p0, int64_t p1, int64_t n_rows,
            const int32_t* __restrict__ rows, int64_t n_long, int l2pol,
            const int64_t* __restrict__ side_off, const int32_t* __restrict__ side_col,
            const T* __restrict__ side_val) {
    constexpr int WPB = kThreads / 32;
    __shared__ T stage[WPB][kSeg * 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * WPB + warp;
    if (k >= n_long) return;
    const int64_t p = rows[k];
    if (p < p0 || p >= p1) return;
    const uint64_t pol_s = make_policy(l2pol & 0xf);
    const uint64_t pol_x = make_policy((l2pol >> 4) & 0xf);
    const int64_t chunk = p / C;
    if (side_off) {
        const int64_t o = side_off[k];
        long_row_at<T, ACC, ORD>(side_val + o, side_col + o, 1, rl[p], cl[chunk], x, y, order, p,
                                 n_rows, lane, pol_s, pol_x, stage[warp]);
    } else {
        const int64_t base = cs[chunk] + (p - chunk * C);
        long_row_at<T, ACC, ORD>(val + base, col + base, C, rl[p], cl[chunk], x, y, order, p,
                                 n_rows, lane, pol_s, pol_x, stage[warp]);
    }
}

// The packed copy: its long rows (rows longer than kPackedLong) by the
// warp-per-row role on the highest-priority side stream, started first; the
// row-run kernel (MODE 1) on the caller's stream; joined.
template <typename T, bool ACC, int ORD>
int launch_packed(const sellb_mat* m, const void* x, void* y, int64_t p0, int64_t p1,
                  cudaStream_t st) {
    const int64_t n_long = m->long_rows ? m->n_long : 0;
    sellb_mat* mm = const_cast<sellb_mat*>(m);
    std::unique_lock<std::mutex> lk(mm->long_mu, std::defer_lock);
    if (n_long) {
        lk.lock();
        if (!mm->long_ready) {
            int prio_lo = 0, prio_hi = 0;
            SELLB_CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
            SELLB_CU(cudaStreamCreateWithPriority(&mm->s_long, cudaStreamNonBlocking, prio_hi));
            SELLB_CU(cudaEventCreateWithFlags(&mm->ev_fork, cudaEventDisableTiming));
            SELLB_CU(cudaEventCreateWithFlags(&mm->ev_join, cudaEventDisableTiming));
            mm->long_ready = true;
        }
        SELLB_CU(cudaEventRecord(mm->ev_fork, st));
        SELLB_CU(cudaStreamWaitEvent(mm->s_long, mm->ev_fork, 0));
        const bool side = m->side_off && m->n_rest == n_long;
        const int l2pol = (int64_t)m->n_cols * (int64_t)sizeof(T) > (64LL << 20) ? 0x21 : 0x20;
        k_long_rows<T, ACC, ORD><<<(unsigned)grid_for(n_long, kThreads / 32), kThreads, 0,
                                   mm->s_long>>>(
            m->cs, m->cl, m->rl, m->col, (const T*)m->val, (const T*)x, (T*)y, m->order, m->C,
            p0, p1, m->n_rows, side ? m->long_rest : m->long_rows, n_long, l2pol,
            side ? m->side_off : nullptr, side ? m->side_col : nullptr,
            (const T*)(side ? m->side_val : nullptr));
        count_launches();
        SELLB_CU(cudaEventRecord(mm->ev_join, mm->s_long));
    }
    launch_rows<T, ACC, false, 1, ORD>(m->prpt, m->pcol, m->pval, x, y, p0, p1, m->order, m->cl,
                                       m->rl, m->n_rows, st);
    if (n_long) SELLB_CU(cudaStreamWaitEvent(st, mm->ev_join, 0));
    return 0;
}

template <typename T, int CC, bool SKIP, bool ACC, int ORD>
int dispatch_u(const sellb_mat* m, const void* x, void* y, int64_t p0, int64_t p1,
               cudaStream_t st, const int32_t* ordp) {
    const int64_t rows = p1 - p0;
    if (rows <= 0) return 0;
    const int64_t n_long = m->long_rows ? m->n_long : 0;
    constexpr int bt = kThreads;   // 64 / 128-thread blocks measured within noise (r01_bt_ab.txt)
    const int64_t long_blocks = (n_long + bt / 32 - 1) / (bt / 32);
    unsigned grid = (unsigned)(grid_for(rows, bt) + long_blocks);
    // L2 policies: matrix streams (low nibble) and x gathers (high nibble);
    // 0 evict_first, 1 evict_normal, 2 evict_last.  x is always evict_last;
    // the matrix stream is evict_first while x fits comfortably in L2 and
    // evict_normal once it does not (measured: cfg2 987 vs 939
    // GF/s, cfg5 612 vs 713 GF/s).  SELLB_L2POL overrides.
    static const int l2pol_env = [] {
        const char* e = getenv("SELLB_L2POL");
        return e ? (int)strtol(e, nullptr, 0) : -1;
    }();
    // bit 8: vector x loads for consecutive-column batches (gather_x);
    // needs a 16-byte aligned x.  SELLB_VX=0 disables.
    static const int vx_env = [] {
        const char* e = getenv("SELLB_VX");
        return e ? atoi(e) : 1;
    }();
    const int vx = (vx_env && ((uintptr_t)x & 15) == 0) ? 0x100 : 0;
    const int l2pol = (l2pol_env >= 0 ? l2pol_env
                       : ((int64_t)m->n_cols * (int64_t)sizeof(T) > (64LL << 20) ? 0x21 : 0x20))
                      | vx;
    // slots batched per load round: 8 for fp32 (half the bytes per slot),
    // long rows (N_nzr >= 24) and skewed matrices (some chunk wider than 64),
    // else 4 (measured, tools/ab_env.sh: cfg2 f32 1230 -> 1377 GF/s, cfg3
    // sigma=128 261 -> 310; cfg1 443 -> 376 and cfg5 878 -> 864 prefer 4).
    static const int u_env = [] {
        const char* e = getenv("SELLB_U");
        return e ? atoi(e) : 0;
    }();
    // rows of 16..24 entries (the cfg5 banded matrix: 19.7): 8 slots per batch
    // for the pad-skipping bulk, 6 for the pad-inclusive one (measured on
    // cfg5, one box: sigma=1 pad-skip U 4 / 6 / 8 -> 728 / 806 / 845 GF/s,
    // sigma=512 pad-incl 889 / 918 / 908; cfg2 at 26.6 per row keeps U = 8)
    const bool mid_rows = m->n_rows > 0 && m->nnz >= 16 * m->n_rows &&
                          m->nnz < 24 * m->n_rows;
    const bool u8 = u_env ? u_env == 8
                          : (sizeof(T) == 4 || m->max_cl > 64 ||
                             (m->n_rows > 0 && m->nnz >= 24 * m->n_rows) || (SKIP && mid_rows));
#define SELLB_LAUNCH(UU, LL, LR, NL, TH, SD)                                                    \
    do {                                                                                        \
        /* LONG instances run next to the row-group kernel: reserve shared */ \
        /* memory for one group CTA per SM up front (30 %), so an SM never */ \
        /* has to drain its bulk blocks to change its carve-out when a     */ \
        /* group CTA arrives (cfg3 sigma=N 495 -> 757 GF/s, tools/         */ \
        /* long_cfg_ab.sh; neutral in the fused mode)                      */ \
        if (LL) {                                                                               \
            static unsigned set_ = 0;   /* per-device bit */                                    \
            int dev_ = 0;                                                                       \
            cudaGetDevice(&dev_);                                                               \
            if (!(set_ & (1u << (dev_ & 31)))) {                                                \
                cudaFuncSetAttribute(k_spmv_sell<T, CC, SKIP, ACC, ORD, UU, LL>,                \
                                     cudaFuncAttributePreferredSharedMemoryCarveout, 30);       \
                set_ |= 1u << (dev_ & 31);                                                      \
            }                                                                                   \
        }                                                                                       \
        k_spmv_sell<T, CC, SKIP, ACC, ORD, UU, LL><<<grid, bt, 0, st>>>(                        \
            m->cs, m->cl, m->rl, m->col, (const T*)m->val, (const T*)x, (T*)y, ordp,        \
            m->C, p0, p1, m->n_rows, LR, NL, TH, m->chunk_th, l2pol,                            \
            (SD) ? m->side_off : nullptr, (SD) ? m->side_col : nullptr,                         \
            (const T*)((SD) ? m->side_val : nullptr));                                          \
        count_launches();                                                                       \
    } while (0)
    // very short chunks (every chunk <= 2 slots): K chunks per warp
    // (k_spmv_sell_short).  Measured on 16 M rows (tools/short_ab.sh): width 1
    // 126 -> 74 us (K = 4, 6.3 TB/s), width 2 138 -> 111 us (K = 2); width 3
    // gains nothing (152 vs 156 us) and stays on the default grid.
    // SELLB_SHORT=0 disables.
    static const int short_env = [] {
        const char* e = getenv("SELLB_SHORT");
        return e ? atoi(e) : 1;
    }();
    if (CC == 32 && !n_long && short_env && m->max_cl <= 2) {
        const int64_t chunks = (p1 - p0) / 32;
#define SELLB_SHORT_LAUNCH(KK, WW)                                                              \
    k_spmv_sell_short<T, SKIP, ACC, ORD, KK, WW>                                                \
        <<<(unsigned)((chunks + (kThreads / 32) * KK - 1) / ((kThreads / 32) * KK)), kThreads, 0, \
           st>>>(m->cs, m->cl, m->rl, m->col, (const T*)m->val, (const T*)x, (T*)y, ordp,   \
                 p0 / 32, p1 / 32, m->n_rows, l2pol)
        if (m->max_cl <= 1) SELLB_SHORT_LAUNCH(4, 1);
        else SELLB_SHORT_LAUNCH(2, 2);
        count_launches();
#undef SELLB_SHORT_LAUNCH
        return 0;
    }
    // long rows: SELLB_LONG_MODE 0 = warp-per-row role fused into the bulk
    // launch; 1 = long-row kernels, then the bulk, on the caller's stream;
    // 2 (default) = long-row kernels on a side stream forked from and joined
    // back into the caller's stream, overlapping the bulk.  The side stream
    // has the device's greatest priority: the block scheduler dispatches its
    // CTAs ahead of pending bulk blocks (at equal priority they were
    // sometimes queued behind the whole bulk grid: cfg4 43 vs 86 us).
    static const int long_mode = [] {
        const char* e = getenv("SELLB_LONG_MODE");
        return e ? atoi(e) : 2;
    }();
    if (n_long && long_mode != 0 && m->n_groups) {
        sellb_mat* mm = const_cast<sellb_mat*>(m);
        std::unique_lock<std::mutex> lk(mm->long_mu, std::defer_lock);
        cudaStream_t ls = st;
        if (long_mode == 2) {
            lk.lock();
            if (!mm->long_ready) {
                int prio_lo = 0, prio_hi = 0;
                SELLB_CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
                SELLB_CU(cudaStreamCreateWithPriority(&mm->s_long, cudaStreamNonBlocking,
                                                      prio_hi));
                SELLB_CU(cudaEventCreateWithFlags(&mm->ev_fork, cudaEventDisableTiming));
                SELLB_CU(cudaEventCreateWithFlags(&mm->ev_join, cudaEventDisableTiming));
                mm->long_ready = true;
            }
            SELLB_CU(cudaEventRecord(mm->ev_fork, st));
            SELLB_CU(cudaStreamWaitEvent(mm->s_long, mm->ev_fork, 0));
            ls = mm->s_long;
        }
        {
            constexpr size_t smem_ = grp_smem<T, 4, 64>();
            static unsigned attr_ = 0;      // per-device bit
            int dev_ = 0;
            cudaGetDevice(&dev_);
            if (!(attr_ & (1u << (dev_ & 31)))) {
                cudaFuncSetAttribute(k_spmv_long_grp<T, ACC, ORD, 4, 2, 64>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_);
                attr_ |= 1u << (dev_ & 31);
            }
            // waves of at most grp_ctas CTAs (longest groups first): the
            // shared-memory carve-out stays off most SMs, and the bulk next to
            // it relies on L1 hits for x (cfg3 sigma=N lost a third of its
            // speed with a group CTA on every SM).  SELLB_GRP_CTAS caps a wave.
            static const int grp_ctas = [] {
                const char* e = getenv("SELLB_GRP_CTAS");
                return e ? std::max(1, atoi(e)) : 1 << 30;
            }();
            for (int64_t g_ = 0; g_ < m->n_groups; g_ += grp_ctas) {
                const int64_t ng_ = std::min<int64_t>(m->n_groups - g_, grp_ctas);
                k_spmv_long_grp<T, ACC, ORD, 4, 2, 64><<<(unsigned)ng_, kGT, smem_, ls>>>(
                    m->cs, m->cl, m->rl, m->col, (const T*)m->val, (const T*)x, (T*)y, ordp,
                    m->C, p0, p1, m->n_rows, m->long_groups + g_, ng_, m->chunk_th, l2pol);
                count_launches();
            }
        }
        SELLB_CU(cudaGetLastError());
        // the bulk: rows above their chunk's threshold are skipped (LONG
        // template); the other long rows (isolated in chunks of short rows)
        // keep the fused warp-per-row role
        grid = (unsigned)grid_for(rows, bt);
        if (long_mode == 2) SELLB_CU(cudaEventRecord(mm->ev_join, ls));
        const int32_t* rest = m->long_rest;
        const int64_t n_rest = m->n_rest;
        grid += (unsigned)((n_rest + bt / 32 - 1) / (bt / 32));
        const bool side = m->side_off != nullptr;   // side table is indexed like long_rest
        if (u8) SELLB_LAUNCH(8, true, rest, n_rest, m->long_th, side);
        else SELLB_LAUNCH(4, true, rest, n_rest, m->long_th, side);
        if (long_mode == 2) SELLB_CU(cudaStreamWaitEvent(st, mm->ev_join, 0));
    } else if (n_long) {
        // no row groups: long_rest holds every long row (same order), so the
        // side table applies unless the fused warp-per-row role is forced
        const bool side = long_mode != 0 && m->side_off && m->n_rest == n_long;
        const int32_t* lr = side ? m->long_rest : m->long_rows;
        if (u8) SELLB_LAUNCH(8, true, lr, n_long, m->long_th, side);
        else SELLB_LAUNCH(4, true, lr, n_long, m->long_th, side);
    } else if (u_env == 6 ||
               (!u_env && sizeof(T) == 8 && ((m->max_cl > 4 && m->max_cl <= 6) ||
                                             (!SKIP && !u8 && mid_rows)))) {
        // every chunk fits one 6-slot batch (5-point stencils): one round
        // trip; or pad-inclusive rows of 16..24 entries (above)
        SELLB_LAUNCH(6, false, nullptr, 0, 0x7fffffff, false);
    } else {
        if (u8) SELLB_LAUNCH(8, false, nullptr, 0, 0x7fffffff, false);
        else SELLB_LAUNCH(4, false, nullptr, 0, 0x7fffffff, false);
    }
#undef SELLB_LAUNCH
    return 0;
}

template <typename T, int CC, bool SKIP>
int dispatch_acc(const sellb_mat* m, const void* x, void* y, int64_t p0, int64_t p1, int acc,
                 int ord, cudaStream_t st) {
    if (acc) {
        return ord ? dispatch_u<T, CC, SKIP, true, 1>(m, x, y, p0, p1, st, m->order)
                   : dispatch_u<T, CC, SKIP, true, 0>(m, x, y, p0, p1, st, m->order);
    }
    return ord ? dispatch_u<T, CC, SKIP, false, 1>(m, x, y, p0, p1, st, m->order)
               : dispatch_u<T, CC, SKIP, false, 0>(m, x, y, p0, p1, st, m->order);
}

// the whole matrix through its SELL-32 shadow (build_shadow: sigma = N, or
// 512 for x far larger than L2), sums
// scattered through the flagged maps (ORD 2)
template <typename T>
int dispatch_shadow(const sellb_mat* m, const void* x, void* y, int acc, int ord,
                    cudaStream_t st) {
    const sellb_mat* sh = m->shadow;
    const int32_t* o = ord ? m->sh_ord_or : m->sh_ord_st;
    if (sh->variant == SELLB_VARIANT_PAD_SKIP)
        return acc ? dispatch_u<T, 32, true, true, 2>(sh, x, y, 0, sh->n_pad, st, o)
                   : dispatch_u<T, 32, true, false, 2>(sh, x, y, 0, sh->n_pad, st, o);
    return acc ? dispatch_u<T, 32, false, true, 2>(sh, x, y, 0, sh->n_pad, st, o)
               : dispatch_u<T, 32, false, false, 2>(sh, x, y, 0, sh->n_pad, st, o);
}

template <typename T>
int dispatch_sell(const sellb_mat* m, const void* x, void* y, int64_t p0, int64_t p1, int acc,
                  int ord, cudaStream_t st) {
    const bool skip = m->variant == SELLB_VARIANT_PAD_SKIP && m->rl;
    if (skip && m->pcol && m->C == 32) {
        // the packed stored-order copy through the row-run kernel (MODE 1)
        if (acc) return ord ? launch_packed<T, true, 1>(m, x, y, p0, p1, st)
                            : launch_packed<T, true, 0>(m, x, y, p0, p1, st);
        return ord ? launch_packed<T, false, 1>(m, x, y, p0, p1, st)
                   : launch_packed<T, false, 0>(m, x, y, p0, p1, st);
    }
    if (m->C == 32) {
        return skip ? dispatch_acc<T, 32, true>(m, x, y, p0, p1, acc, ord, st)
                    : dispatch_acc<T, 32, false>(m, x, y, p0, p1, acc, ord, st);
    }
    return skip ? dispatch_acc<T, 0, true>(m, x, y, p0, p1, acc, ord, st)
                : dispatch_acc<T, 0, false>(m, x, y, p0, p1, acc, ord, st);
}

}  // namespace

namespace sellb {

int launch_spmv(const sellb_mat* m, const void* x, void* y, int64_t c0, int64_t c1,
                int accumulate, int out_order, cudaStream_t st) {
    if (c0 < 0 || c1 > m->n_chunks || c0 > c1)
        return set_error(SELLB_EPARAM, "chunk range [%lld, %lld) outside [0, %lld)",
                         (long long)c0, (long long)c1, (long long)m->n_chunks);
    if (out_order == SELLB_ORDER_ORIGINAL && !m->order)
        return set_error(SELLB_EPARAM, "original-order output needs the row permutation");
    if (c0 == c1) return 0;
    if (m->shadow && c0 == 0 && c1 == m->n_chunks) {
        const int ord = out_order == SELLB_ORDER_ORIGINAL;
        int rc = m->dtype == SELLB_F32 ? dispatch_shadow<float>(m, x, y, accumulate, ord, st)
                                       : dispatch_shadow<double>(m, x, y, accumulate, ord, st);
        if (rc) return rc;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
            return set_error(SELLB_ERESOURCE, "spmv launch failed: %s", cudaGetErrorString(e));
        return 0;
    }
    // TMA bulk-copy path (sellb_tma.cu) for C = 32 pad-inclusive layouts:
    // default for fp32 (cfg2: 1503 vs 1472 GF/s), slower for fp64 (914 vs
    // ~1030: too few consumer warps hide the gather latency).  SELLB_TMA=0/1
    // forces it off/on.
    static const int tma_env = [] {
        const char* e = getenv("SELLB_TMA");
        return e ? atoi(e) : -1;
    }();
    const bool tma = tma_env >= 0 ? tma_env == 1 : m->dtype == SELLB_F32;
    if (tma && m->C == 32 && m->variant == SELLB_VARIANT_PAD_INCL &&
        out_order == SELLB_ORDER_STORED && !m->n_long) {
        sellb_mat* mm = const_cast<sellb_mat*>(m);
        if ((int64_t)mm->h_cs.size() != m->n_chunks + 1) {
            std::lock_guard<std::mutex> lk(mm->hcs_mu);
            if ((int64_t)mm->h_cs.size() != m->n_chunks + 1) {
                std::vector<int64_t> h(m->n_chunks + 1);
                SELLB_CU(cudaMemcpy(h.data(), m->cs, h.size() * 8, cudaMemcpyDeviceToHost));
                mm->h_cs.swap(h);
            }
        }
        if (launch_spmv_tma(m, x, y, c0, c1, accumulate, st, mm->h_cs.data())) {
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess)
                return set_error(SELLB_ERESOURCE, "tma spmv launch failed: %s",
                                 cudaGetErrorString(e));
            return 0;
        }
    }
    int rc = m->dtype == SELLB_F32
                 ? dispatch_sell<float>(m, x, y, c0 * m->C, c1 * m->C, accumulate, out_order, st)
                 : dispatch_sell<double>(m, x, y, c0 * m->C, c1 * m->C, accumulate, out_order, st);
    if (rc) return rc;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SELLB_ERESOURCE, "spmv launch failed: %s", cudaGetErrorString(e));
    return 0;
}

int launch_spmv_list(const sellb_mat* m, const int32_t* ids, int64_t n_ids, const void* x,
                     void* y, int accumulate, cudaStream_t st) {
    if (n_ids <= 0) return 0;
    const bool skip = m->variant == SELLB_VARIANT_PAD_SKIP && m->rl;
    const unsigned grid = (unsigned)grid_for(n_ids * m->C, kThreads);
#define SELLB_LIST(T, S, A)                                                                   \
    k_spmv_sell_list<T, S, A><<<grid, kThreads, 0, st>>>(m->cs, m->cl, m->rl, m->col,         \
                                                         (const T*)m->val, (const T*)x,      \
                                                         (T*)y, ids, n_ids, m->C)
    if (m->dtype == SELLB_F32) {
        if (skip) { if (accumulate) SELLB_LIST(float, true, true); else SELLB_LIST(float, true, false); }
        else { if (accumulate) SELLB_LIST(float, false, true); else SELLB_LIST(float, false, false); }
    } else {
        if (skip) { if (accumulate) SELLB_LIST(double, true, true); else SELLB_LIST(double, true, false); }
        else { if (accumulate) SELLB_LIST(double, false, true); else SELLB_LIST(double, false, false); }
    }
    count_launches();
#undef SELLB_LIST
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SELLB_ERESOURCE, "spmv launch failed: %s", cudaGetErrorString(e));
    return 0;
}

int launch_spmv_crs(const int64_t* rpt, const int32_t* col, const void* val, int32_t dtype,
                    const void* x, void* y, int64_t r0, int64_t r1, int accumulate, int unrolled,
                    cudaStream_t st) {
    if (r1 <= r0) return 0;
    // SELLB_CRS_SCALAR=1: the one-thread-per-row kernels (A/B reference)
    static const bool scalar = getenv("SELLB_CRS_SCALAR") && atoi(getenv("SELLB_CRS_SCALAR"));
    if (!scalar) {
#define SELLB_CRST(T, A, UN)                                                                  \
    launch_rows<T, A, UN, 0, 0>(rpt, col, val, x, y, r0, r1, nullptr, nullptr, nullptr, 0, st)
        if (dtype == SELLB_F32) {
            if (unrolled) { if (accumulate) SELLB_CRST(float, true, true); else SELLB_CRST(float, false, true); }
            else { if (accumulate) SELLB_CRST(float, true, false); else SELLB_CRST(float, false, false); }
        } else {
            if (unrolled) { if (accumulate) SELLB_CRST(double, true, true); else SELLB_CRST(double, false, true); }
            else { if (accumulate) SELLB_CRST(double, true, false); else SELLB_CRST(double, false, false); }
        }
#undef SELLB_CRST
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
            return set_error(SELLB_ERESOURCE, "crs launch failed: %s", cudaGetErrorString(e));
        return 0;
    }
    const unsigned grid = (unsigned)grid_for(r1 - r0, kThreads);
#define SELLB_CRS(K, T, A) K<T, A><<<grid, kThreads, 0, st>>>(rpt, col, (const T*)val, (const T*)x, (T*)y, r0, r1)
    if (dtype == SELLB_F32) {
        if (unrolled) { if (accumulate) SELLB_CRS(k_spmv_crs_unrolled, float, true); else SELLB_CRS(k_spmv_crs_unrolled, float, false); }
        else { if (accumulate) SELLB_CRS(k_spmv_crs, float, true); else SELLB_CRS(k_spmv_crs, float, false); }
    } else {
        if (unrolled) { if (accumulate) SELLB_CRS(k_spmv_crs_unrolled, double, true); else SELLB_CRS(k_spmv_crs_unrolled, double, false); }
        else { if (accumulate) SELLB_CRS(k_spmv_crs, double, true); else SELLB_CRS(k_spmv_crs, double, false); }
    }
#undef SELLB_CRS
    count_launches();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SELLB_ERESOURCE, "crs launch failed: %s", cudaGetErrorString(e));
    return 0;
}

}  // namespace sellb

// ===========================================================================
// ABI
// ===========================================================================
extern "C" {

int sellb_spmv(const sellb_mat* m, const void* x, void* y, int64_t c0, int64_t c1,
               int32_t accumulate, int32_t out_order, void* stream) {
    clear_error();
    NvtxRange nvtx_("sellb_spmv");
    if (!m || (!x && m->slots) || !y) return set_error(SELLB_EPARAM, "NULL argument");
    DeviceGuard guard(m->device);
    return launch_spmv(m, x, y, c0, c1, accumulate, out_order, (cudaStream_t)stream);
}

int sellb_spmv_chunk_list(const sellb_mat* m, const int32_t* chunk_ids, int64_t n_ids,
                          const void* x, void* y, int32_t accumulate, void* stream) {
    clear_error();
    if (!m || !y || (n_ids && !chunk_ids)) return set_error(SELLB_EPARAM, "NULL argument");
    DeviceGuard guard(m->device);
    return launch_spmv_list(m, chunk_ids, n_ids, x, y, accumulate, (cudaStream_t)stream);
}

int sellb_chunk_flags(const sellb_mat* m, const uint8_t* row_flag, uint8_t* chunk_flag,
                      void* stream) {
    clear_error();
    if (!m || !row_flag || !chunk_flag) return set_error(SELLB_EPARAM, "NULL argument");
    if (!m->order && m->n_rows) return set_error(SELLB_EPARAM, "matrix has no permutation");
    if (m->n_chunks == 0) return 0;
    DeviceGuard guard(m->device);
    k_chunk_flags<<<(unsigned)grid_for(m->n_chunks * 32, kThreads), kThreads, 0,
                    (cudaStream_t)stream>>>(m->order, m->n_rows, m->n_chunks, m->C, row_flag,
                                            chunk_flag);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SELLB_ERESOURCE, "chunk-flag launch failed: %s", cudaGetErrorString(e));
    return 0;
}

int sellb_pad_fixup(const sellb_mat* m, const void* x0, void* y, void* stream) {
    clear_error();
    if (!m || !x0 || !y) return set_error(SELLB_EPARAM, "NULL argument");
    if (!m->rl) return set_error(SELLB_EPARAM, "pad fix-up needs row_lengths");
    if (m->n_pad == 0) return 0;
    DeviceGuard guard(m->device);
    const unsigned grid = (unsigned)grid_for(m->n_pad, kThreads);
    cudaStream_t st = (cudaStream_t)stream;
    if (m->dtype == SELLB_F32)
        k_pad_fixup<float><<<grid, kThreads, 0, st>>>(m->cl, m->rl, m->C, m->n_pad,
                                                     (const float*)x0, (float*)y);
    else
        k_pad_fixup<double><<<grid, kThreads, 0, st>>>(m->cl, m->rl, m->C, m->n_pad,
                                                      (const double*)x0, (double*)y);
    count_launches();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(SELLB_ERESOURCE, "fix-up launch failed: %s", cudaGetErrorString(e));
    return 0;
}

}  // extern "C"

namespace {

// per-chunk maximum column index (real slots and padding alike; padding
// holds column 0 so it never raises the maximum)
__global__ void k_chunk_maxcol(const int64_t* __restrict__ cs, const int32_t* __restrict__ col,
                               int64_t n_chunks, int32_t* __restrict__ out) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n_chunks) return;
    int32_t mx = 0;
    for (int64_t k = cs[w] + lane; k < cs[w + 1]; k += 32) mx = max(mx, col[k]);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) out[w] = mx;
}

// One-time setup of the pipelined host path: row blocks of equal chunk
// count, x pieces of equal column count, and for every row block the last x
// piece its columns reach (so its kernel can start as soon as that piece has
// landed).
int pipe_setup(sellb_mat* m) {
    if (m->pipe_ready) return 0;
    // cfg5: depth 4 / 8 / 16 -> pinned 13.9 / 13.0 / 12.6 ms per step (y by DMA),
    // pageable staged 28.0 / 25.9 ms (depth 4 / 8); cfg2 is flat from 4 up
    int want = 16;
    if (const char* e = getenv("SELLB_PIPE")) want = std::max(1, std::min(atoi(e), sellb_mat::kPipe));
    const int P = (int)std::min<int64_t>(want, std::max<int64_t>(m->n_chunks, 1));
    std::vector<int32_t> maxcol(std::max<int64_t>(m->n_chunks, 1), 0);
    if (m->n_chunks) {
        int32_t* d = nullptr;
        SELLB_CU(cudaMalloc(&d, m->n_chunks * 4));
        k_chunk_maxcol<<<(unsigned)grid_for(m->n_chunks * 32, kThreads), kThreads>>>(
            m->cs, m->col, m->n_chunks, d);
        cudaError_t e = cudaMemcpy(maxcol.data(), d, m->n_chunks * 4, cudaMemcpyDeviceToHost);
        cudaFree(d);
        SELLB_CU(e);
    }
    // x piece b ends just past the highest column row block b reads, so block
    // b can start as soon as piece b has landed (for banded matrices the
    // pieces then track the row blocks and H2D, compute and D2H overlap)
    // Equal row blocks (geometrically growing ones measured slower on cfg2,
    // 0.546 vs 0.499 ms: with both PCIe directions busy each runs at ~40
    // GB/s, and the y drain of a block is as long as the next block's x
    // transfer anyway).
    m->n_pieces = P;
    m->x_off[0] = 0;
    m->blk_c[0] = 0;
    for (int b = 0; b < P; ++b) {
        m->blk_c[b + 1] = m->n_chunks * (b + 1) / P;
        int64_t mx = -1;
        for (int64_t c = m->blk_c[b]; c < m->blk_c[b + 1]; ++c) mx = std::max<int64_t>(mx, maxcol[c]);
        int64_t end = std::min<int64_t>(std::max<int64_t>(m->x_off[b], mx + 1), m->n_cols);
        m->x_off[b + 1] = (b + 1 == P) ? m->n_cols : end;
        m->blk_need[b] = b;
    }
    SELLB_CU(cudaStreamCreateWithFlags(&m->s_h2d, cudaStreamNonBlocking));
    SELLB_CU(cudaStreamCreateWithFlags(&m->s_comp, cudaStreamNonBlocking));
    SELLB_CU(cudaStreamCreateWithFlags(&m->s_d2h, cudaStreamNonBlocking));
    const unsigned evf = getenv("SELLB_PIPE_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
    SELLB_CU(cudaEventCreateWithFlags(&m->ev_start, evf));
    for (int i = 0; i < sellb_mat::kPipe; ++i) {
        SELLB_CU(cudaEventCreateWithFlags(&m->ev_x[i], evf));
        SELLB_CU(cudaEventCreateWithFlags(&m->ev_blk[i], evf));
    }
    m->pipe_ready = true;
    return 0;
}

// y = A x with host x / y: x streams in column pieces on one copy engine,
// row blocks start as soon as the x they read has landed, and each block's
// y streams back while later blocks compute.
//
// Pinned caller buffers: DMA straight from x_host; the kernels store y
// straight into the mapped y_host (no D2H pass).  Pageable caller buffers
// (ordinary NumPy arrays, the reference's call, spmv.py:105-122): x piece i
// is copied by the host thread pool into the pinned mirror hx while piece
// i-1 is on the wire; the kernels store y into the mapped mirror hy and
// every finished row block is copied out by the pool while later blocks
// compute.  Either way every byte crosses PCIe once, at pinned speed.
int spmv_host_pipelined(sellb_mat* m, const void* x_host, void* y_host, cudaStream_t user) {
    if (int rc = pipe_setup(m)) return rc;
    const size_t vs = vsize(m->dtype);
    const int P = m->n_pieces;
    const bool x_pinned = is_pinned(x_host);
    const bool y_pinned = is_pinned(y_host);
    // y of a pinned caller buffer goes back by DMA per row block (cfg5, depth
    // 16: 12.6 ms vs 13.2 ms with the kernels storing over PCIe); a pageable
    // y is stored by the kernels straight into the mapped mirror (one PCIe
    // crossing, no pageable D2H copy: 27 ms vs 128 ms per step)
    static const bool no_zc = getenv("SELLB_NO_ZEROCOPY") != nullptr;
    const bool zero_copy = !no_zc && !y_pinned;
    if (!x_pinned) {
        if (int rc = ensure_host_mirror(&m->hx, (size_t)m->n_cols * vs)) return rc;
    }
    if (!y_pinned && zero_copy) {
        if (int rc = ensure_host_mirror(&m->hy, (size_t)m->n_pad * vs)) return rc;
    }
    // where the kernels write y: the caller's pinned buffer or our mirror
    // (mapped; device pointer from the runtime), else y_buf + D2H copies
    void* y_dev_view = nullptr;
    if (zero_copy) {
        void* host_y = y_pinned ? y_host : m->hy;
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, host_y) == cudaSuccess && at.devicePointer)
            y_dev_view = at.devicePointer;
        cudaGetLastError();
    }
    const char* xsrc = x_pinned ? (const char*)x_host : (const char*)m->hx;
    SELLB_CU(cudaEventRecord(m->ev_start, user));
    SELLB_CU(cudaStreamWaitEvent(m->s_h2d, m->ev_start, 0));
    SELLB_CU(cudaStreamWaitEvent(m->s_comp, m->ev_start, 0));
    // x piece i, then every row block whose last needed piece is i
    int waited = -1;
    int next_blk = 0;
    for (int i = 0; i < P; ++i) {
        const int64_t a = m->x_off[i], b = m->x_off[i + 1];
        if (b > a) {
            if (!x_pinned)
                host_parallel_copy((char*)m->hx + a * vs, (const char*)x_host + a * vs,
                                   (b - a) * vs);
            SELLB_CU(cudaMemcpyAsync((char*)m->x_buf + a * vs, xsrc + a * vs, (b - a) * vs,
                                     cudaMemcpyHostToDevice, m->s_h2d));
        }
        SELLB_CU(cudaEventRecord(m->ev_x[i], m->s_h2d));
        for (; next_blk < P && m->blk_need[next_blk] <= i; ++next_blk) {
            const int bk = next_blk;
            if (m->blk_need[bk] > waited) {
                SELLB_CU(cudaStreamWaitEvent(m->s_comp, m->ev_x[m->blk_need[bk]], 0));
                waited = m->blk_need[bk];
            }
            if (int rc = launch_spmv(m, m->x_buf, y_dev_view ? y_dev_view : m->y_buf,
                                     m->blk_c[bk], m->blk_c[bk + 1], 0, SELLB_ORDER_STORED,
                                     m->s_comp))
                return rc;
            SELLB_CU(cudaEventRecord(m->ev_blk[bk], m->s_comp));
            if (y_dev_view) continue;
            SELLB_CU(cudaStreamWaitEvent(m->s_d2h, m->ev_blk[bk], 0));
            const int64_t y0 = m->blk_c[bk] * m->C, y1 = m->blk_c[bk + 1] * m->C;
            if (y1 > y0)
                SELLB_CU(cudaMemcpyAsync((char*)y_host + y0 * vs,
                                         (const char*)m->y_buf + y0 * vs, (y1 - y0) * vs,
                                         cudaMemcpyDeviceToHost, m->s_d2h));
        }
    }
    if (y_dev_view && !y_pinned) {
        // copy each finished row block out of the mirror while later ones run
        for (int bk = 0; bk < P; ++bk) {
            SELLB_CU(cudaEventSynchronize(m->ev_blk[bk]));
            const int64_t y0 = m->blk_c[bk] * m->C, y1 = m->blk_c[bk + 1] * m->C;
            if (y1 > y0)
                host_parallel_copy((char*)y_host + y0 * vs, (const char*)m->hy + y0 * vs,
                                   (y1 - y0) * vs);
        }
    }
    SELLB_CU(cudaStreamSynchronize(y_dev_view ? m->s_comp : m->s_d2h));
    SELLB_CU(cudaStreamSynchronize(m->s_h2d));
    if (getenv("SELLB_PIPE_TRACE")) {        // debug timeline (events carry timing)
        float t;
        fprintf(stderr, "pipe x:");
        for (int i = 0; i < P; ++i) {
            cudaEventElapsedTime(&t, m->ev_start, m->ev_x[i]);
            fprintf(stderr, " %.3f", t);
        }
        fprintf(stderr, "\npipe k:");
        for (int i = 0; i < P; ++i) {
            cudaEventElapsedTime(&t, m->ev_start, m->ev_blk[i]);
            fprintf(stderr, " %.3f", t);
        }
        fprintf(stderr, "\n");
    }
    return 0;
}

}  // namespace

extern "C" {

int sellb_spmv_host(sellb_mat* m, const void* x_host, void* y_host, int64_t c0, int64_t c1,
                    int32_t accumulate, int32_t out_order, void* stream) {
    clear_error();
    NvtxRange nvtx_("sellb_spmv_host");
    if (!m || !y_host || (!x_host && m->n_cols)) return set_error(SELLB_EPARAM, "NULL argument");
    if (c0 < 0 || c1 > m->n_chunks || c0 > c1)
        return set_error(SELLB_EPARAM, "chunk range outside the matrix");
    DeviceGuard guard(m->device);
    std::lock_guard<std::mutex> lk(m->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t vs = vsize(m->dtype);
    const int64_t ny = out_order == SELLB_ORDER_ORIGINAL ? m->n_rows : m->n_pad;
    if (!m->x_buf) SELLB_CU(cudaMalloc(&m->x_buf, std::max<int64_t>(m->n_cols, 1) * vs));
    if (!m->y_buf) SELLB_CU(cudaMalloc(&m->y_buf, std::max<int64_t>(m->n_pad, 1) * vs));
    if (!accumulate && out_order == SELLB_ORDER_STORED && c0 == 0 && c1 == m->n_chunks &&
        m->n_chunks >= 4 * sellb_mat::kPipe && !getenv("SELLB_NO_PIPELINE"))
        return spmv_host_pipelined(m, x_host, y_host, st);
    if (m->n_cols)
        SELLB_CU(cudaMemcpyAsync(m->x_buf, x_host, m->n_cols * vs, cudaMemcpyHostToDevice, st));
    // rows touched by the range
    int64_t y0 = c0 * m->C, y1 = c1 * m->C;
    if (out_order == SELLB_ORDER_ORIGINAL) { y0 = 0; y1 = ny; }
    if (accumulate && y1 > y0)
        SELLB_CU(cudaMemcpyAsync((char*)m->y_buf + y0 * vs, (const char*)y_host + y0 * vs,
                                 (y1 - y0) * vs, cudaMemcpyHostToDevice, st));
    if (out_order == SELLB_ORDER_ORIGINAL && !accumulate && (c0 != 0 || c1 != m->n_chunks)) {
        // rows outside the range keep the caller's values
        SELLB_CU(cudaMemcpyAsync(m->y_buf, y_host, ny * vs, cudaMemcpyHostToDevice, st));
    }
    if (int rc = launch_spmv(m, m->x_buf, m->y_buf, c0, c1, accumulate, out_order, st)) return rc;
    if (y1 > y0)
        SELLB_CU(cudaMemcpyAsync((char*)y_host + y0 * vs, (const char*)m->y_buf + y0 * vs,
                                 (y1 - y0) * vs, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    return 0;
}

int sellb_spmv_sell_range_host(const int64_t* cs, const int32_t* cl, int32_t C,
                               const int32_t* col, const double* val, int64_t n_slots,
                               int64_t n_chunks, const double* x, int64_t n_x, double* y,
                               int64_t n_y, int64_t c0, int64_t c1, int32_t accumulate,
                               int32_t device) {
    clear_error();
    if (C < 1) return set_error(SELLB_EPARAM, "chunk height C must be >= 1");
    if (c0 < 0 || c1 > n_chunks || c0 > c1) return set_error(SELLB_EPARAM, "bad chunk range");
    if (n_y < n_chunks * (int64_t)C) return set_error(SELLB_EDIM, "y shorter than n_chunks*C");
    if (c0 == c1) return 0;
    if (cs[n_chunks] != n_slots) return set_error(SELLB_ESTRUCT, "cs[n_chunks] != len(val)");
    sellb_mat* m = nullptr;
    int rc = sellb_import(cs, cl, col, val, nullptr, nullptr, SELLB_F64, n_chunks * C, n_x, C, 1,
                          n_chunks, n_slots, 0, device, nullptr, 0, &m);
    if (rc) return rc;
    rc = sellb_spmv_host(m, x, y, c0, c1, accumulate, SELLB_ORDER_STORED, nullptr);
    sellb_free(m);
    return rc;
}

int sellb_spmv_crs(const int64_t* rpt, const int32_t* col, const void* val, int32_t dtype,
                   const void* x, void* y, int64_t r0, int64_t r1, int32_t accumulate,
                   int32_t unrolled, void* stream) {
    clear_error();
    if (!rpt || !y) return set_error(SELLB_EPARAM, "NULL argument");
    return launch_spmv_crs(rpt, col, val, dtype, x, y, r0, r1, accumulate, unrolled,
                           (cudaStream_t)stream);
}

int sellb_spmv_crs_range_host(const int64_t* rpt, int64_t n_rows, const int32_t* col,
                              const double* val, int64_t nnz, const double* x, int64_t n_x,
                              double* y, int64_t r0, int64_t r1, int32_t accumulate,
                              int32_t unrolled, int32_t device) {
    clear_error();
    if (r0 < 0 || r1 > n_rows || r0 > r1) return set_error(SELLB_EPARAM, "bad row range");
    if (r0 == r1) return 0;
    DeviceGuard guard(device);
    if (!guard.ok) return set_error(SELLB_ERESOURCE, "cannot select CUDA device %d", device);
    cudaStream_t st = 0;
    DBuf d_rpt, d_col, d_val, d_x, d_y;
    SELLB_CU(d_rpt.alloc((n_rows + 1) * 8, st));
    SELLB_CU(d_col.alloc(nnz * 4, st));
    SELLB_CU(d_val.alloc(nnz * 8, st));
    SELLB_CU(d_x.alloc(n_x * 8, st));
    SELLB_CU(d_y.alloc(n_rows * 8, st));
    SELLB_CU(cudaMemcpyAsync(d_rpt.p, rpt, (n_rows + 1) * 8, cudaMemcpyHostToDevice, st));
    if (nnz) {
        SELLB_CU(cudaMemcpyAsync(d_col.p, col, nnz * 4, cudaMemcpyHostToDevice, st));
        SELLB_CU(cudaMemcpyAsync(d_val.p, val, nnz * 8, cudaMemcpyHostToDevice, st));
    }
    if (n_x) SELLB_CU(cudaMemcpyAsync(d_x.p, x, n_x * 8, cudaMemcpyHostToDevice, st));
    if (accumulate)
        SELLB_CU(cudaMemcpyAsync(d_y.as<double>() + r0, y + r0, (r1 - r0) * 8,
                                 cudaMemcpyHostToDevice, st));
    if (int rc = launch_spmv_crs(d_rpt.as<int64_t>(), d_col.as<int32_t>(), d_val.p, SELLB_F64,
                                 d_x.p, d_y.p, r0, r1, accumulate, unrolled, st))
        return rc;
    SELLB_CU(cudaMemcpyAsync(y + r0, d_y.as<double>() + r0, (r1 - r0) * 8,
                             cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    return 0;
}

}  // extern "C"
