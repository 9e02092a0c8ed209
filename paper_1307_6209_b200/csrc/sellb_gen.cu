// sellb_gen.cu -- row-addressable generator of the cfg5 banded-random
// "Hamiltonian" matrix directly in device memory (BASELINE.json configs[4]:
// N = 2^26, ~1.3e9 nonzeros, 16 GB of CRS that never crosses PCIe).
//
// Entry (i, i+d) for d in the sorted offset set exists iff d == 0 or
// u(seed, i, d) < keep, with u = (splitmix64(key) >> 11) * 2^-53 and
// key = i * 0x100000001B3 ^ (d + seed) (64-bit wrap-around); its value is
// (splitmix64(h ^ 0xD1B54A32D192ED03) >> 11) * 2^-52 - 1, exact in fp64.
// Bit-identical to the NumPy definition in
// paper_1307_6209_b200/generate.py:hamiltonian_rows (checked by
// tests/test_gpu_parity.py::test_cfg5_generator_matches_numpy).
#include <cub/cub.cuh>

#include "sellb_internal.cuh"

using namespace sellb;

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ bool keep_entry(int64_t i, int64_t d, int64_t col, int64_t n,
                                           double keep, uint64_t seed, uint64_t* h_out) {
    const uint64_t key = ((uint64_t)i * 0x100000001B3ull) ^ ((uint64_t)d + seed);
    const uint64_t h = splitmix64(key);
    *h_out = h;
    if (col < 0 || col >= n) return false;
    if (d == 0) return true;
    const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    return u < keep;
}

__global__ void k_ham_count(int64_t n, int64_t r0, int64_t r1, const int64_t* __restrict__ offs,
                            int n_off, double keep, uint64_t seed, int64_t* __restrict__ counts) {
    const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    int64_t c = 0;
    uint64_t h;
    for (int k = 0; k < n_off; ++k) c += keep_entry(r, offs[k], r + offs[k], n, keep, seed, &h);
    counts[r - r0] = c;
}

template <typename T>
__global__ void k_ham_fill(int64_t n, int64_t r0, int64_t r1, const int64_t* __restrict__ offs,
                           int n_off, double keep, uint64_t seed,
                           const int64_t* __restrict__ rpt, int32_t* __restrict__ col,
                           T* __restrict__ val) {
    const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    int64_t k0 = rpt[r - r0];
    uint64_t h;
    for (int k = 0; k < n_off; ++k) {
        const int64_t c = r + offs[k];
        if (!keep_entry(r, offs[k], c, n, keep, seed, &h)) continue;
        const uint64_t vh = splitmix64(h ^ 0xD1B54A32D192ED03ull);
        const double v = (double)(vh >> 11) * (2.0 / 9007199254740992.0) - 1.0;
        col[k0] = (int32_t)c;
        val[k0] = (T)v;
        ++k0;
    }
}

// cfg3 power-law generator (BASELINE configs[2]), row-addressable like the
// one above; bit-identical to generate.py:powerlaw_rows.  Row i:
//   u    = (splitmix64(i ^ (seed * 0xA24BAED4963EE407)) >> 11) * 2^-53
//   len  = clip(floor(base / sqrt(1 - u)), 1, min(lmax, n))
//          (the inverse CDF of base * (1 + Pareto(2)): mean ~2 base, zeta ~2)
//   h    = splitmix64(i ^ seed);  start = clip(i + h % (2 band + 1) - band,
//          0, n - len); columns start .. start + len - 1
//   value of entry k: (splitmix64((i * 0x100000001B3) ^ (k + seed + 0x5851F42D4C957F2D))
//          >> 11) * 2^-52 - 1
// 1 - u is exact, sqrt and the division are correctly rounded in IEEE
// double on both sides (__dsqrt_rn / __ddiv_rn here, NumPy there).
__device__ __forceinline__ int64_t pl_len(int64_t i, int64_t n, double base, int64_t lmax,
                                          uint64_t seed) {
    const uint64_t hu = splitmix64((uint64_t)i ^ (seed * 0xA24BAED4963EE407ull));
    const double u = (double)(hu >> 11) * (1.0 / 9007199254740992.0);
    const double q = __ddiv_rn(base, __dsqrt_rn(1.0 - u));
    int64_t len = (int64_t)floor(q);
    const int64_t cap = lmax < n ? lmax : n;
    if (len < 1) len = 1;
    if (len > cap) len = cap;
    return len;
}

__global__ void k_pl_count(int64_t n, int64_t r0, int64_t r1, double base, int64_t lmax,
                           uint64_t seed, int64_t* __restrict__ counts) {
    const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r1) return;
    counts[r - r0] = pl_len(r, n, base, lmax, seed);
}

template <typename T>
__global__ void k_pl_fill(int64_t n, int64_t r0, int64_t r1, double base, int64_t lmax,
                          int64_t band, uint64_t seed, const int64_t* __restrict__ rpt,
                          int32_t* __restrict__ col, T* __restrict__ val) {
    // one warp per row: lanes over the row's entries (coalesced stores)
    const int64_t r = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= r1) return;
    const int64_t len = pl_len(r, n, base, lmax, seed);
    const uint64_t h = splitmix64((uint64_t)r ^ seed);
    int64_t start = r + (int64_t)(h % (uint64_t)(2 * band + 1)) - band;
    if (start > n - len) start = n - len;
    if (start < 0) start = 0;
    const int64_t k0 = rpt[r - r0];
    const uint64_t rk = (uint64_t)r * 0x100000001B3ull;
    for (int64_t k = lane; k < len; k += 32) {
        const uint64_t vh = splitmix64(rk ^ ((uint64_t)k + seed + 0x5851F42D4C957F2Dull));
        col[k0 + k] = (int32_t)(start + k);
        val[k0 + k] = (T)((double)(vh >> 11) * (2.0 / 9007199254740992.0) - 1.0);
    }
}

}  // namespace

extern "C" {

int sellb_gen_powerlaw_rpt(int64_t n, int64_t r0, int64_t r1, double base, int64_t lmax,
                           uint64_t seed, int64_t* rpt_dev, int64_t* nnz_out, void* stream) {
    clear_error();
    if (n < 0 || r0 < 0 || r1 < r0 || r1 > n || base <= 0.0 || lmax < 1)
        return set_error(SELLB_EPARAM, "bad generator parameters");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = r1 - r0;
    SELLB_CU(cudaMemsetAsync(rpt_dev, 0, 8, st));
    if (rows) {
        DBuf cnt, tmp;
        SELLB_CU(cnt.alloc(rows * 8, st));
        k_pl_count<<<(unsigned)grid_for(rows, 256), 256, 0, st>>>(n, r0, r1, base, lmax, seed,
                                                                  cnt.as<int64_t>());
        SELLB_CU(cudaGetLastError());
        size_t tb = 0;
        SELLB_CU(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.as<int64_t>(), rpt_dev + 1,
                                               (int64_t)rows, st));
        SELLB_CU(tmp.alloc(tb, st));
        SELLB_CU(cub::DeviceScan::InclusiveSum(tmp.p, tb, cnt.as<int64_t>(), rpt_dev + 1,
                                               (int64_t)rows, st));
    }
    int64_t nnz = 0;
    SELLB_CU(cudaMemcpyAsync(&nnz, rpt_dev + rows, 8, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    if (nnz_out) *nnz_out = nnz;
    return 0;
}

int sellb_gen_powerlaw_fill(int64_t n, int64_t r0, int64_t r1, double base, int64_t lmax,
                            int64_t band, uint64_t seed, const int64_t* rpt_dev, int32_t* col_dev,
                            void* val_dev, int32_t dtype, void* stream) {
    clear_error();
    if (n < 0 || r0 < 0 || r1 < r0 || r1 > n || band < 0)
        return set_error(SELLB_EPARAM, "bad generator parameters");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = r1 - r0;
    if (!rows) return 0;
    const unsigned grid = (unsigned)grid_for(rows * 32, 256);
    if (dtype == SELLB_F32)
        k_pl_fill<float><<<grid, 256, 0, st>>>(n, r0, r1, base, lmax, band, seed, rpt_dev,
                                               col_dev, (float*)val_dev);
    else
        k_pl_fill<double><<<grid, 256, 0, st>>>(n, r0, r1, base, lmax, band, seed, rpt_dev,
                                                col_dev, (double*)val_dev);
    SELLB_CU(cudaGetLastError());
    return 0;
}

int sellb_gen_hamiltonian_rpt(int64_t n, int64_t r0, int64_t r1, const int64_t* offs_dev,
                              int32_t n_off, double keep, uint64_t seed, int64_t* rpt_dev,
                              int64_t* nnz_out, void* stream) {
    clear_error();
    if (n < 0 || r0 < 0 || r1 < r0 || r1 > n || n_off < 0)
        return set_error(SELLB_EPARAM, "bad generator range");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = r1 - r0;
    SELLB_CU(cudaMemsetAsync(rpt_dev, 0, 8, st));
    if (rows) {
        DBuf cnt, tmp;
        SELLB_CU(cnt.alloc(rows * 8, st));
        k_ham_count<<<(unsigned)grid_for(rows, 256), 256, 0, st>>>(
            n, r0, r1, offs_dev, n_off, keep, seed, cnt.as<int64_t>());
        SELLB_CU(cudaGetLastError());
        size_t tb = 0;
        SELLB_CU(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.as<int64_t>(), rpt_dev + 1,
                                               (int64_t)rows, st));
        SELLB_CU(tmp.alloc(tb, st));
        SELLB_CU(cub::DeviceScan::InclusiveSum(tmp.p, tb, cnt.as<int64_t>(), rpt_dev + 1,
                                               (int64_t)rows, st));
    }
    int64_t nnz = 0;
    SELLB_CU(cudaMemcpyAsync(&nnz, rpt_dev + rows, 8, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    if (nnz_out) *nnz_out = nnz;
    return 0;
}

int sellb_gen_hamiltonian_fill(int64_t n, int64_t r0, int64_t r1, const int64_t* offs_dev,
                               int32_t n_off, double keep, uint64_t seed, const int64_t* rpt_dev,
                               int32_t* col_dev, void* val_dev, int32_t dtype, void* stream) {
    clear_error();
    if (n < 0 || r0 < 0 || r1 < r0 || r1 > n) return set_error(SELLB_EPARAM, "bad range");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = r1 - r0;
    if (!rows) return 0;
    if (dtype == SELLB_F32)
        k_ham_fill<float><<<(unsigned)grid_for(rows, 256), 256, 0, st>>>(
            n, r0, r1, offs_dev, n_off, keep, seed, rpt_dev, col_dev, (float*)val_dev);
    else
        k_ham_fill<double><<<(unsigned)grid_for(rows, 256), 256, 0, st>>>(
            n, r0, r1, offs_dev, n_off, keep, seed, rpt_dev, col_dev, (double*)val_dev);
    SELLB_CU(cudaGetLastError());
    return 0;
}

}  // extern "C"
