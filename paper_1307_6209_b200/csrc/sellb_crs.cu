// sellb_crs.cu -- device-resident CRS handles for the reference's CRS kernel
// protocol (_kernels.pyx:17-62, spmv.py:76-102).  The kernels module calls
// spmv_crs_range(rpt, col, val, x, y, r0, r1, accumulate) on host arrays;
// the matrix arrays are uploaded once per handle (the Python layer caches
// handles by buffer identity, containers being immutable, formats.py:7) and
// every call moves only x in and the y range out.
#include <algorithm>
#include <mutex>

#include "sellb_internal.cuh"

using namespace sellb;

struct sellb_crs {
    int64_t n_rows = 0, n_cols = 0, nnz = 0;
    int32_t dtype = SELLB_F64, device = 0;
    int64_t* rpt = nullptr;
    int32_t* col = nullptr;
    void* val = nullptr;
    void* x_buf = nullptr;
    void* y_buf = nullptr;
    std::mutex mu;
};

namespace {

void free_crs(sellb_crs* m) {
    if (!m) return;
    DeviceGuard g(m->device);
    cudaFree(m->rpt);
    cudaFree(m->col);
    cudaFree(m->val);
    cudaFree(m->x_buf);
    cudaFree(m->y_buf);
    delete m;
}

}  // namespace

extern "C" {

int sellb_crs_import(const int64_t* rpt, const int32_t* col, const void* val, int32_t dtype,
                     int64_t n_rows, int64_t n_cols, int64_t nnz, int32_t device,
                     sellb_crs** out) {
    clear_error();
    if (!out) return set_error(SELLB_EPARAM, "out must not be NULL");
    *out = nullptr;
    if (dtype != SELLB_F64 && dtype != SELLB_F32)
        return set_error(SELLB_EPARAM, "dtype must be SELLB_F64 or SELLB_F32");
    if (n_rows < 0 || n_cols < 0 || nnz < 0) return set_error(SELLB_ESTRUCT, "negative dimension");
    if (!rpt || (nnz && (!col || !val))) return set_error(SELLB_EPARAM, "NULL array");
    // the CRSMatrix invariants the kernels index by (formats.py:140-155)
    if (rpt[0] != 0 || rpt[n_rows] != nnz)
        return set_error(SELLB_ESTRUCT, "rpt must start at 0 and end at nnz");
    for (int64_t i = 0; i < n_rows; ++i)
        if (rpt[i + 1] < rpt[i]) return set_error(SELLB_ESTRUCT, "rpt must be non-decreasing");
    for (int64_t k = 0; k < nnz; ++k)
        if (col[k] < 0 || (int64_t)col[k] >= n_cols)
            return set_error(SELLB_ESTRUCT, "column index out of bounds");
    DeviceGuard guard(device);
    if (!guard.ok) return set_error(SELLB_ERESOURCE, "cannot select CUDA device %d", device);
    sellb_crs* m = new (std::nothrow) sellb_crs();
    if (!m) return set_error(SELLB_ERESOURCE, "host allocation failed");
    m->n_rows = n_rows; m->n_cols = n_cols; m->nnz = nnz; m->dtype = dtype; m->device = device;
    const size_t vs = vsize(dtype);
    cudaError_t e = cudaMalloc(&m->rpt, (n_rows + 1) * 8);
    if (e == cudaSuccess) e = cudaMalloc(&m->col, std::max<int64_t>(nnz, 1) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&m->val, std::max<int64_t>(nnz, 1) * vs);
    if (e == cudaSuccess) e = cudaMalloc(&m->x_buf, std::max<int64_t>(n_cols, 1) * vs);
    if (e == cudaSuccess) e = cudaMalloc(&m->y_buf, std::max<int64_t>(n_rows, 1) * vs);
    if (e == cudaSuccess) e = cudaMemcpy(m->rpt, rpt, (n_rows + 1) * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(m->col, col, nnz * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(m->val, val, nnz * vs, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        free_crs(m);
        return set_error(SELLB_ERESOURCE, "CRS upload failed: %s", cudaGetErrorString(e));
    }
    *out = m;
    return 0;
}

int sellb_crs_spmv_host(sellb_crs* m, const void* x_host, void* y_host, int64_t r0, int64_t r1,
                        int32_t accumulate, int32_t unrolled) {
    clear_error();
    NvtxRange nvtx_("sellb_crs_spmv_host");
    if (!m || !y_host || (!x_host && m->n_cols)) return set_error(SELLB_EPARAM, "NULL argument");
    if (r0 < 0 || r1 > m->n_rows || r0 > r1) return set_error(SELLB_EPARAM, "bad row range");
    if (r0 == r1) return 0;
    DeviceGuard guard(m->device);
    std::lock_guard<std::mutex> lk(m->mu);
    const size_t vs = vsize(m->dtype);
    cudaStream_t st = 0;
    if (m->n_cols)
        SELLB_CU(cudaMemcpyAsync(m->x_buf, x_host, m->n_cols * vs, cudaMemcpyHostToDevice, st));
    if (accumulate)
        SELLB_CU(cudaMemcpyAsync((char*)m->y_buf + r0 * vs, (const char*)y_host + r0 * vs,
                                 (r1 - r0) * vs, cudaMemcpyHostToDevice, st));
    if (int rc = launch_spmv_crs(m->rpt, m->col, m->val, m->dtype, m->x_buf, m->y_buf, r0, r1,
                                 accumulate, unrolled, st))
        return rc;
    SELLB_CU(cudaMemcpyAsync((char*)y_host + r0 * vs, (const char*)m->y_buf + r0 * vs,
                             (r1 - r0) * vs, cudaMemcpyDeviceToHost, st));
    SELLB_CU(cudaStreamSynchronize(st));
    return 0;
}

void sellb_crs_free(sellb_crs* m) { free_crs(m); }

}  // extern "C"
