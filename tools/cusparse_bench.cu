// cusparse_bench.cu -- library comparison arm for tools/cusparse_compare.py
// ("compare against cuSPARSE CSR and Sliced-ELL on the same
// box").  Not part of the product; built into tools/_build/ by
// tools/cusparse_compare.py.  All pointers are device pointers.
#include <cuda_runtime.h>
#include <cusparse.h>
#include <cstdint>
#include <cstdio>

#define CK(x)                                                                     \
    do {                                                                          \
        cusparseStatus_t s_ = (x);                                                \
        if (s_ != CUSPARSE_STATUS_SUCCESS) {                                      \
            fprintf(stderr, "cusparse %s:%d: %s\n", __FILE__, __LINE__,           \
                    cusparseGetErrorString(s_));                                  \
            return -1;                                                            \
        }                                                                         \
    } while (0)

extern "C" {

// fmt: 0 = CSR ALG1, 1 = CSR ALG2, 2 = SELL (sliced ELL) ALG1
// CSR:  ptr = int32 row offsets [n_rows+1], col int32 [nnz], val [nnz]
// SELL: ptr = int32 slice offsets [n_slices+1], col int32 [val_size] (-1 pads),
//       val [val_size], slice = slice size
// ms_out: average ms per SpMV over `reps` launches (one event pair around all)
int csp_spmv(int fmt, int f32, int64_t n_rows, int64_t n_cols, int64_t nnz, int64_t val_size,
             int slice, const void* ptr, const int32_t* col, const void* val, const void* x,
             void* y, int warmup, int reps, float* ms_out) {
    cusparseHandle_t h;
    CK(cusparseCreate(&h));
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    CK(cusparseSetStream(h, st));
    const cudaDataType vt = f32 ? CUDA_R_32F : CUDA_R_64F;
    cusparseSpMatDescr_t A;
    cusparseSpMVAlg_t alg;
    if (fmt == 2) {
        CK(cusparseCreateSlicedEll(&A, n_rows, n_cols, nnz, val_size, slice, (void*)ptr,
                                   (void*)col, (void*)val, CUSPARSE_INDEX_32I,
                                   CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO, vt));
        alg = CUSPARSE_SPMV_SELL_ALG1;
    } else {
        CK(cusparseCreateCsr(&A, n_rows, n_cols, nnz, (void*)ptr, (void*)col, (void*)val,
                             CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO,
                             vt));
        alg = fmt == 0 ? CUSPARSE_SPMV_CSR_ALG1 : CUSPARSE_SPMV_CSR_ALG2;
    }
    cusparseDnVecDescr_t X, Y;
    CK(cusparseCreateDnVec(&X, n_cols, (void*)x, vt));
    CK(cusparseCreateDnVec(&Y, n_rows, y, vt));
    double a64 = 1.0, b64 = 0.0;
    float a32 = 1.0f, b32 = 0.0f;
    const void* alpha = f32 ? (const void*)&a32 : (const void*)&a64;
    const void* beta = f32 ? (const void*)&b32 : (const void*)&b64;
    size_t bsz = 0;
    CK(cusparseSpMV_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, X, beta, Y, vt,
                               alg, &bsz));
    void* buf = nullptr;
    if (bsz) cudaMalloc(&buf, bsz);
    CK(cusparseSpMV_preprocess(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, X, beta, Y, vt,
                               alg, buf));
    for (int i = 0; i < warmup; ++i)
        CK(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, X, beta, Y, vt, alg,
                        buf));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaStreamSynchronize(st);
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps; ++i)
        CK(cusparseSpMV(h, CUSPARSE_OPERATION_NON_TRANSPOSE, alpha, A, X, beta, Y, vt, alg,
                        buf));
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_out = reps ? ms / reps : 0.f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (buf) cudaFree(buf);
    cusparseDestroyDnVec(X);
    cusparseDestroyDnVec(Y);
    cusparseDestroySpMat(A);
    cudaStreamDestroy(st);
    cusparseDestroy(h);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
}
