// Dependent-chain latency of DADD / DMUL / FADD on this GPU (clock64 cycles).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a) {
    double s = out[0], t = out[1];
    float f = (float)out[2];
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, a);
    long long c1 = clock64();
    for (int i = 0; i < n; ++i) t = __dmul_rn(t, a);
    long long c2 = clock64();
    for (int i = 0; i < n; ++i) f = __fadd_rn(f, (float)a);
    long long c3 = clock64();
    out[0] = s; out[1] = t; out[2] = f;
    cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2;
}
int main() {
    double* o; long long* c;
    cudaMalloc(&o, 24); cudaMalloc(&c, 24);
    cudaMemset(o, 0, 24);
    const int n = 1 << 16;
    for (int rep = 0; rep < 2; ++rep) k<<<1, 1>>>(o, c, n, 1.0000001);
    long long h[3];
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: DADD %.2f  DMUL %.2f  FADD %.2f\n", (double)h[0] / n,
           (double)h[1] / n, (double)h[2] / n);
    return 0;
}
