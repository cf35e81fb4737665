// Dependent-chain latency of DADD / DMUL / FADD on this GPU (clock64 around
// 4096 dependent ops in one thread), and the throughput of independent chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, double x, double y) {
    double a = x;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < 4096; ++i) a = __dadd_rn(a, y);
    long long t1 = clock64();
    double m = x;
#pragma unroll 64
    for (int i = 0; i < 4096; ++i) m = __dmul_rn(m, y);
    long long t2 = clock64();
    float f = (float)x;
#pragma unroll 64
    for (int i = 0; i < 4096; ++i) f = __fadd_rn(f, (float)y);
    long long t3 = clock64();
    out[threadIdx.x] = a + m + f;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
    k_lat<<<1, 32>>>(out, cyc, 1.0, 1e-300);
    cudaDeviceSynchronize();
    k_lat<<<1, 32>>>(out, cyc, 1.0, 1e-300);
    cudaDeviceSynchronize();
    printf("DADD %.2f DMUL %.2f FADD %.2f cycles per dependent op\n", cyc[0] / 4096.0, cyc[1] / 4096.0, cyc[2] / 4096.0);
    return 0;
}
