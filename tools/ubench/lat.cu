// Dependent-chain latency microbenchmark (one warp): cycles per op for fp64
// add, mul, MAX (compare + select), fp64 division, shared-memory load and
// warp shuffle on the B200 this runs on.  Build: nvcc -arch=sm_100a --fmad=false
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(double *out, long long *cyc, double x0, double y0) {
    __shared__ double sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = (double)threadIdx.x;
    __syncthreads();
    double x = x0 + threadIdx.x, y = y0;
    long long t0, t1;
    // DADD
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x + y;
    t1 = clock64(); cyc[0] = t1 - t0;
    // DMUL
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = x * y;
    t1 = clock64(); cyc[1] = t1 - t0;
    // MAX as compare + select (the kernels' dmax)
    double z = y;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) { x = (z > x) ? z : x; z = z + 0.0; }
    t1 = clock64(); cyc[2] = t1 - t0;
    // MAX then ADD (one Algorithm 1 step: st = MAX(st, e); en = st + dF)
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) { double m = (y > x) ? y : x; x = m + 1e-300; }
    t1 = clock64(); cyc[3] = t1 - t0;
    // division
    t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N / 8; ++i) x = y / x;
    t1 = clock64(); cyc[4] = (t1 - t0) * 8;
    // LDS chain (address from the loaded value)
    int a = threadIdx.x & 31;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) a = ((int)sm[a]) & 31;
    t1 = clock64(); cyc[5] = t1 - t0;
    // SHFL chain
    double s = x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1);
    t1 = clock64(); cyc[6] = t1 - t0;
    // integer add chain
    int q = threadIdx.x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) q = q + a;
    t1 = clock64(); cyc[7] = t1 - t0;
    // 4 independent DADD chains (throughput of one warp)
    double x1 = x + 1, x2 = x + 2, x3 = x + 3;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) { x = x + y; x1 = x1 + y; x2 = x2 + y; x3 = x3 + y; }
    t1 = clock64(); cyc[8] = t1 - t0;
    out[threadIdx.x] = x + z + s + (double)a + (double)q + x1 + x2 + x3;
}
int main() {
    double *o; long long *c, h[9];
    cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 9 * 8);
    k<<<1, 32>>>(o, c, 1.0, 1.0000001);
    k<<<1, 32>>>(o, c, 1.0, 1.0000001);
    cudaMemcpy(h, c, 9 * 8, cudaMemcpyDeviceToHost);
    const char *nm[9] = {"dadd", "dmul", "dmax(cmp+sel)", "dmax+dadd", "ddiv", "lds", "shfl.f64", "iadd", "4x dadd (per iter)"};
    for (int i = 0; i < 9; ++i) printf("%-20s %.2f cycles/op\n", nm[i], (double)h[i] / N);
    return 0;
}
