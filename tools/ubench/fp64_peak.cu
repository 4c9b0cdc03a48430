// Measured fp64 pipe throughput on this B200 (the roofline denominator of the
// event-loop kernels, bound "alu"): DADD and DMUL, 8 independent chains per
// thread, 148 x 8 CTAs of 256 threads, timed with CUDA events (best of 5).
// Also the fp64 instruction expansions of the correctly rounded division and
// square root and of the kernels' exp_neg are counted separately from SASS
// (tools/ubench/expansions.cu).  Build: nvcc -arch=sm_100a -O3 --fmad=false
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
template <int OP>
__global__ void k(double *out, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 8
    for (int i = 0; i < ITERS; ++i) {
        if (OP == 0) {
            x0 = x0 + a; x1 = x1 + a; x2 = x2 + a; x3 = x3 + a; x4 = x4 + a; x5 = x5 + a; x6 = x6 + a; x7 = x7 + a;
        } else {
            x0 = x0 * b; x1 = x1 * b; x2 = x2 * b; x3 = x3 * b; x4 = x4 * b; x5 = x5 * b; x6 = x6 * b; x7 = x7 * b;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <int OP>
double run(double *o, int grid, int block) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        k<OP><<<grid, block>>>(o, 1e-300, 1.0000000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    return (double)grid * block * ITERS * 8 / (best * 1e-3) / 1e12;
}
int main() {
    int dev = 0, sms = 0, mhz = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, dev);
    const int grid = sms * 8, block = 256;
    double *o; cudaMalloc(&o, (size_t)grid * block * 8);
    const double add = run<0>(o, grid, block), mul = run<1>(o, grid, block);
    const double nominal = 64.0 * sms * (mhz / 1e3) * 1e6 / 1e12;
    printf("{\"dadd_tops\": %.3f, \"dmul_tops\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, "
           "\"nominal_64_lanes_tops\": %.3f, \"how\": \"8 independent chains/thread, %d CTAs x %d threads x %d iters, best of 5 (CUDA events)\"}\n",
           add, mul, sms, mhz / 1000, nominal, grid, block, ITERS);
    return 0;
}
