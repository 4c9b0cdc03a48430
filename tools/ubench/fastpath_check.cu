// Bitwise check of lmx::fast's branch-free fast-path replicas (rcp_fastpath,
// div_fastpath, sqrt_fastpath) against the IEEE operations ptxas expands
// (1.0 / x, a / b, sqrt(x)): wherever a replica reports its fast path taken,
// the result must carry the same bits.  Inputs: random bit patterns over the
// whole exponent range, the integer ranges Eq. 2 feeds in (counts, variances),
// Eq. 3-shaped quotients, and special values.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I include \
//        -I paper_2507_21276_b200/csrc tools/ubench/fastpath_check.cu -o /tmp/fpc
#include <cstdio>
#include <cstdint>
#include "lemix_fast.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double pick(uint64_t r, int mode)
{
    switch (mode) {
    case 0: return __longlong_as_double((long long)r);                        // any bits
    case 1: return (double)(1 + (r % 4000000ull));                           // counts
    case 2: return (double)(r >> 11);                                        // integer variances < 2^53
    case 3: return __longlong_as_double((long long)((r & 0x800fffffffffffffull) | ((0x3c0ull + (r >> 52) % 0x80ull) << 52)));   // |x| in [2^-63, 2^65)
    default: {
        const double sp[] = {0.0, -0.0, 1.0, -1.0, __longlong_as_double(0x7ff0000000000000ll), __longlong_as_double(0xfff0000000000000ll),
                             __longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(1ll), __longlong_as_double(0x0010000000000000ll),
                             __longlong_as_double(0x7fefffffffffffffll), 1e-300, 1e300};
        return sp[r % 12];
    }
    }
}
__global__ void check(uint64_t seed, long long n, unsigned long long *bad, unsigned long long *taken)
{
    unsigned long long b = 0, t = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint64_t r1 = mix(seed ^ (uint64_t)i), r2 = mix(r1), r3 = mix(r2);
        const int m1 = (int)(r3 % 5), m2 = (int)((r3 >> 8) % 5);
        const double x = pick(r1, m1), y = pick(r2, m2);
        bool ok;
        double v = lmx::dev::rcp_fastpath(x, ok);
        if (ok) { t++; b += __double_as_longlong(v) != __double_as_longlong(1.0 / x); }
        v = lmx::dev::div_fastpath(x, y, ok);
        if (ok) { t++; b += __double_as_longlong(v) != __double_as_longlong(x / y); }
        v = lmx::dev::sqrt_fastpath(fabs(x), ok);
        if (ok) { t++; b += __double_as_longlong(v) != __double_as_longlong(sqrt(fabs(x))); }
    }
    atomicAdd(bad, b);
    atomicAdd(taken, t);
}
int main()
{
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    const long long n = 1ll << 32;
    check<<<148 * 8, 256>>>(0x1234567ull, n, d, d + 1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("{\"inputs\": %lld, \"fast_path_results\": %llu, \"mismatches\": %llu, \"err\": \"%s\"}\n", n, h[1], h[0],
           cudaGetErrorString(cudaGetLastError()));
    return h[0] != 0;
}
