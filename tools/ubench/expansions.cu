// One correctly rounded fp64 division, one sqrt and one exp_neg (the event
// loop's Eq. 2 routine) in isolation: `cuobjdump -sass` of this file's kernels
// counts the fp64 pipe instructions each expands to on sm_100a (the weights
// bench.py's roofline uses).  Build: nvcc -arch=sm_100a -O3 --fmad=false -cubin
#include "../../paper_2507_21276_b200/csrc/lemix_device.cuh"
extern "C" __global__ void k_div(const double *a, double *o) { o[0] = a[0] / a[1]; }
extern "C" __global__ void k_sqrt(const double *a, double *o) { o[0] = sqrt(a[0]); }
extern "C" __global__ void k_exp(const double *a, double *o) { o[0] = lmx::dev::exp_neg(a[0]); }
