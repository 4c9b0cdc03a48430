// lemix_fast.cu -- instantiations of the one-node-per-lane LeMix kernel
// (see lemix_fast.cuh): pipeline depth S in {1, 2, 4} x tile width T.
#include "lemix_fast.cuh"

namespace lmx {
typedef void (*tile_kernel_fn)(const KParams);

template <int S>
static tile_kernel_fn pick_fast_t(int T)
{
    switch (T) {
    case 2: return fast::fast_loop_kernel<S, 2>;
    case 4: return fast::fast_loop_kernel<S, 4>;
    case 8: return fast::fast_loop_kernel<S, 8>;
    case 16: return fast::fast_loop_kernel<S, 16>;
    default: return fast::fast_loop_kernel<S, 32>;
    }
}

tile_kernel_fn pick_fast(const KParams &p)
{
    switch (p.S) {
    case 1: return pick_fast_t<1>(p.T);
    case 2: return pick_fast_t<2>(p.T);
    default: return pick_fast_t<4>(p.T);
    }
}

bool fast_applies(const KParams &p) { return fast::applies(p); }
int fast_smem_bytes(const KParams &p) { return fast::smem_bytes(p.N, p.S); }
}  // namespace lmx
