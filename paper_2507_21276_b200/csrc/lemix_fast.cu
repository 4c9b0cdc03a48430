// lemix_fast.cu -- instantiations of the one-node-per-lane LeMix kernel
// (see lemix_fast.cuh): pipeline depth S in {1, 2, 4} x tile width T (one-warp
// tiles), and the wide kernel, S in {2, 4, 8} x 2 or 4 warps per trace.
#include "lemix_fast.cuh"

namespace lmx {
typedef void (*tile_kernel_fn)(const KParams);

template <int S, bool LEAN>
static tile_kernel_fn pick_fast_t(int T)
{
    switch (T) {
    case 2: return fast::fast_loop_kernel<S, 2, 1, LEAN>;
    case 4: return fast::fast_loop_kernel<S, 4, 1, LEAN>;
    case 8: return fast::fast_loop_kernel<S, 8, 1, LEAN>;
    case 16: return fast::fast_loop_kernel<S, 16, 1, LEAN>;
    default: return fast::fast_loop_kernel<S, 32, 1, LEAN>;
    }
}

template <int TW, bool LEAN>
static tile_kernel_fn pick_wide(int S)
{
    switch (S) {
    case 2: return fast::fast_loop_kernel<2, 32, TW, LEAN>;
    case 4: return fast::fast_loop_kernel<4, 32, TW, LEAN>;
    default: return fast::fast_loop_kernel<8, 32, TW, LEAN>;
    }
}

tile_kernel_fn pick_fast(const KParams &p)
{
    const bool lean = fast::lean(p);
    if (p.N > 32) {
        if (fast::tile_warps(p) == 2) return lean ? pick_wide<2, true>(p.S) : pick_wide<2, false>(p.S);
        return lean ? pick_wide<4, true>(p.S) : pick_wide<4, false>(p.S);
    }
    switch (p.S) {
    case 1: return lean ? pick_fast_t<1, true>(p.T) : pick_fast_t<1, false>(p.T);
    case 2: return lean ? pick_fast_t<2, true>(p.T) : pick_fast_t<2, false>(p.T);
    default: return lean ? pick_fast_t<4, true>(p.T) : pick_fast_t<4, false>(p.T);
    }
}

bool fast_applies(const KParams &p) { return fast::applies(p); }
int fast_smem_bytes(const KParams &p) { return fast::smem_bytes(p.N, p.S, fast::tile_warps(p)); }
int fast_block_threads(const KParams &p) { return fast::block_threads(fast::tile_warps(p)); }
}  // namespace lmx
