// lemix_tile_lemix_mem.cu -- instantiations of the tile event-loop kernel for the
// LeMix policy with the memory model of Algorithm 2 (see lemix_tile.cuh).
#include "lemix_tile.cuh"

namespace lmx {
typedef void (*tile_kernel_fn)(const KParams);
tile_kernel_fn pick_tile_lemix_mem(const KParams &p) { return tile::pick<true, tile::kMem>(p); }
}  // namespace lmx
