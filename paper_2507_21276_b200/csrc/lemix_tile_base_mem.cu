// lemix_tile_base_mem.cu -- instantiations of the tile event-loop kernel for the
// baseline policies (RR / Separate / Fixed) with the memory model of Algorithm 2 (see lemix_tile.cuh).
#include "lemix_tile.cuh"

namespace lmx {
typedef void (*tile_kernel_fn)(const KParams);
tile_kernel_fn pick_tile_base_mem(const KParams &p) { return tile::pick<false, tile::kMem>(p); }
}  // namespace lmx
