// lemix_tile_base_cb.cu -- instantiations of the tile event-loop kernel for the
// baseline policies (RR / Separate / Fixed / Mix-LUF) with Algorithm 3
// continuous batching + decode (see lemix_tile.cuh).
#include "lemix_tile.cuh"

namespace lmx {
typedef void (*tile_kernel_fn)(const KParams);
tile_kernel_fn pick_tile_base_cb(const KParams &p) { return tile::pick<false, tile::kCb>(p); }
}  // namespace lmx
