// lemix_tile_lemix.cu -- instantiations of the tile event-loop kernel for
// the LeMix policy (see lemix_tile.cuh).
#include "lemix_tile.cuh"

namespace lmx {
typedef void (*tile_kernel_fn)(const KParams);
tile_kernel_fn pick_tile_lemix(const KParams &p) { return tile::pick<true, tile::kPlain>(p); }
}  // namespace lmx
