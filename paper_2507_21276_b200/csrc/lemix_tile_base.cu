// lemix_tile_base.cu -- instantiations of the tile event-loop kernel for
// the baselines (RR / Separate / Fixed) (see lemix_tile.cuh).
#include "lemix_tile.cuh"

namespace lmx {
typedef void (*tile_kernel_fn)(const KParams);
tile_kernel_fn pick_tile_base(const KParams &p) { return tile::pick<false, tile::kPlain>(p); }
}  // namespace lmx
