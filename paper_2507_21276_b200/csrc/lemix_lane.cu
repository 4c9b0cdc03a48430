// lemix_lane.cu -- instantiations and launcher of the lane-per-trace event
// loop (lemix_lane.cuh): small clusters, N <= 4 nodes, S <= 2 stages, without
// the Algorithm 2 memory model or per-cell parameters (those run on the tile
// kernel, lemix_tile.cuh).
#include "lemix_lane.cuh"

namespace lmx {

bool lane_supported(const KParams &p)
{
    return p.N <= 4 && (p.S == 1 || p.S == 2) && !p.mem_enable && p.cell_par == nullptr;
}

int lane_nodes_bucket(int N) { return lane::nmax_bucket(N); }

int lane_block_threads() { return lane::kBlock; }

int lane_smem_bytes(const KParams &p) { return lane::smem_bytes(p.N, p.S, lane::nmax_bucket(p.N)); }

static lane::kernel_fn lane_pick(const KParams &p)
{
    return p.policy == LMX_LEMIX ? lane::pick<true>(p) : lane::pick<false>(p);
}

int lane_occupancy(const KParams &p, int *err)
{
    lane::kernel_fn f = lane_pick(p);
    const int smem = lane_smem_bytes(p);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int blocks = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, f, lane::kBlock, smem);
    *err = (int)e;
    return blocks;
}

int launch_lane_loop(const KParams &p, int grid, void *stream)
{
    lane::kernel_fn f = lane_pick(p);
    f<<<grid, lane::kBlock, lane_smem_bytes(p), (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace lmx
