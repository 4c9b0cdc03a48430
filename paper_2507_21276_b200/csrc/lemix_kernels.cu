// lemix_kernels.cu -- launchers of the sm_100a kernels of the LeMix placement
// step: the tile event loop (templates in lemix_tile.cuh, instantiated in
// lemix_tile_lemix.cu / lemix_tile_base.cu) and the cell reduction (K5, here).
//
// K1 profile staging : the fp64 SoA profile table (eta_f, eta_b) is copied
//                      into shared memory once per CTA with a TMA bulk copy
//                      (cp.async.bulk + mbarrier).
// K2-K4 event loop   : one persistent kernel.  A "tile" of T lanes of a warp
//                      owns one trace at a time; lane l plans nodes l, l+T, ...
//                      (Algorithm 1) and scores them (Eq. 1-3,
//                      PAPER.md:546-565); a tile shuffle takes the arg-best with
//                      the lowest-index tie-break; the owning
//                      lane commits.  Eq. 4 is a tile min.
//                      Tiles claim traces from a global counter until none are
//                      left, so long and short traces balance across SMs.
// K5 cell reduction  : per-cell sums of the per-trace summaries in a fixed
//                      order (deterministic), ready for one NCCL all-reduce.
//
// Compiled with --fmad=false: see lemix_device.cuh for the fp64 discipline.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "lemix_tile.cuh"

namespace lmx {

namespace {

constexpr int kBlock = 128;                 // 4 warps per CTA
using dev::kInf;
using dev::task_batch;
using dev::task_len;
using dev::task_w;

// ---- K5: per-cell sums of the per-trace summaries, fixed order ----
constexpr int kCellBlock = 256;

__global__ void __launch_bounds__(kCellBlock) cells_kernel(const CellParams c)
{
    __shared__ long long si[kCellBlock][LMX_CELL_NI];
    __shared__ double sf[kCellBlock][LMX_CELL_NF];
    const int cell = blockIdx.x;
    long long ai[LMX_CELL_NI];
    double af[LMX_CELL_NF];
#pragma unroll
    for (int k = 0; k < LMX_CELL_NI; ++k) ai[k] = 0;
#pragma unroll
    for (int k = 0; k < LMX_CELL_NF; ++k) af[k] = 0.0;
    // the cell's traces only (a CSR over traces sorted by cell, built on the
    // host), in a fixed order: thread k folds members k, k + 256, ...
    const long long b = c.cell_start ? c.cell_start[cell] : 0;
    const long long e = c.cell_start ? c.cell_start[cell + 1] : c.n_traces;
    for (long long m = b + threadIdx.x; m < e; m += kCellBlock) {
        const long long t = c.order ? c.order[m] : m;
        const lmx_summary s = c.summaries[t];
        ai[0] += 1;
        if (s.status != LMX_OK) { ai[1] += 1; continue; }
        ai[2] += s.n_tasks; ai[3] += s.n_inf; ai[4] += s.n_train; ai[5] += s.n_slo_met;
        ai[6] += s.n_deferrals; ai[7] += s.active_nodes; ai[8] += s.sum_version;
        af[0] = af[0] + s.makespan; af[1] = af[1] + s.throughput; af[2] = af[2] + s.sum_ttft;
        af[3] = af[3] + s.mean_ttft; af[4] = af[4] + s.slo_attainment; af[5] = af[5] + s.mean_util;
        af[6] = af[6] + s.mean_len_std;
    }
#pragma unroll
    for (int k = 0; k < LMX_CELL_NI; ++k) si[threadIdx.x][k] = ai[k];
#pragma unroll
    for (int k = 0; k < LMX_CELL_NF; ++k) sf[threadIdx.x][k] = af[k];
    __syncthreads();
    for (int h = kCellBlock / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) {
#pragma unroll
            for (int k = 0; k < LMX_CELL_NI; ++k) si[threadIdx.x][k] += si[threadIdx.x + h][k];
#pragma unroll
            for (int k = 0; k < LMX_CELL_NF; ++k) sf[threadIdx.x][k] = sf[threadIdx.x][k] + sf[threadIdx.x + h][k];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < LMX_CELL_NI; ++k) c.cell_i[cell * LMX_CELL_NI + k] = si[0][k];
#pragma unroll
        for (int k = 0; k < LMX_CELL_NF; ++k) c.cell_f[cell * LMX_CELL_NF + k] = sf[0][k];
    }
}

typedef void (*kernel_fn)(const KParams);

}  // namespace

kernel_fn pick_tile_lemix(const KParams &p);
kernel_fn pick_tile_base(const KParams &p);
kernel_fn pick_tile_lemix_mem(const KParams &p);
kernel_fn pick_tile_base_mem(const KParams &p);
kernel_fn pick_tile_lemix_cb(const KParams &p);
kernel_fn pick_tile_base_cb(const KParams &p);
kernel_fn pick_fast(const KParams &p);
bool fast_applies(const KParams &p);
int fast_smem_bytes(const KParams &p);
int fast_block_threads(const KParams &p);

namespace {

// LMX_KERNEL=generic (developer override): the tile kernel for every run,
// also where the one-node-per-lane LeMix kernel applies
bool use_fast(const KParams &p)
{
    static const bool generic = [] {
        const char *e = getenv("LMX_KERNEL");
        return e != nullptr && strcmp(e, "generic") == 0;
    }();
    return !generic && fast_applies(p);
}

kernel_fn pick(const KParams &p)
{
    if (use_fast(p)) return pick_fast(p);
    if (p.mem_enable) return p.policy == LMX_LEMIX ? pick_tile_lemix_mem(p) : pick_tile_base_mem(p);
    if (p.cb_cmax > 0) return p.policy == LMX_LEMIX ? pick_tile_lemix_cb(p) : pick_tile_base_cb(p);
    return p.policy == LMX_LEMIX ? pick_tile_lemix(p) : pick_tile_base(p);
}

}  // namespace

int max_stages_bucket(int S) { return tile::stages_bucket(S); }

int npl_bucket(int npl) { return tile::npl_bucket(npl); }

int event_loop_smem_bytes(const KParams &p)
{
    if (use_fast(p)) return fast_smem_bytes(p);
    const int W = tile::window_entries(p.S);
    const int npl = npl_bucket(p.npl);
    return (int)tile::profile_bytes(p.N * p.S, p.cb_cmax > 0) + (W > 0 ? kBlock * npl * W * ring_words(p.S, p.mem_enable != 0) * 16 : 0) +
           kBlock * (npl * tile::cold_words(p.S, npl > 1) + (p.cell_par ? tile::kTraceWords : 4)) * 8;
}

int event_loop_block_threads(const KParams &p) { return use_fast(p) ? fast_block_threads(p) : kBlock; }

int event_loop_traces_per_block(const KParams &p)
{
    // the wide kernel (several warps per trace) places one trace per CTA
    return use_fast(p) && p.N > 32 ? 1 : event_loop_block_threads(p) / p.T;
}

int event_loop_occupancy(const KParams &p, int *err)
{
    kernel_fn f = pick(p);
    const int smem = event_loop_smem_bytes(p);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int blocks = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, f, event_loop_block_threads(p), smem);
    *err = (int)e;
    return blocks;
}

int launch_event_loop(const KParams &p, int grid, void *stream)
{
    kernel_fn f = pick(p);
    const int smem = event_loop_smem_bytes(p);
    f<<<grid, event_loop_block_threads(p), smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

int launch_cells(const CellParams &c, void *stream)
{
    cells_kernel<<<c.n_cells, kCellBlock, 0, (cudaStream_t)stream>>>(c);
    return (int)cudaGetLastError();
}

}  // namespace lmx
