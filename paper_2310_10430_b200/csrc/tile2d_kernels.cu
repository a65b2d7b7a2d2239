// TMA-pipelined 2D sweep kernel (structured right-triangle meshes, BDIA slot
// order [0, -W-1, -W, -1, +1, +W, +W+1]).  One outer iteration of the
// Jacobi-in-time inverted scheme with the block
// preconditioner (L238-262), the damped update and the per-step norms fused.
//
// Work tile = 8 consecutive grid columns x 64 time steps x a range of grid rows,
// marched upward.  A producer warp streams, for every grid row r of the tile
// (plus the halo rows), one TMA tensor box -- the 10-node strip (8 columns + 2
// halo) x 3 components x 66 time steps (t0-2 .. t0+63) of the space-time panel --
// and one bulk copy of the 8 row nodes' aux records (kappa-dependent pressure
// entries, load, preconditioner diagonals) into a 6-stage shared-memory ring
// (full/empty mbarriers).  Consumer warp w computes node (r, i0+w) from shared
// memory only: its 7 neighbours are in the ring stages of rows r-1, r, r+1.
// Every x value is read from HBM/L2 once per tile (+25% halo from L2), and the
// compute warps issue no global loads except for boundary-class nodes.
//
// Interior nodes share one stencil (uniform lambda, mu, alpha, S and mesh):
// their blocks are passed once as kernel parameters (constant bank operands);
// only the kappa-dependent pressure-pressure entry of AA varies per node and
// comes from the aux record.  Nodes whose blocks differ from the template
// (boundary rows/columns, Dirichlet masking) read their full blocks from global
// memory.  All arithmetic goes through dev::node_epilogue with the same FMA order
// as the generic kernel, so iterates are bitwise identical to it.
#include <cuda.h>
#include <cstdint>

#include "node_update.cuh"
#include "sweep_kernels.cuh"

namespace biot {

namespace {

using namespace dev;

constexpr int kSeg = 8;                     // row nodes per tile
constexpr int kStrip = kSeg + 2;            // with halo columns
constexpr int kT = 2;                       // time steps per lane
constexpr int kCh = 32 * kT;                // time steps per tile
constexpr int kChp = kCh + 2;               // + halo steps t0-2, t0-1
constexpr int kXRows = kStrip * 3;          // tensor rows per stage
constexpr uint32_t kXBytes = kXRows * kChp * 8;           // 15840
constexpr uint32_t kAuxOff = (kXBytes + 127) / 128 * 128; // 15872
constexpr uint32_t kAuxBytes = kSeg * Tile2dArgs::kAux * 8;  // 1024
constexpr uint32_t kStageBytes = (kAuxOff + kAuxBytes + 127) / 128 * 128;
constexpr int kStages = 6;
constexpr int kConsumers = 8;
constexpr int kThreadsT = (kConsumers + 1) * 32;

// (row delta, column delta) of the 7 BDIA slots in storage order
__device__ constexpr int kDr[7] = {0, -1, -1, 0, 0, 1, 1};
__device__ constexpr int kDc[7] = {0, -1, 0, -1, 1, 0, 1};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct TileGeom {
    int64_t n_seg, n_jr, n_chunks, n_tiles;
    __device__ TileGeom(const Tile2dArgs &a) {
        n_seg = (a.row_w + kSeg - 1) / kSeg;
        n_jr = (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
        n_chunks = (a.n_tl + kCh - 1) / kCh;
        n_tiles = n_seg * n_jr * n_chunks;
    }
};

__global__ void __launch_bounds__(kThreadsT, 2)
    tile2d_kernel(const __grid_constant__ CUtensorMap tmx, const Tile2dArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    __shared__ double red[kConsumers][kCh][2];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TileGeom g(a);
    const int64_t W = a.row_w;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kConsumers) {
        // ------------------------------- producer -------------------------------
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t tile = blockIdx.x; tile < g.n_tiles; tile += gridDim.x) {
                const int chunk = (int)(tile % g.n_chunks);
                const int64_t grp = tile / g.n_chunks;
                const int64_t seg = grp % g.n_seg, jr = grp / g.n_seg;
                const int ja = (int)(jr * a.rows_per_tile);
                const int jb = min(a.n_rows, ja + a.rows_per_tile);
                const int64_t i0 = seg * kSeg;
                for (int r = ja - 1; r <= jb; ++r, ++it) {
                    const int st = it % kStages;
                    if (it >= (uint32_t)kStages) mbar_wait(&empty[st], ((it / kStages) - 1) & 1);
                    unsigned char *base = smem + (size_t)st * kStageBytes;
                    const bool real = (r >= 0 && r < a.n_rows);
                    mbar_expect_tx(&full[st], kXBytes + (real ? kAuxBytes : 0u));
                    const int64_t node0 = (int64_t)r * W + i0 - 1;
                    tma_load_2d(base, &tmx, chunk * kCh - 2, (int)((node0 + a.pad_nodes) * 3), &full[st]);
                    if (real)
                        bulk_g2s(base + kAuxOff, a.aux + ((int64_t)r * W + i0) * Tile2dArgs::kAux, kAuxBytes,
                                 &full[st]);
                }
            }
        }
        return;
    }

    // ------------------------------- consumers ------------------------------
    uint32_t it = 0;
    const int tw = warp;                       // column within the segment
    for (int64_t tile = blockIdx.x; tile < g.n_tiles; tile += gridDim.x) {
        const int chunk = (int)(tile % g.n_chunks);
        const int64_t grp = tile / g.n_chunks;
        const int64_t seg = grp % g.n_seg, jr = grp / g.n_seg;
        const int ja = (int)(jr * a.rows_per_tile);
        const int jb = min(a.n_rows, ja + a.rows_per_tile);
        const int64_t i0 = seg * kSeg;
        const int64_t col = i0 + tw;
        const int t0 = chunk * kCh + lane * kT;
        double nu[kT], npn[kT], sv[kT];
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
            nu[tt] = 0.0;
            npn[tt] = 0.0;
            sv[tt] = (t0 + tt < a.n_tl) ? a.s[t0 + tt] : 0.0;
        }
        const uint32_t it0 = it;               // item of row ja-1
        // rows ja-1 and ja
        mbar_wait(&full[it0 % kStages], (it0 / kStages) & 1);
        mbar_wait(&full[(it0 + 1) % kStages], ((it0 + 1) / kStages) & 1);
        for (int j = ja; j < jb; ++j) {
            const uint32_t ic = it0 + 1 + (j - ja);           // item of row j
            const uint32_t in = ic + 1;
            mbar_wait(&full[in % kStages], (in / kStages) & 1);
            const double *rowp[3] = {
                reinterpret_cast<const double *>(smem + (size_t)((ic - 1) % kStages) * kStageBytes),
                reinterpret_cast<const double *>(smem + (size_t)(ic % kStages) * kStageBytes),
                reinterpret_cast<const double *>(smem + (size_t)(in % kStages) * kStageBytes)};
            const double *aux = reinterpret_cast<const double *>(smem + (size_t)(ic % kStages) * kStageBytes +
                                                                 kAuxOff) + tw * Tile2dArgs::kAux;
            if (col < W) {
                const int64_t i = (int64_t)j * W + col;
                const bool interior = aux[13] != 0.0;
                double acc[3][kT], q[kT];
#pragma unroll
                for (int tt = 0; tt < kT; ++tt) {
                    q[tt] = 0.0;
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[c][tt] = 0.0;
                }
                const double *gb = a.blk + i * (7 * 10);          // boundary-class blocks
#pragma unroll
                for (int s = 0; s < 7; ++s) {
                    const double *xs_ = rowp[1 + kDr[s]] + ((tw + 1 + kDc[s]) * 3) * kChp + 2 + lane * kT;
                    double cf[10];
                    if (interior) {
#pragma unroll
                        for (int k = 0; k < 10; ++k) cf[k] = a.tmpl[s][k];
                        cf[8] = aux[s];                                // kappa-dependent AA_pp entry
                    } else {
#pragma unroll
                        for (int k = 0; k < 10; ++k) cf[k] = __ldg(gb + s * 10 + k);
                    }
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) {
                        const double2 w2 = *reinterpret_cast<const double2 *>(xs_ + cc * kChp);
                        const double v[kT] = {w2.x, w2.y};
#pragma unroll
                        for (int c = 0; c < 3; ++c)
#pragma unroll
                            for (int tt = 0; tt < kT; ++tt) acc[c][tt] = fma(cf[c * 3 + cc], v[tt], acc[c][tt]);
                        const double qc = (cc < 2) ? cf[2 * 3 + cc] : cf[9];
#pragma unroll
                        for (int tt = 0; tt < kT; ++tt) q[tt] = fma(qc, v[tt], q[tt]);
                    }
                }
                double qprev = __shfl_up_sync(0xffffffffu, q[kT - 1], 1);
                if (lane == 0) {
                    const bool use_ghost = (t0 == 0);
                    double qg = 0.0;
#pragma unroll
                    for (int s = 0; s < 7; ++s) {
                        const double *xs1 = rowp[1 + kDr[s]] + ((tw + 1 + kDc[s]) * 3) * kChp + 1;
                        const int64_t jn = i + a.off[s];
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) {
                            double qc;
                            if (interior) qc = (cc < 2) ? a.tmpl[s][2 * 3 + cc] : a.tmpl[s][9];
                            else qc = (cc < 2) ? __ldg(gb + s * 10 + 2 * 3 + cc) : __ldg(gb + s * 10 + 9);
                            const double xv = use_ghost ? __ldg(a.ghost + jn * 3 + cc) : xs1[cc * kChp];
                            qg = fma(qc, xv, qg);
                        }
                    }
                    qprev = qg;
                }
                double F[3], Dv[3], xs[3][kT];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    F[c] = aux[7 + c];
                    Dv[c] = aux[10 + c];
                    const double2 w2 = *reinterpret_cast<const double2 *>(rowp[1] + ((tw + 1) * 3 + c) * kChp + 2 +
                                                                          lane * kT);
                    xs[c][0] = w2.x;
                    xs[c][1] = w2.y;
                }
                node_epilogue<2, kT>(a, i, t0, acc, q, qprev, F, Dv, xs, sv, nu, npn);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[(ic - 1) % kStages]);   // row j-1 no longer needed
        }
        // rows jb-1 and jb are released at the end of the tile
        const uint32_t ilast = it0 + 1 + (jb - ja);                  // item of row jb
        if (lane == 0) {
            mbar_arrive(&empty[(ilast - 1) % kStages]);
            mbar_arrive(&empty[ilast % kStages]);
        }
        it = ilast + 1;
        // per-step norm partials of this tile (fixed reduction order over warps)
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
            red[tw][lane * kT + tt][0] = nu[tt];
            red[tw][lane * kT + tt][1] = npn[tt];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
        for (int k = threadIdx.x; k < kCh * 2; k += kConsumers * 32) {
            const int tl = k >> 1, part = k & 1;
            const int t = chunk * kCh + tl;
            if (t < a.n_tl) {
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < kConsumers; ++w) sum += red[w][tl][part];
                a.partial[(grp * a.n_tl + t) * 2 + part] = sum;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
    }
}

}  // namespace

int64_t tile2d_groups(const Tile2dArgs &a) {
    const int64_t n_seg = (a.row_w + kSeg - 1) / kSeg;
    const int64_t n_jr = (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
    return n_seg * n_jr;
}

int tile2d_chunk() { return kCh; }

cudaError_t tile2d_shape(int device, LaunchShape *out) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)kStages * kStageBytes;
    e = cudaFuncSetAttribute(tile2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile2d_kernel, kThreadsT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    out->smem = smem;
    return cudaSuccess;
}

cudaError_t launch_tile2d(const CUtensorMap &tmx, const Tile2dArgs &a, const LaunchShape &sh,
                          cudaStream_t st) {
    tile2d_kernel<<<sh.grid, kThreadsT, sh.smem, st>>>(tmx, a);
    return cudaGetLastError();
}

// box of the x tensor map: {time steps incl. halo, tensor rows}
void tile2d_box(uint32_t *box) {
    box[0] = kChp;
    box[1] = kXRows;
}

}  // namespace biot
