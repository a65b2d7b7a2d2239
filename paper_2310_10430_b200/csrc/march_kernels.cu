// 2D row-march sweep kernel (structured right-triangle meshes, BDIA offsets
// {0, +-1, +-W, +-(W+1)}): one outer iteration of the Jacobi-in-time inverted
// scheme with the block preconditioner (L238-262) fused.
//
// Tile = 8 consecutive grid columns x (32*T) time steps x a range of grid rows.
// Warp w owns column seg*8 + w and walks the rows upward, so the 8 warps of a
// CTA touch rows j-1, j, j+1 of a 10-column strip: those rows are served by L1
// (each x value is fetched from L2/HBM about once per tile instead of once per
// neighbouring row node) and row j+2 is prefetched into L1 one step ahead.
// The 8 nodes of a row are consecutive, so their coefficient blocks (8 x 7 x 10
// doubles) are one contiguous 4480-B TMA bulk copy (cp.async.bulk + mbarrier,
// double-buffered one row ahead); the compute reads them with warp-uniform LDS.
// Per-node arithmetic is dev::node_update -- the same FMA order as the generic
// kernel, so both produce bitwise identical iterates.
#include <cstdint>

#include "node_update.cuh"
#include "sweep_kernels.cuh"

namespace biot {

namespace {

using namespace dev;

constexpr int kRowNodes = 8;
constexpr int kCoefRow = kRowNodes * 7 * 10;        // doubles per staged row
constexpr uint32_t kCoefBytes = kCoefRow * 8;       // 4480 B, multiple of 16

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
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

template <int T>
__global__ void __launch_bounds__(kThreads, 2) march2d_kernel(const SweepArgs a) {
    constexpr int CH = 32 * T;
    constexpr int NC = 3;
    constexpr int S = 7;
    constexpr int WB = 10;                                // block pitch (doubles)
    __shared__ alignas(128) double coef[2][kCoefRow];
    __shared__ double red[8][CH][2];
    __shared__ uint64_t bar[2];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_chunks = (a.n_tl + CH - 1) / CH;
    const int64_t W = a.row_w;
    const int64_t n_seg = (W + kRowNodes - 1) / kRowNodes;
    const int64_t n_jr = (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
    const int64_t n_tiles = n_seg * n_jr * n_chunks;
    const int64_t P = a.pitch;

    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase[2] = {0u, 0u};

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int chunk = (int)(tile % n_chunks);
        const int64_t grp = tile / n_chunks;              // = jr * n_seg + seg
        const int64_t seg = grp % n_seg, jr = grp / n_seg;
        const int t0 = chunk * CH + lane * T;
        const int64_t col = seg * kRowNodes + warp;
        double nu[T], npn[T], sv[1][T];
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
            nu[tt] = 0.0;
            npn[tt] = 0.0;
            sv[0][tt] = (t0 + tt < a.n_tl) ? a.s[t0 + tt] : 0.0;
        }
        const int ja = (int)(jr * a.rows_per_tile);
        const int jb = min(a.n_rows, ja + a.rows_per_tile);
        constexpr int LPR = CH * 8 / 128;                  // 128-B lines per (node, comp) row
        const int pf = threadIdx.x;
        const bool do_pf = pf < (kRowNodes + 1) * NC * LPR;
        const int pf_node = pf / (NC * LPR), pf_comp = (pf / LPR) % NC, pf_line = pf % LPR;

        // coefficients of the first row
        if (threadIdx.x == 0)
            bulk_g2s(coef[ja & 1], a.blk + ((int64_t)ja * W + seg * kRowNodes) * (S * WB), kCoefBytes,
                     &bar[ja & 1]);
        for (int j = ja; j < jb; ++j) {
            const int st = j & 1;
            if (threadIdx.x == 0 && j + 1 < jb)   // next row's coefficients, one row ahead
                bulk_g2s(coef[st ^ 1], a.blk + ((int64_t)(j + 1) * W + seg * kRowNodes) * (S * WB),
                         kCoefBytes, &bar[st ^ 1]);
            if (do_pf && j + 2 < a.n_rows) {      // x of row j+2 (the +W neighbours of row j+1)
                const double *pp = a.x + (((int64_t)(j + 2) * W + seg * kRowNodes + pf_node) * NC + pf_comp) * P +
                                   chunk * CH + pf_line * 16;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(pp));
            }
            mbar_wait(&bar[st], phase[st]);
            phase[st] ^= 1u;
            if (col < W)
                node_update<2, S, false, T, true>(a, (int64_t)j * W + col, coef[st] + warp * (S * WB), t0, lane,
                                                  sv, nu, npn);
            __syncthreads();                      // stage st is refilled at row j+2
        }
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
            red[warp][lane * T + tt][0] = nu[tt];
            red[warp][lane * T + tt][1] = npn[tt];
        }
        __syncthreads();
        for (int k = threadIdx.x; k < CH * 2; k += kThreads) {
            const int tl = k >> 1, part = k & 1;
            const int t = chunk * CH + tl;
            if (t < a.n_tl) {
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < 8; ++w) sum += red[w][tl][part];
                a.partial[(grp * a.n_tl + t) * 2 + part] = sum;
            }
        }
        __syncthreads();
    }
}

template <int T>
cudaError_t march_shape_t(int device, LaunchShape *out) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    // favour L1: rows j-1..j+2 of each tile live there
    e = cudaFuncSetAttribute(march2d_kernel<T>, cudaFuncAttributePreferredSharedMemoryCarveout, 20);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, march2d_kernel<T>, kThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    out->smem = 0;
    return cudaSuccess;
}

}  // namespace

cudaError_t march_shape(int T, int device, LaunchShape *out) {
    if (T == 2) return march_shape_t<2>(device, out);
    if (T == 4) return march_shape_t<4>(device, out);
    return cudaErrorInvalidValue;
}

cudaError_t launch_march(int T, const SweepArgs &a, const LaunchShape &sh, cudaStream_t st) {
    if (T == 2) march2d_kernel<2><<<sh.grid, kThreads, 0, st>>>(a);
    else if (T == 4) march2d_kernel<4><<<sh.grid, kThreads, 0, st>>>(a);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace biot
