// Panel kernels of the per-step GMRES (Alg. 3 with K = GMRES, reading R23):
// per-time-step dot products of space-time panels and per-step linear combinations.
// A panel holds one row per (node, component), time-contiguous: p[row * pitch + t];
// the Krylov vectors of all N_t step-systems live in one panel each, so every
// operation below is column-wise (one independent value per time step).
#include <cuda_runtime.h>
#include <cstdint>

#include "sweep_kernels.cuh"

namespace biot {

namespace {

constexpr int kCols = 64;     // time steps per block (threads along t: coalesced rows)
constexpr int kRowsY = 4;     // row lanes per block
constexpr int kMaxVec = 17;   // Krylov vectors a dot / combine call may touch (k <= 16)

// Stage 1: block (column block bx, row chunk by) sums rows [by*chunk, ..) of
// a[row][t] * b_i[row][t] for i < nb, in a fixed split over the kRowsY row lanes,
// then in fixed lane order; out[(by * nb + i) * n_tl + t].
__global__ void dots_stage1(const double *__restrict__ a, const double *const *__restrict__ b, int boff, int nb,
                            int64_t rows, int64_t pitch, int n_tl, int64_t chunk, double *__restrict__ out) {
    __shared__ double sm[kRowsY][kMaxVec][kCols];
    const int t = blockIdx.x * kCols + threadIdx.x;
    const int64_t r0 = blockIdx.y * chunk, r1 = min(rows, r0 + chunk);
    double acc[kMaxVec];
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) acc[i] = 0.0;
    if (t < n_tl) {
        for (int64_t r = r0 + threadIdx.y; r < r1; r += kRowsY) {
            const double av = a[r * pitch + t];
#pragma unroll
            for (int i = 0; i < kMaxVec; ++i)
                if (i < nb) acc[i] = fma(av, b[i][r * pitch + boff + t], acc[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i)
        if (i < nb) sm[threadIdx.y][i][threadIdx.x] = acc[i];
    __syncthreads();
    if (threadIdx.y == 0 && t < n_tl) {
        for (int i = 0; i < nb; ++i) {
            double s = 0.0;
            for (int y = 0; y < kRowsY; ++y) s += sm[y][i][threadIdx.x];
            out[((int64_t)blockIdx.y * nb + i) * n_tl + t] = s;
        }
    }
}

// Stage 2: fixed-order sum over the row chunks.
__global__ void dots_stage2(const double *__restrict__ part, int chunks, int nb, int n_tl, double *__restrict__ out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= (int64_t)nb * n_tl) return;
    const int i = (int)(k / n_tl), t = (int)(k % n_tl);
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += part[((int64_t)c * nb + i) * n_tl + t];
    out[(int64_t)i * n_tl + t] = s;
}

// dst[row][t] = scale[t] * (base[row][t] + sign * sum_i coef[i][t] * b_i[row][boff + t])
// (scale == nullptr: 1; base may alias dst).
__global__ void combine_kernel(double *dst, const double *base, const double *const *__restrict__ b, int boff,
                               const double *__restrict__ coef, int nb, double sign,
                               const double *__restrict__ scale, int64_t rows, int64_t pitch, int n_tl) {
    const int t = blockIdx.x * kCols + threadIdx.x;
    if (t >= n_tl) return;
    double c[kMaxVec];
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) c[i] = i < nb ? sign * coef[(int64_t)i * n_tl + t] : 0.0;
    const double sc = scale ? scale[t] : 1.0;
    for (int64_t r = blockIdx.y * (int64_t)blockDim.y + threadIdx.y; r < rows; r += (int64_t)gridDim.y * blockDim.y) {
        double v = base[r * pitch + t];
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i)
            if (i < nb) v = fma(c[i], b[i][r * pitch + boff + t], v);
        dst[r * pitch + t] = sc * v;
    }
}

}  // namespace

int gmres_max_vectors() { return kMaxVec; }

int64_t gmres_dots_scratch(int64_t rows, int n_tl, int nb, int64_t *chunk, int *chunks) {
    // ~512 row chunks: enough blocks for the GPU at any n_tl
    int64_t ch = (rows + 511) / 512;
    if (ch < 256) ch = 256;
    *chunk = ch;
    *chunks = (int)((rows + ch - 1) / ch);
    return (int64_t)(*chunks) * nb * n_tl;
}

cudaError_t gmres_dots(const double *a, const double *const *b_dev, int boff, int nb, int64_t rows, int64_t pitch,
                       int n_tl, double *scratch, double *out, cudaStream_t st) {
    if (nb < 1 || nb > kMaxVec) return cudaErrorInvalidValue;
    int64_t chunk;
    int chunks;
    gmres_dots_scratch(rows, n_tl, nb, &chunk, &chunks);
    dots_stage1<<<dim3((n_tl + kCols - 1) / kCols, chunks), dim3(kCols, kRowsY), 0, st>>>(a, b_dev, boff, nb, rows,
                                                                                          pitch, n_tl, chunk, scratch);
    const int64_t n = (int64_t)nb * n_tl;
    dots_stage2<<<(int)((n + 255) / 256), 256, 0, st>>>(scratch, chunks, nb, n_tl, out);
    return cudaGetLastError();
}

cudaError_t gmres_combine(double *dst, const double *base, const double *const *b_dev, int boff, const double *coef,
                          int nb, double sign, const double *scale, int64_t rows, int64_t pitch, int n_tl,
                          cudaStream_t st) {
    if (nb < 0 || nb > kMaxVec) return cudaErrorInvalidValue;
    const int gy = (int)((rows + 7) / 8 < 4096 ? (rows + 7) / 8 : 4096);
    combine_kernel<<<dim3((n_tl + kCols - 1) / kCols, gy), dim3(kCols, 8), 0, st>>>(dst, base, b_dev, boff, coef, nb,
                                                                                    sign, scale, rows, pitch, n_tl);
    return cudaGetLastError();
}

}  // namespace biot
