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

// Block shapes: COLS threads along t (coalesced row segments) x 256 / COLS row lanes.
// Wide windows use COLS = 64; the narrow windows of the Gauss-Seidel wavefront (a few
// steps) use COLS = 16, 8 or 2 so that most threads still have a column to work on.
// Narrow windows keep their Krylov basis COMPACT (pitch = window width, rows adjacent):
// a window of 16 steps in the full panel layout is one 128-B run every 8 KB, which HBM
// serves at ~1/3 of its streaming rate (biot_api.cu gmres_cycle).
constexpr int kThr = 256;
constexpr int kMaxVec = 17;   // Krylov vectors a dot / combine call may touch (k <= 16)

// Stage 1: for every row chunk c (rows [c*chunk, ..)) the partial sums of
// a[row][t] * b_i[row][boff + t], i < NB, in a fixed split over kLanes = 16 row lanes (lane l:
// rows = l mod 16, in order) and then in fixed lane order; out[(c * NB + i) * n_tl + t].  A
// block holds kCols columns x 16 lanes x kCPB chunks, so the summation order of a column
// depends only on the (fixed) chunk size, not on the block shape chosen for the window
// width: results are independent of how many columns a call covers (time slabs stay
// bitwise).  16 lanes x ~2048 chunks: a 16-column window still fills the GPU with
// independent row streams, and each chunk reads 16 adjacent rows at a time.  NB is a
// template parameter so the loads of one row are issued together (no predicates).
constexpr int kLanes = 16;
template <int kCols>
struct DotsShape {
    static constexpr int kCPB = kCols * kLanes >= kThr ? 1 : kThr / (kCols * kLanes);
    static constexpr int kThreads = kCols * kLanes * kCPB;
};

template <int NB, int kCols>
__global__ void __launch_bounds__(DotsShape<kCols>::kThreads)
    dots_stage1(const double *__restrict__ a, const double *const *__restrict__ b, int boff, int64_t rows,
                int64_t pitch, int n_tl, int64_t chunk, int chunks, double *__restrict__ out) {
    constexpr int kCPB = DotsShape<kCols>::kCPB;
    extern __shared__ double sm[];   // [kCPB][kLanes][NB][kCols]
    const int lane = threadIdx.y % kLanes, z = threadIdx.y / kLanes;
    const int t = blockIdx.x * kCols + threadIdx.x;
    const int c = blockIdx.y * kCPB + z;
    const int64_t r0 = (int64_t)c * chunk, r1 = c < chunks ? min(rows, r0 + chunk) : r0;
    const double *bp[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) bp[i] = b[i] + boff;
    double acc[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) acc[i] = 0.0;
    if (t < n_tl) {
        // two rows of the lane per step, every load issued before the FMAs consume them
        // (the compiler interleaves them otherwise: too few loads in flight on narrow windows)
        int64_t r = r0 + lane;
        for (; r + kLanes < r1; r += 2 * kLanes) {
            const int64_t o0 = r * pitch + t, o1 = o0 + kLanes * pitch;
            double a0 = a[o0], a1 = a[o1], v0[NB], v1[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                v0[i] = bp[i][o0];
                v1[i] = bp[i][o1];
            }
#pragma unroll
            for (int i = 0; i < NB; ++i) acc[i] = fma(a0, v0[i], acc[i]);
#pragma unroll
            for (int i = 0; i < NB; ++i) acc[i] = fma(a1, v1[i], acc[i]);
        }
        if (r < r1) {
            const int64_t o = r * pitch + t;
            const double av = a[o];
#pragma unroll
            for (int i = 0; i < NB; ++i) acc[i] = fma(av, bp[i][o], acc[i]);
        }
    }
    double *smz = sm + (size_t)z * kLanes * NB * kCols;
#pragma unroll
    for (int i = 0; i < NB; ++i) smz[(lane * NB + i) * kCols + threadIdx.x] = acc[i];
    __syncthreads();
    // lane l of each chunk sums vector i = l, l + 16, ... over the lanes in fixed order
    if (t < n_tl && c < chunks)
        for (int i = lane; i < NB; i += kLanes) {
            double s = 0.0;
#pragma unroll
            for (int y = 0; y < kLanes; ++y) s += smz[(y * NB + i) * kCols + threadIdx.x];
            out[((int64_t)c * NB + i) * n_tl + t] = s;
        }
}

// Stage 2: fixed-order sum over the row chunks, then by mode:
//   dots: out[i][t] = s, and (hacc != null) hacc[i * n_tl + t] += s  (Hessenberg column);
//   norm (nb = 1): n = sqrt(s), out[t] = 1 / n (0 if n = 0: the normalisation scale),
//                  and (hacc != null) hacc[t] = n  (beta or the subdiagonal entry).
// One block of kS2 threads per output (i, t): thread j sums chunks j, j + kS2, ... in order,
// then a fixed shared-memory tree (the order depends on the chunk count only).
constexpr int kS2 = 128;

__global__ void __launch_bounds__(kS2) dots_stage2(const double *__restrict__ part, int chunks, int nb, int n_tl,
                                                   double *__restrict__ out, double *__restrict__ hacc, int norm) {
    __shared__ double red[kS2];
    const int i = blockIdx.x / n_tl, t = blockIdx.x % n_tl;
    double s = 0.0;
    for (int c = threadIdx.x; c < chunks; c += kS2) s += part[((int64_t)c * nb + i) * n_tl + t];
    red[threadIdx.x] = s;
    __syncthreads();
#pragma unroll
    for (int w = kS2 / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    s = red[0];
    if (norm) {
        const double n = sqrt(s);
        out[t] = n > 0.0 ? 1.0 / n : 0.0;
        if (hacc) hacc[t] = n;
    } else {
        out[(int64_t)i * n_tl + t] = s;
        if (hacc) hacc[(int64_t)i * n_tl + t] += s;
    }
}

// Per time step t: y = argmin || beta e1 - H y || for the (k+1) x k upper Hessenberg H of
// step t (entry (i, j) at H[(i + j (k+1)) n_tl + t]) by Givens rotations, then back
// substitution; zero pivots (breakdown) give zero coefficients.  y[j * n_tl + t].
__global__ void lsq_kernel(const double *__restrict__ H, const double *__restrict__ beta, int k, int n_tl,
                           double *__restrict__ y) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tl) return;
    const int ld = k + 1;
    double h[(kMaxVec) * (kMaxVec - 1)], g[kMaxVec], yy[kMaxVec - 1];
    for (int e = 0; e < ld * k; ++e) h[e] = H[(int64_t)e * n_tl + t];
    for (int i = 0; i <= k; ++i) g[i] = 0.0;
    g[0] = beta[t];
    for (int j = 0; j < k; ++j) {
        const double a = h[j + j * ld], b = h[j + 1 + j * ld];
        const double rr = hypot(a, b);
        if (rr == 0.0) continue;
        const double c = a / rr, sn = b / rr;
        for (int jj = j; jj < k; ++jj) {
            const double u = h[j + jj * ld], v = h[j + 1 + jj * ld];
            h[j + jj * ld] = c * u + sn * v;
            h[j + 1 + jj * ld] = -sn * u + c * v;
        }
        const double gu = g[j], gv = g[j + 1];
        g[j] = c * gu + sn * gv;
        g[j + 1] = -sn * gu + c * gv;
    }
    for (int j = k - 1; j >= 0; --j) {
        double v = g[j];
        for (int jj = j + 1; jj < k; ++jj) v -= h[j + jj * ld] * yy[jj];
        const double d = h[j + j * ld];
        yy[j] = (fabs(d) > 1e-300) ? v / d : 0.0;
    }
    for (int j = 0; j < k; ++j) y[(int64_t)j * n_tl + t] = yy[j];
}

// dst[row][t] = scale[t] * (base[row][t] + sign * sum_i coef[i][t] * b_i[row][boff + t])
// (scale == nullptr: 1; base may alias dst); rows of dst, base and the b_i at their own
// pitches (full panel or compact basis); dst2 (optional): a second copy of the result.
template <int NB, int kCols>
__global__ void __launch_bounds__(kThr)
    combine_kernel(double *dst, const double *base, const double *const *__restrict__ b, int boff,
                   const double *__restrict__ coef, double sign, const double *__restrict__ scale, int64_t rows,
                   GmresPitch pt, int n_tl, double *dst2) {
    const int t = blockIdx.x * kCols + threadIdx.x;
    if (t >= n_tl) return;
    double c[NB > 0 ? NB : 1];
    const double *bp[NB > 0 ? NB : 1];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        c[i] = sign * coef[(int64_t)i * n_tl + t];
        bp[i] = b[i] + boff;
    }
    const double sc = scale ? scale[t] : 1.0;
#pragma unroll 2
    for (int64_t r = blockIdx.y * (int64_t)blockDim.y + threadIdx.y; r < rows; r += (int64_t)gridDim.y * blockDim.y) {
        const int64_t ov = r * pt.v + t;
        double v = base[r * pt.base + t];
#pragma unroll
        for (int i = 0; i < NB; ++i) v = fma(c[i], bp[i][ov], v);
        v = sc * v;
        dst[r * pt.dst + t] = v;
        if (dst2) dst2[r * pt.dst2 + t] = v;
    }
}

}  // namespace

int gmres_max_vectors() { return kMaxVec; }

cudaError_t gmres_lsq(const double *H, const double *beta, int k, int n_tl, double *y, cudaStream_t st) {
    if (k < 1 || k > kMaxVec - 1) return cudaErrorInvalidValue;
    lsq_kernel<<<(n_tl + 127) / 128, 128, 0, st>>>(H, beta, k, n_tl, y);
    return cudaGetLastError();
}

int cols_for(int n_tl) { return n_tl > 16 ? 64 : n_tl > 8 ? 16 : n_tl > 2 ? 8 : 2; }
int dots_cols_for(int n_tl) { return n_tl > 16 ? 32 : n_tl > 8 ? 16 : n_tl > 2 ? 8 : 2; }

template <int NB, int C>
void launch_dots1(dim3 g1, size_t sh, cudaStream_t st, const double *a, const double *const *b, int boff,
                  int64_t rows, int64_t pitch, int n_tl, int64_t chunk, int chunks, double *out) {
    static bool attr = false;   // > 48 KB of partials for the widest shapes
    if (!attr) {
        cudaFuncSetAttribute(dots_stage1<NB, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             DotsShape<C>::kThreads * kMaxVec * (int)sizeof(double));
        attr = true;
    }
    dots_stage1<NB, C><<<g1, dim3(C, DotsShape<C>::kThreads / C), sh, st>>>(a, b, boff, rows, pitch, n_tl, chunk,
                                                                            chunks, out);
}

int64_t gmres_dots_scratch(int64_t rows, int n_tl, int nb, int64_t *chunk, int *chunks) {
    // ~2048 row chunks of 16 lanes whatever the window width (the summation order depends
    // on it only): enough independent rows in flight for the narrow windows of the wavefront
    (void)n_tl;
    int64_t ch = (rows + 2047) / 2048;
    if (ch < 64) ch = 64;
    *chunk = ch;
    *chunks = (int)((rows + ch - 1) / ch);
    return (int64_t)(*chunks) * nb * n_tl;
}

cudaError_t gmres_dots(const double *a, const double *const *b_dev, int boff, int nb, int64_t rows, int64_t pitch,
                       int n_tl, double *scratch, double *out, double *hacc, bool norm, cudaStream_t st) {
    if (norm && nb != 1) return cudaErrorInvalidValue;
    if (nb < 1 || nb > kMaxVec) return cudaErrorInvalidValue;
    int64_t chunk;
    int chunks;
    gmres_dots_scratch(rows, n_tl, nb, &chunk, &chunks);
    const int cols = dots_cols_for(n_tl);
    const int thr = cols * kLanes >= kThr ? cols * kLanes : kThr, cpb = thr / (cols * kLanes);
    const dim3 g1((n_tl + cols - 1) / cols, (chunks + cpb - 1) / cpb);
    const size_t sh = (size_t)thr * nb * sizeof(double);
    switch (nb * 100 + cols) {
#define BIOT_D1(N, C) case N * 100 + C: launch_dots1<N, C>(g1, sh, st, a, b_dev, boff, rows, pitch, n_tl, chunk, chunks, scratch); break;
#define BIOT_D(N) BIOT_D1(N, 32) BIOT_D1(N, 16) BIOT_D1(N, 8) BIOT_D1(N, 2)
        BIOT_D(1) BIOT_D(2) BIOT_D(3) BIOT_D(4) BIOT_D(5) BIOT_D(6) BIOT_D(7) BIOT_D(8) BIOT_D(9)
        BIOT_D(10) BIOT_D(11) BIOT_D(12) BIOT_D(13) BIOT_D(14) BIOT_D(15) BIOT_D(16) BIOT_D(17)
#undef BIOT_D
#undef BIOT_D1
    }
    const int64_t n = (int64_t)nb * n_tl;
    dots_stage2<<<(int)n, kS2, 0, st>>>(scratch, chunks, nb, n_tl, out, hacc, norm ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t gmres_combine(double *dst, const double *base, const double *const *b_dev, int boff, const double *coef,
                          int nb, double sign, const double *scale, int64_t rows, GmresPitch pitch, int n_tl,
                          cudaStream_t st, double *dst2) {
    if (nb < 0 || nb > kMaxVec) return cudaErrorInvalidValue;
    const int cols = cols_for(n_tl), ry = kThr / cols;
    const int gy = (int)((rows + ry - 1) / ry < 4096 ? (rows + ry - 1) / ry : 4096);
    const dim3 g2((n_tl + cols - 1) / cols, gy), b2(cols, ry);
    switch (nb * 100 + cols) {
#define BIOT_C1(N, C) case N * 100 + C: combine_kernel<N, C><<<g2, b2, 0, st>>>(dst, base, b_dev, boff, coef, sign, scale, rows, pitch, n_tl, dst2); break;
#define BIOT_C(N) BIOT_C1(N, 64) BIOT_C1(N, 16) BIOT_C1(N, 8) BIOT_C1(N, 2)
        BIOT_C(0) BIOT_C(1) BIOT_C(2) BIOT_C(3) BIOT_C(4) BIOT_C(5) BIOT_C(6) BIOT_C(7) BIOT_C(8) BIOT_C(9)
        BIOT_C(10) BIOT_C(11) BIOT_C(12) BIOT_C(13) BIOT_C(14) BIOT_C(15) BIOT_C(16) BIOT_C(17)
#undef BIOT_C
#undef BIOT_C1
    }
    return cudaGetLastError();
}

}  // namespace biot
