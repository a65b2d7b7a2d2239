// Register-blocked sweep for structured simplicial meshes (the BASELINE.json
// configs): same arithmetic as sweep_kernels.cu (one outer iteration of the
// Jacobi-in-time inverted scheme, with the block
// preconditioner of L238-262 fused), specialised to the two stencils whose
// BDIA offsets decompose into a few runs of consecutive offsets:
//
//   2D right triangles (BL->TR diagonal), W = n+1:
//       {-W + (-1,0)}, {0 + (-1,0,1)}, {W + (0,1)}                 (7 slots)
//   3D Kuhn tetrahedra, W = n+1, V = W^2:
//       {-W-V + (-1,0)}, {-V + (-1,0)}, {-W + (-1,0)}, {0 + (-1,0,1)},
//       {W + (0,1)}, {V + (0,1)}, {W+V + (0,1)}                    (15 slots)
//
// A warp owns R consecutive row nodes i0..i0+R-1 and a chunk of 32*T time steps
// (lane = T consecutive steps).  It walks each run's columns once; a gathered
// column x_j(t..t+T-1) (all d+1 components) feeds every row r of the block with
// j - (i0 + r) in the run: per R rows it loads (2D) 3R+4 columns instead of 7R,
// (3D) 7R+8 instead of 15R.  Coefficient blocks are read with warp-uniform
// 16-B loads.  Accumulation order per output = ascending column offset, the same
// in the main loop and in lane 0's recomputation of q(t0-1) (bitwise identical).
#include "sweep_kernels.cuh"

namespace biot {

namespace {

template <int D>
struct Stencil;

template <>
struct Stencil<2> {
    static constexpr int NG = 3;
    __host__ __device__ static constexpr int amin(int g) { return g == 2 ? 0 : -1; }
    __host__ __device__ static constexpr int amax(int g) { return g == 0 ? 0 : 1; }
};

template <>
struct Stencil<3> {
    static constexpr int NG = 7;
    __host__ __device__ static constexpr int amin(int g) { return g <= 3 ? -1 : 0; }
    __host__ __device__ static constexpr int amax(int g) { return g >= 3 ? 1 : 0; }
};

template <int D, int R, int T>
__device__ __forceinline__ void group_update(const StencilArgs &a, int64_t i0, int t0, int lane,
                                             const double (&sv)[T], double (&nu)[T], double (&npn)[T]) {
    using St = Stencil<D>;
    constexpr int NC = D + 1;
    constexpr int WP = StencilArgs::kBlockPitch<D>;   // padded block width (doubles)
    constexpr int S = D == 2 ? 7 : 15;
    const int64_t P = a.pitch;

    double acc[R][NC][T], q[R][T];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
            q[r][tt] = 0.0;
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[r][c][tt] = 0.0;
        }

#pragma unroll
    for (int g = 0; g < St::NG; ++g) {
        const double *__restrict__ gcol = a.x + (i0 + a.gbase[g]) * NC * P + t0;
#pragma unroll
        for (int m = St::amin(g); m <= R - 1 + St::amax(g); ++m) {
            double v[NC][T];
#pragma unroll
            for (int cc = 0; cc < NC; ++cc) {
                const double *src = gcol + ((int64_t)m * NC + cc) * P;
#pragma unroll
                for (int h = 0; h < T; h += 2) {
                    const double2 w2 = __ldg(reinterpret_cast<const double2 *>(src + h));
                    v[cc][h] = w2.x;
                    v[cc][h + 1] = w2.y;
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int off = m - r;
                if (off < St::amin(g) || off > St::amax(g)) continue;
                const int s = a.slot[g][off - St::amin(g)];
                const double *__restrict__ bp = a.blk + ((i0 + r) * S + s) * WP;
                double cf[WP];
#pragma unroll
                for (int k = 0; k < WP; k += 2) {
                    const double2 w2 = __ldg(reinterpret_cast<const double2 *>(bp + k));
                    cf[k] = w2.x;
                    cf[k + 1] = w2.y;
                }
#pragma unroll
                for (int cc = 0; cc < NC; ++cc) {
#pragma unroll
                    for (int c = 0; c < NC; ++c)
#pragma unroll
                        for (int tt = 0; tt < T; ++tt)
                            acc[r][c][tt] = fma(cf[c * NC + cc], v[cc][tt], acc[r][c][tt]);
                    const double qc = (cc < D) ? cf[D * NC + cc] : cf[NC * NC];
#pragma unroll
                    for (int tt = 0; tt < T; ++tt) q[r][tt] = fma(qc, v[cc][tt], q[r][tt]);
                }
            }
        }
    }

    // previous-step coupling of each lane's first step
    double qprev[R];
#pragma unroll
    for (int r = 0; r < R; ++r) qprev[r] = __shfl_up_sync(0xffffffffu, q[r][T - 1], 1);
    if (lane == 0) {
        const bool use_ghost = (t0 == 0);
        double qg[R];
#pragma unroll
        for (int r = 0; r < R; ++r) qg[r] = 0.0;
#pragma unroll
        for (int g = 0; g < St::NG; ++g) {
#pragma unroll
            for (int m = St::amin(g); m <= R - 1 + St::amax(g); ++m) {
                const int64_t j = i0 + a.gbase[g] + m;
                double v1[NC];
#pragma unroll
                for (int cc = 0; cc < NC; ++cc)
                    v1[cc] = use_ghost ? __ldg(a.ghost + j * NC + cc) : __ldg(a.x + (j * NC + cc) * P + t0 - 1);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int off = m - r;
                    if (off < St::amin(g) || off > St::amax(g)) continue;
                    const int s = a.slot[g][off - St::amin(g)];
                    const double *__restrict__ bp = a.blk + ((i0 + r) * S + s) * WP;
#pragma unroll
                    for (int cc = 0; cc < NC; ++cc) {
                        const double qc = (cc < D) ? __ldg(bp + D * NC + cc) : __ldg(bp + NC * NC);
                        qg[r] = fma(qc, v1[cc], qg[r]);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) qprev[r] = qg[r];
    }

    const int n_tl = a.n_tl;
    const int mode = a.mode;
    const double omega = a.omega;
    const bool full = (t0 + T <= n_tl);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t i = i0 + r;
        double F[NC], Dv[NC], xs[NC][T];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            F[c] = __ldg(a.load + i * NC + c);
            Dv[c] = __ldg(a.dinv + i * NC + c);
            const double *src = a.x + (i * NC + c) * P + t0;
#pragma unroll
            for (int h = 0; h < T; h += 2) {
                const double2 w2 = __ldg(reinterpret_cast<const double2 *>(src + h));
                xs[c][h] = w2.x;
                xs[c][h + 1] = w2.y;
            }
        }
        double outx[NC][T], outz[NC][T];
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
            const double qp = (tt == 0) ? qprev[r] : q[r][tt - 1];
            double rr[NC];
#pragma unroll
            for (int c = 0; c < D; ++c) rr[c] = sv[tt] * F[c] - acc[r][c][tt];
            rr[D] = (sv[tt] * F[D] + qp) - acc[r][D][tt];
            double su = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) su = fma(rr[c], rr[c], su);
            nu[tt] += su;
            npn[tt] = fma(rr[D], rr[D], npn[tt]);
            double z[NC];
#pragma unroll
            for (int c = 0; c < D; ++c) z[c] = Dv[c] * rr[c];
            z[D] = -(Dv[D] * rr[D]);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                outx[c][tt] = fma(omega, z[c], xs[c][tt]);
                outz[c][tt] = (c < D) ? z[c] : rr[D];
            }
        }
        if (mode == MODE_RESIDUAL) continue;
        const int ncw = (mode == MODE_UPDATE_P2) ? NC : D;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (c >= ncw) break;
            double *dst = a.xn + (i * NC + c) * P + t0;
            if (full) {
#pragma unroll
                for (int h = 0; h < T; h += 2)
                    *reinterpret_cast<double2 *>(dst + h) = make_double2(outx[c][h], outx[c][h + 1]);
            } else {
#pragma unroll
                for (int tt = 0; tt < T; ++tt)
                    if (t0 + tt < n_tl) dst[tt] = outx[c][tt];
            }
        }
        if (mode == MODE_P1_PASS1) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                double *dst = a.zbuf + (i * NC + c) * P + t0;
                if (full) {
#pragma unroll
                    for (int h = 0; h < T; h += 2)
                        *reinterpret_cast<double2 *>(dst + h) = make_double2(outz[c][h], outz[c][h + 1]);
                } else {
#pragma unroll
                    for (int tt = 0; tt < T; ++tt)
                        if (t0 + tt < n_tl) dst[tt] = outz[c][tt];
                }
            }
        }
        if (a.sendbuf && i < a.n_nodes) {
            const int tl = n_tl - 1 - t0;
            if (tl >= 0 && tl < T) {
#pragma unroll
                for (int tt = 0; tt < T; ++tt)
                    if (tt == tl)
#pragma unroll
                        for (int c = 0; c < NC; ++c)
                            if (c < ncw) a.sendbuf[i * NC + c] = outx[c][tt];
            }
        }
    }
}

// Occupancy target: 2 CTAs (16 warps) per SM where the accumulators allow it.
template <int D, int R, int T>
constexpr int stencil_min_blocks() { return (R * (D + 2) * T <= 32) ? 2 : 1; }

template <int D, int R, int T>
__global__ void __launch_bounds__(kThreads, stencil_min_blocks<D, R, T>()) stencil_kernel(const StencilArgs a) {
    extern __shared__ double red[];
    constexpr int CH = 32 * T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tw = a.tw, nwp = (kThreads / 32) / tw;
    const int cw = warp % tw, nw = warp / tw;
    const int n_chunks = (a.n_tl + CH - 1) / CH;
    const int n_tlp = n_chunks * CH;
    const int64_t n_groups = (a.n_nodes + R - 1) / R;

    for (int chunk = cw; chunk < n_chunks; chunk += tw) {
        const int t0 = chunk * CH + lane * T;
        double nu[T], npn[T], sv[T];
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
            nu[tt] = 0.0;
            npn[tt] = 0.0;
            sv[tt] = (t0 + tt < a.n_tl) ? a.s[t0 + tt] : 0.0;
        }
        for (int64_t ng = (int64_t)blockIdx.x * nwp + nw; ng < n_groups; ng += (int64_t)gridDim.x * nwp)
            group_update<D, R, T>(a, ng * R, t0, lane, sv, nu, npn);
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
            red[((int64_t)nw * n_tlp + t0 + tt) * 2 + 0] = nu[tt];
            red[((int64_t)nw * n_tlp + t0 + tt) * 2 + 1] = npn[tt];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.n_tl; t += kThreads) {
        double su = 0.0, sp = 0.0;
        for (int w = 0; w < nwp; ++w) {
            su += red[((int64_t)w * n_tlp + t) * 2 + 0];
            sp += red[((int64_t)w * n_tlp + t) * 2 + 1];
        }
        a.partial[((int64_t)blockIdx.x * a.n_tl + t) * 2 + 0] = su;
        a.partial[((int64_t)blockIdx.x * a.n_tl + t) * 2 + 1] = sp;
    }
}

using StencilFn = void (*)(const StencilArgs);

StencilFn pick_stencil(int dim, int R, int T) {
#define BIOT_SCASE(D_, R_, T_) \
    if (dim == D_ && R == R_ && T == T_) return stencil_kernel<D_, R_, T_>;
    BIOT_SCASE(2, 2, 2)
    BIOT_SCASE(2, 2, 4)
    BIOT_SCASE(2, 4, 2)
    BIOT_SCASE(2, 4, 4)
    BIOT_SCASE(3, 2, 2)
    BIOT_SCASE(3, 2, 4)
    BIOT_SCASE(3, 4, 2)
#undef BIOT_SCASE
    return nullptr;
}

}  // namespace

bool stencil_supported(int dim, int R, int T) { return pick_stencil(dim, R, T) != nullptr; }

cudaError_t stencil_shape(int dim, int R, int T, int device, LaunchShape *out) {
    StencilFn f = pick_stencil(dim, R, T);
    if (!f) return cudaErrorInvalidValue;
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    if (out->smem > 48 * 1024) {
        e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)out->smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kThreads, out->smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    return cudaSuccess;
}

cudaError_t launch_stencil(int dim, int R, int T, const StencilArgs &a, const LaunchShape &sh,
                           cudaStream_t st) {
    StencilFn f = pick_stencil(dim, R, T);
    if (!f) return cudaErrorInvalidValue;
    f<<<sh.grid, kThreads, sh.smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace biot
