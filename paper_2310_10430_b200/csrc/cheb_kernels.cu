// Chebyshev inner inverses for the block preconditioner P~2 (SURVEY §8(f) NEXT-1,
// reading R22): z = P~2^{-1} r with A^{-1} and S~p^{-1} (PAPER.md eq. p2)
// each replaced by m steps of Chebyshev iteration preconditioned by the diagonal, on
// [lambda_max / alpha, lambda_max] of D^{-1} M (Gershgorin lambda_max per block).
//
// The outer iteration's residual r (with the previous-step coupling and the norms) comes
// from the main kernel in its P~1 first-pass mode, which leaves Z = (D_A^{-1} r_u, r_p)
// in a panel.  The Chebyshev recurrence then runs on the scaled residual s = D^{-1} r
// (s_u = Z_u, s_p = D_S^{-1} Z_p), all time steps at once (the inner operators have no
// time coupling):
//     d_0 = s_0 / theta,  y_1 = d_0,
//     s_k = s_{k-1} - D^{-1} M d_{k-1},
//     d_k = rho_k rho_{k-1} d_{k-1} + (2 rho_k / delta) s_k,   y_{k+1} = y_k + d_k,
// per block (M = A for the displacement rows, M = S~p = -AA_pp for the pressure rows,
// each with its own theta, delta, rho), and finally x^{k+1} = x^k + omega (y_u, -y_p).
// Panels are time-contiguous rows as everywhere: p[(node*nc + c)*pitch + t].
#include <cuda_runtime.h>
#include <cstdint>

#include "node_update.cuh"
#include "sweep_kernels.cuh"

namespace biot {

namespace {

using namespace dev;

constexpr int kCThreads = 256;

// Elementwise start: s = D^{-1} r (in place on the Z panel: only the pressure rows
// change), d_0 = s / theta; with m = 1 directly x^{k+1} = x + omega (d_u, -d_p).
__global__ void __launch_bounds__(kCThreads) cheb_init_kernel(const ChebArgs a) {
    const int nc = a.nc, d = nc - 1;
    const int64_t n_rows = a.n_nodes * nc;
    const int64_t tot = n_rows * a.n_tl;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < tot;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = k / a.n_tl;
        const int t = (int)(k % a.n_tl);
        const int c = (int)(row % nc);
        const int64_t o = row * a.pitch + t;
        const bool p = c == d;
        if (!(a.rows & (p ? 2 : 1))) continue;
        const double sv = p ? __ldg(a.dinv + row) * a.s[o] : a.s[o];
        const double dv = sv * (p ? a.inv_theta_p : a.inv_theta_u);
        if (a.last) {
            const double xv = a.x[o] + a.omega * (p ? a.p_sign * dv : dv);
            a.xn[o] = xv;
            if (a.sendbuf && t == a.n_tl - 1) a.sendbuf[row] = xv;
        } else {
            if (p) a.s[o] = sv;
            a.dn[o] = dv;
        }
    }
}

// One Chebyshev step for node i over the lane's kT steps: M d from the operator blocks
// (displacement-displacement entries and -AA_pp only: the inner operators are the
// diagonal blocks of P~2), then the recurrence above.
template <int D, int S, bool ELL>
__global__ void __launch_bounds__(kCThreads) cheb_step_kernel(const ChebArgs a) {
    constexpr int NC = D + 1;
    constexpr int W = (NC * NC + 2) / 2 * 2;
    const int lane = threadIdx.x & 31;
    const int n_chunks = (a.n_tl + kChunk - 1) / kChunk;
    const int64_t P = a.pitch;
    const int64_t n_warps = a.n_nodes * n_chunks;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
#ifdef BIOT_CHEB_NODE_MAJOR
        const int64_t i = w / n_chunks;
        const int t0 = (int)(w % n_chunks) * kChunk + lane * kT;
#else
        // chunk-major: the warps of a block (and of neighbouring blocks) take consecutive
        // nodes of one chunk, so the gathered neighbour columns are shared in L1 / L2
        const int64_t i = w % a.n_nodes;
        const int t0 = (int)(w / a.n_nodes) * kChunk + lane * kT;
#endif
        if (t0 >= a.n_tl) continue;
        const double *__restrict__ bp = a.blk + i * (int64_t)(S * W);
        double acc[NC][kT];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int tt = 0; tt < kT; ++tt) acc[c][tt] = 0.0;
        const bool first = a.first != 0;
        const double *__restrict__ dsrc = first ? a.s : a.d;
        for (int s = 0; s < S; ++s) {
            const int64_t j = column<S, ELL>(a.cols, a.off, i, s);
            const double *__restrict__ dj = dsrc + j * NC * P + t0;
            double v[NC][kT];
#pragma unroll
            for (int cc = 0; cc < NC; ++cc) {
                const double2 v01 = __ldg(reinterpret_cast<const double2 *>(dj + cc * P));
                const double2 v23 = __ldg(reinterpret_cast<const double2 *>(dj + cc * P + 2));
                v[cc][0] = v01.x;
                v[cc][1] = v01.y;
                v[cc][2] = v23.x;
                v[cc][3] = v23.y;
            }
            if (first) {   // d_0 = s_0 / theta, s_0 = (Z_u, D_S^{-1} Z_p), as cheb_init_kernel
                const double dsj = __ldg(a.dinv + j * NC + D);
#pragma unroll
                for (int tt = 0; tt < kT; ++tt) {
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) v[cc][tt] = v[cc][tt] * a.inv_theta_u;
                    v[D][tt] = (dsj * v[D][tt]) * a.inv_theta_p;
                }
            }
#pragma unroll
            for (int c = 0; c < D; ++c)
#pragma unroll
                for (int cc = 0; cc < D; ++cc) {
                    const double cf = __ldg(bp + s * W + c * NC + cc);
#pragma unroll
                    for (int tt = 0; tt < kT; ++tt) acc[c][tt] = fma(cf, v[cc][tt], acc[c][tt]);
                }
            const double cpp = -__ldg(bp + s * W + D * NC + D);   // S~p = -AA_pp
#pragma unroll
            for (int tt = 0; tt < kT; ++tt) acc[D][tt] = fma(cpp, v[D][tt], acc[D][tt]);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int64_t o = (i * NC + c) * P + t0;
            const bool p = c == D;
            if (!(a.rows & (p ? 2 : 1))) continue;
            const double dv = __ldg(a.dinv + i * NC + c);
            const double c1 = p ? a.c1_p : a.c1_u, c2 = p ? a.c2_p : a.c2_u;
#pragma unroll
            for (int tt = 0; tt < kT; ++tt) {
                if (t0 + tt >= a.n_tl) break;
                double so, dold;
                if (first) {   // the start of this node, as cheb_init_kernel computes it
                    so = p ? dv * a.s[o + tt] : a.s[o + tt];
                    dold = so * (p ? a.inv_theta_p : a.inv_theta_u);
                } else {
                    so = a.s[o + tt];
                    dold = a.d[o + tt];
                }
                const double sn = so - dv * acc[c][tt];
                const double dn = fma(c1, dold, c2 * sn);
                const double yn = (a.y ? a.y[o + tt] : dold) + dn;   // y_1 = d_0
                if (a.last) {
                    const double xv = fma(a.omega, p ? a.p_sign * yn : yn, a.x[o + tt]);
                    a.xn[o + tt] = xv;
                    if (a.sendbuf && t0 + tt == a.n_tl - 1) a.sendbuf[i * NC + c] = xv;
                } else {
                    (a.sn ? a.sn : a.s)[o + tt] = sn;
                    a.dn[o + tt] = dn;
                    a.yn[o + tt] = yn;
                }
            }
        }
    }
}

// P~1 between the blocks (PAPER.md eq. p1: z_p = S~p^{-1} (B^T z_u - r_p)): the right-hand
// side of the pressure block from z_u (all neighbours), its Chebyshev start, and the
// displacement update x_u + omega z_u of the node.
template <int D, int S, bool ELL>
__global__ void __launch_bounds__(kCThreads) cheb_p1_rhs_kernel(const ChebArgs a) {
    constexpr int NC = D + 1;
    constexpr int W = (NC * NC + 2) / 2 * 2;
    const int lane = threadIdx.x & 31;
    const int n_chunks = (a.n_tl + kChunk - 1) / kChunk;
    const int64_t P = a.pitch;
    const int64_t n_warps = a.n_nodes * n_chunks;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
#ifdef BIOT_CHEB_NODE_MAJOR
        const int64_t i = w / n_chunks;
        const int t0 = (int)(w % n_chunks) * kChunk + lane * kT;
#else
        // chunk-major: the warps of a block (and of neighbouring blocks) take consecutive
        // nodes of one chunk, so the gathered neighbour columns are shared in L1 / L2
        const int64_t i = w % a.n_nodes;
        const int t0 = (int)(w / a.n_nodes) * kChunk + lane * kT;
#endif
        if (t0 >= a.n_tl) continue;
        const double *__restrict__ bp = a.blk + i * (int64_t)(S * W);
        double bt[kT] = {0.0, 0.0, 0.0, 0.0};
        for (int s = 0; s < S; ++s) {
            const int64_t j = column<S, ELL>(a.cols, a.off, i, s);
#pragma unroll
            for (int cc = 0; cc < D; ++cc) {
                const double cf = __ldg(bp + s * W + D * NC + cc);
                const double *src = a.zu + (j * NC + cc) * P + t0;
                const double2 v01 = __ldg(reinterpret_cast<const double2 *>(src));
                const double2 v23 = __ldg(reinterpret_cast<const double2 *>(src + 2));
                bt[0] = fma(cf, v01.x, bt[0]);
                bt[1] = fma(cf, v01.y, bt[1]);
                bt[2] = fma(cf, v23.x, bt[2]);
                bt[3] = fma(cf, v23.y, bt[3]);
            }
        }
        const double dvp = __ldg(a.dinv + i * NC + D);
        const int64_t op = (i * NC + D) * P + t0;
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
            if (t0 + tt >= a.n_tl) break;
            const double sp = dvp * (bt[tt] - a.s[op + tt]);   // s holds r_p here
            const double dp = sp * a.inv_theta_p;
            if (a.last) {
                const double xv = fma(a.omega, dp, a.x[op + tt]);
                a.xn[op + tt] = xv;
                if (a.sendbuf && t0 + tt == a.n_tl - 1) a.sendbuf[i * NC + D] = xv;
            } else {
                a.s[op + tt] = sp;
                a.dn[op + tt] = dp;
            }
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const int64_t o = (i * NC + c) * P + t0;
#pragma unroll
            for (int tt = 0; tt < kT; ++tt) {
                if (t0 + tt >= a.n_tl) break;
                const double xv = fma(a.omega, a.zu[o + tt], a.x[o + tt]);
                a.xn[o + tt] = xv;
                if (a.sendbuf && t0 + tt == a.n_tl - 1) a.sendbuf[i * NC + c] = xv;
            }
        }
    }
}

using StepFn = void (*)(const ChebArgs);

StepFn pick_step(int dim, int path, int S, bool rhs = false) {
#define BIOT_CS(D_, S_, ELL_) \
    if (dim == D_ && S == S_ && (path == 2) == ELL_) \
        return rhs ? cheb_p1_rhs_kernel<D_, S_, ELL_> : cheb_step_kernel<D_, S_, ELL_>;
    BIOT_CS(2, 7, false)
    BIOT_CS(3, 15, false)
    BIOT_CS(2, 8, true)
    BIOT_CS(2, 16, true)
    BIOT_CS(2, 32, true)
    BIOT_CS(3, 8, true)
    BIOT_CS(3, 16, true)
    BIOT_CS(3, 32, true)
#undef BIOT_CS
    return nullptr;
}

int grid_for(int64_t work, int per_block) {
    const int64_t g = (work + per_block - 1) / per_block;
    return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

cudaError_t launch_cheb_init(const ChebArgs &a, cudaStream_t st) {
    cheb_init_kernel<<<grid_for(a.n_nodes * a.nc * a.n_tl, kCThreads), kCThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_cheb_step(int dim, int path, int n_slots, const ChebArgs &a, cudaStream_t st) {
    StepFn f = pick_step(dim, path, n_slots);
    if (!f) return cudaErrorInvalidValue;
    const int64_t n_chunks = (a.n_tl + kChunk - 1) / kChunk;
    f<<<grid_for(a.n_nodes * n_chunks * 32, kCThreads), kCThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_cheb_p1_rhs(int dim, int path, int n_slots, const ChebArgs &a, cudaStream_t st) {
    StepFn f = pick_step(dim, path, n_slots, true);
    if (!f) return cudaErrorInvalidValue;
    const int64_t n_chunks = (a.n_tl + kChunk - 1) / kChunk;
    f<<<grid_for(a.n_nodes * n_chunks * 32, kCThreads), kCThreads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace biot
