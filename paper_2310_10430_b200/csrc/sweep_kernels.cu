// Hot-path kernels: one outer iteration of the inverted time-stepping scheme
// over all local time steps at once (Algorithm 2, Jacobi in
// time per BASELINE.json), fused with the block preconditioner (L238-262), the
// damped update and the per-step residual-norm reduction.  sm_100a, fp64.
//
// Data layout (HBM): the space-time iterate is a "panel" with one row per
// (node, component) and the local time steps contiguous in the row:
//     x[(i*nc + c)*pitch + t]
// so each operator entry multiplies a contiguous, 16-B-vectorised, coalesced run
// of time steps (lane l of a warp owns steps t0..t0+3, t0 = chunk*128 + 4l).
// The operator is stored as (d+1)x(d+1) node blocks per neighbour slot, read
// with warp-uniform loads (one L1 transaction serves all 32 lanes); every
// gathered x value feeds d+2 FMAs (d+1 block rows + the previous-step row).
//
// Previous-step coupling A' x_{n-1} is fused without reloading x at t-1: each
// lane accumulates q(t) = (A' x_t)_p for its own steps and the output at t uses
// q(t-1), taken from the neighbouring lane by one shuffle; lane 0 recomputes
// q(t0-1) in the same FMA order (bitwise identical), reading the ghost step
// (the last step of the previous time slab, or x_0) when t0 = 0.
#include "sweep_kernels.cuh"
#include "node_update.cuh"

#include <cmath>


namespace biot {

namespace {

using namespace dev;

template <int D, int S, bool ELL, int NL>
__global__ void __launch_bounds__(kThreads, (D == 2 ? 2 : 1)) sweep_kernel(const SweepArgs a) {
    extern __shared__ double red[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tw = a.tw, nwp = (kThreads / 32) / tw;
    const int cw = warp % tw, nw = warp / tw;
    const int n_chunks = (a.n_tl + kChunk - 1) / kChunk;
    const int n_tlp = n_chunks * kChunk;
    const int64_t N = a.n_nodes;
    const int64_t nb = a.node_block;

    for (int chunk = cw; chunk < n_chunks; chunk += tw) {
        const int t0 = chunk * kChunk + lane * kT;
        double nu[kT], npn[kT], sv[NL][kT];
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
            nu[tt] = 0.0;
            npn[tt] = 0.0;
#pragma unroll
            for (int j = 0; j < NL; ++j) sv[j][tt] = (t0 + tt < a.n_tl) ? a.s[j * a.s_pitch + t0 + tt] : 0.0;
        }
        for (int64_t b = blockIdx.x; b * nb < N; b += gridDim.x) {
            const int64_t i_end = min(N, (b + 1) * nb);
            for (int64_t i = b * nb + nw; i < i_end; i += nwp)
                node_update<D, S, ELL, kT, false, NL>(a, i, a.blk + i * (int64_t)(S * block_pitch<D>()), t0,
                                                  lane, sv, nu, npn);
        }
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
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


// P~1 second pass (PAPER.md eq. p1: z_p = S~p^{-1} (B^T z_u - r_p)).
template <int D, int S, bool ELL>
__global__ void __launch_bounds__(kThreads) pass2_kernel(const Pass2Args a) {
    constexpr int NC = D + 1;
    constexpr int W = (NC * NC + 2) / 2 * 2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tw = a.tw, nwp = (kThreads / 32) / tw;
    const int cw = warp % tw, nw = warp / tw;
    const int n_chunks = (a.n_tl + kChunk - 1) / kChunk;
    const int64_t N = a.n_nodes, P = a.pitch, nb = a.node_block;
    const int n_tl = a.n_tl;
    for (int chunk = cw; chunk < n_chunks; chunk += tw) {
        const int t0 = chunk * kChunk + lane * kT;
        for (int64_t b = blockIdx.x; b * nb < N; b += gridDim.x) {
            const int64_t i_end = min(N, (b + 1) * nb);
            for (int64_t i = b * nb + nw; i < i_end; i += nwp) {
                const double *__restrict__ bp = a.blk + i * (int64_t)(S * W);
                double bt[kT] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int64_t j = column<S, ELL>(a.cols, a.off, i, s);
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) {
                        const double cf = __ldg(bp + s * W + D * NC + cc);
                        const double *src = a.zbuf + (j * NC + cc) * P + a.t_off + t0;
                        const double2 v01 = __ldg(reinterpret_cast<const double2 *>(src));
                        const double2 v23 = __ldg(reinterpret_cast<const double2 *>(src + 2));
                        bt[0] = fma(cf, v01.x, bt[0]);
                        bt[1] = fma(cf, v01.y, bt[1]);
                        bt[2] = fma(cf, v23.x, bt[2]);
                        bt[3] = fma(cf, v23.y, bt[3]);
                    }
                }
                const double dv = __ldg(a.dinv + i * NC + D);
                const double *rp = a.zbuf + (i * NC + D) * P + a.t_off + t0;
                const double *xp = a.x + (i * NC + D) * P + a.t_off + t0;
                double *dst = a.xn + (i * NC + D) * P + a.t_off + t0;
#pragma unroll
                for (int tt = 0; tt < kT; ++tt) {
                    if (t0 + tt < n_tl && t0 + tt >= a.t_lo) {
                        const double zp = dv * (bt[tt] - rp[tt]);
                        const double v = a.pure ? zp : fma(a.omega, zp, xp[tt]);
                        dst[tt] = v;
                        if (a.sendbuf && t0 + tt == n_tl - 1) a.sendbuf[i * NC + D] = v;
                    }
                }
            }
        }
    }
}

// Deterministic second stage of the norm reduction: fixed split of the groups
// over 8 y-lanes, then a fixed-order sum of the 8 lane totals.
// norms: the output, or -- slot_ctr != null (CUDA-graph replays) -- the residual-history
// ring, slot (*slot_ctr + slot_off) % cap of n_tl x 2 doubles
__global__ void finalize_kernel(const double *__restrict__ partial, int groups, int n_tl,
                                double *__restrict__ norms, int *nonfinite, const int64_t *slot_ctr,
                                int64_t slot_off, int cap) {
    if (slot_ctr) norms += ((*slot_ctr + slot_off) % cap) * (int64_t)n_tl * 2;
    __shared__ double sm[8][32][2];
    const int t = blockIdx.x * 32 + threadIdx.x;
    const int y = threadIdx.y;
    double su = 0.0, sp = 0.0;
    if (t < n_tl) {
        for (int g = y; g < groups; g += 8) {
            su += partial[((int64_t)g * n_tl + t) * 2 + 0];
            sp += partial[((int64_t)g * n_tl + t) * 2 + 1];
        }
    }
    sm[y][threadIdx.x][0] = su;
    sm[y][threadIdx.x][1] = sp;
    __syncthreads();
    if (y == 0 && t < n_tl) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < 8; ++k) {
            a += sm[k][threadIdx.x][0];
            b += sm[k][threadIdx.x][1];
        }
        a = sqrt(a);
        b = sqrt(b);
        norms[t * 2 + 0] = a;
        norms[t * 2 + 1] = b;
        if (!isfinite(a) || !isfinite(b)) atomicOr(nonfinite, 1);
    }
}

// First stage for many groups: block column by sums groups [by*kGch, (by+1)*kGch)
// (fixed split over 8 y-lanes, then a fixed-order sum of the lane totals).
constexpr int kGch = 128;
constexpr int kGchT = 32;   // groups per block of the one-launch finalize (4 per y-lane)
__global__ void finalize_stage1_kernel(const double *__restrict__ partial, int groups, int n_tl,
                                       double *__restrict__ out) {
    __shared__ double sm[8][32][2];
    const int t = blockIdx.x * 32 + threadIdx.x;
    const int y = threadIdx.y;
    const int g0 = blockIdx.y * kGch, g1 = min(groups, g0 + kGch);
    double su = 0.0, sp = 0.0;
    if (t < n_tl) {
        for (int g = g0 + y; g < g1; g += 8) {
            su += partial[((int64_t)g * n_tl + t) * 2 + 0];
            sp += partial[((int64_t)g * n_tl + t) * 2 + 1];
        }
    }
    sm[y][threadIdx.x][0] = su;
    sm[y][threadIdx.x][1] = sp;
    __syncthreads();
    if (y == 0 && t < n_tl) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < 8; ++k) {
            a += sm[k][threadIdx.x][0];
            b += sm[k][threadIdx.x][1];
        }
        out[((int64_t)blockIdx.y * n_tl + t) * 2 + 0] = a;
        out[((int64_t)blockIdx.y * n_tl + t) * 2 + 1] = b;
    }
}

// Second stage for a Gauss-Seidel wave: fixed-order sum as finalize_kernel, written to
// the history slot of each step's iteration.
__global__ void finalize_wave_kernel(const double *__restrict__ partial, int groups, int len, int lo, int t_first,
                                     int64_t k0, int cap, int n_tl, double *__restrict__ hist, int *nonfinite) {
    __shared__ double sm[8][32][2];
    const int t = blockIdx.x * 32 + threadIdx.x;
    const int y = threadIdx.y;
    double su = 0.0, sp = 0.0;
    if (t < len) {
        for (int g = y; g < groups; g += 8) {
            su += partial[((int64_t)g * len + t) * 2 + 0];
            sp += partial[((int64_t)g * len + t) * 2 + 1];
        }
    }
    sm[y][threadIdx.x][0] = su;
    sm[y][threadIdx.x][1] = sp;
    __syncthreads();
    if (y == 0 && t < len) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < 8; ++k) {
            a += sm[k][threadIdx.x][0];
            b += sm[k][threadIdx.x][1];
        }
        a = sqrt(a);
        b = sqrt(b);
        const int tg = lo + t;
        if (tg >= t_first) {   // steps below t_first were computed for alignment only
            double *o = hist + (((k0 - tg) % cap) * (int64_t)n_tl + tg) * 2;   // [slot][t][2]
            o[0] = a;
            o[1] = b;
            if (!isfinite(a) || !isfinite(b)) atomicOr(nonfinite, 1);
        }
    }
}

using SweepFn = void (*)(const SweepArgs);
using Pass2Fn = void (*)(const Pass2Args);

bool pick(int dim, int path, int S, bool ml, SweepFn *sf, Pass2Fn *pf) {
#define BIOT_CASE(D_, S_, ELL_)              \
    if (dim == D_ && S == S_ && (path == 2) == ELL_) { \
        *sf = ml ? sweep_kernel<D_, S_, ELL_, kMaxLoads> : sweep_kernel<D_, S_, ELL_, 1>; \
        *pf = pass2_kernel<D_, S_, ELL_>;   \
        return true;                          \
    }
    BIOT_CASE(2, 7, false)
    BIOT_CASE(3, 15, false)
    BIOT_CASE(2, 8, true)
    BIOT_CASE(2, 16, true)
    BIOT_CASE(2, 32, true)
    BIOT_CASE(3, 8, true)
    BIOT_CASE(3, 16, true)
    BIOT_CASE(3, 32, true)
#undef BIOT_CASE
    return false;
}

}  // namespace

cudaError_t sweep_shape(int dim, int path, int n_slots, bool ml, int device, LaunchShape *out) {
    SweepFn sf;
    Pass2Fn pf;
    if (!pick(dim, path, n_slots, ml, &sf, &pf)) return cudaErrorInvalidValue;
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const size_t smem = out->smem;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(sf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sf, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    return cudaSuccess;
}

cudaError_t launch_sweep(int dim, int path, int n_slots, const SweepArgs &a, const LaunchShape &sh,
                         cudaStream_t st) {
    SweepFn sf;
    Pass2Fn pf;
    if (!pick(dim, path, n_slots, a.n_load > 1, &sf, &pf)) return cudaErrorInvalidValue;
    sf<<<sh.grid, kThreads, sh.smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pass2(int dim, int path, int n_slots, const Pass2Args &a, int grid,
                         cudaStream_t st) {
    SweepFn sf;
    Pass2Fn pf;
    if (!pick(dim, path, n_slots, false, &sf, &pf)) return cudaErrorInvalidValue;
    pf<<<grid, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_finalize_wave(const double *partial, int groups, int len, int lo, int t_first, int64_t k0,
                                 int cap, int n_tl, double *hist, int *nonfinite, double *scratch, cudaStream_t st) {
    dim3 block(32, 8);
    if (groups > 2 * kGch) {
        const int g1 = (groups + kGch - 1) / kGch;
        finalize_stage1_kernel<<<dim3((len + 31) / 32, g1), block, 0, st>>>(partial, groups, len, scratch);
        partial = scratch;
        groups = g1;
    }
    finalize_wave_kernel<<<dim3((len + 31) / 32), block, 0, st>>>(partial, groups, len, lo, t_first, k0, cap, n_tl,
                                                                  hist, nonfinite);
    return cudaGetLastError();
}

int64_t finalize_scratch_doubles(int groups, int n_tl) {
    return (int64_t)((groups + kGchT - 1) / kGchT) * n_tl * 2;   // both forms (two-stage, ticketed)
}

__global__ void advance_kernel(int64_t *ctr, int64_t value, int add) {
    if (add) *ctr += value;
    else *ctr = value;
}

cudaError_t launch_counter(int64_t *ctr, int64_t value, bool add, cudaStream_t st) {
    advance_kernel<<<1, 1, 0, st>>>(ctr, value, add ? 1 : 0);
    return cudaGetLastError();
}

// One-launch form of the two stages: block (x, c) sums groups [c kGchT, (c+1) kGchT) of the
// 32 steps of column tile x (fixed split over 8 y-lanes, fixed-order lane sum) into
// scratch[c]; the LAST block of column tile x to finish (ticket counter) sums scratch over
// c in order and writes the norms -- deterministic, since the order is the chunk index, not
// the arrival.  part0 (deferred first step of the overlapped halo): the p-norm of step 0 is
// the fixed-order sum of part0[0..nb0) instead.
__global__ void finalize_ticket_kernel(const double *__restrict__ partial, int groups, int n_tl, double *norms,
                                       int *nonfinite, double *scratch, int *tickets, const double *part0, int nb0,
                                       const int64_t *slot_ctr, int64_t slot_off, int cap) {
    if (slot_ctr) norms += ((*slot_ctr + slot_off) % cap) * (int64_t)n_tl * 2;
    __shared__ double sm[8][32][2];
    __shared__ int last;
    const int t = blockIdx.x * 32 + threadIdx.x, y = threadIdx.y, c = blockIdx.y;
    const int g0 = c * kGchT, g1 = min(groups, g0 + kGchT);
    double su = 0.0, sp = 0.0;
    if (t < n_tl)
        for (int g = g0 + y; g < g1; g += 8) {
            su += partial[((int64_t)g * n_tl + t) * 2 + 0];
            sp += partial[((int64_t)g * n_tl + t) * 2 + 1];
        }
    sm[y][threadIdx.x][0] = su;
    sm[y][threadIdx.x][1] = sp;
    __syncthreads();
    if (y == 0 && t < n_tl) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < 8; ++k) {
            a += sm[k][threadIdx.x][0];
            b += sm[k][threadIdx.x][1];
        }
        scratch[((int64_t)c * n_tl + t) * 2 + 0] = a;
        scratch[((int64_t)c * n_tl + t) * 2 + 1] = b;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && y == 0) last = atomicAdd(&tickets[blockIdx.x], 1) == (int)gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    double p0 = 0.0;
    if (part0 && blockIdx.x == 0) {   // the completed first step's p-norm: fixed-order tree over part0
        __shared__ double r0[256];
        const int tid = y * 32 + threadIdx.x;
        double s = 0.0;
        for (int b = tid; b < nb0; b += 256) s += part0[b];
        r0[tid] = s;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (tid < w) r0[tid] += r0[tid + w];
            __syncthreads();
        }
        p0 = r0[0];
    }
    // chunk sums: fixed split over the 8 y-lanes, then a fixed-order sum of the lane totals
    {
        double a = 0.0, b = 0.0;
        if (t < n_tl)
            for (int k = y; k < (int)gridDim.y; k += 8) {
                a += __ldcg(scratch + ((int64_t)k * n_tl + t) * 2 + 0);
                b += __ldcg(scratch + ((int64_t)k * n_tl + t) * 2 + 1);
            }
        __syncthreads();
        sm[y][threadIdx.x][0] = a;
        sm[y][threadIdx.x][1] = b;
        __syncthreads();
    }
    if (y == 0 && t < n_tl) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < 8; ++k) {
            a += sm[k][threadIdx.x][0];
            b += sm[k][threadIdx.x][1];
        }
        if (part0 && t == 0) b = p0;
        a = sqrt(a);
        b = sqrt(b);
        norms[t * 2 + 0] = a;
        norms[t * 2 + 1] = b;
        if (!isfinite(a) || !isfinite(b)) atomicOr(nonfinite, 1);
    }
    if (threadIdx.x == 0 && y == 0) tickets[blockIdx.x] = 0;   // ready for the next launch
}

int finalize_tickets(int n_tl) { return (n_tl + 31) / 32; }

cudaError_t launch_finalize(const double *partial, int groups, int n_tl, double *norms,
                            int *nonfinite, double *scratch, cudaStream_t st, const int64_t *slot_ctr,
                            int64_t slot_off, int cap, int *tickets, const double *part0, int nb0) {
    dim3 block(32, 8);
    if (tickets) {
        const int g1 = (groups + kGchT - 1) / kGchT;
        finalize_ticket_kernel<<<dim3((n_tl + 31) / 32, g1), block, 0, st>>>(partial, groups, n_tl, norms, nonfinite,
                                                                             scratch, tickets, part0, nb0, slot_ctr,
                                                                             slot_off, cap);
        return cudaGetLastError();
    }
    if (groups > 2 * kGch) {   // two fixed-order stages: many groups would serialise one pass
        const int g1 = (groups + kGch - 1) / kGch;
        finalize_stage1_kernel<<<dim3((n_tl + 31) / 32, g1), block, 0, st>>>(partial, groups, n_tl, scratch);
        partial = scratch;
        groups = g1;
    }
    finalize_kernel<<<dim3((n_tl + 31) / 32), block, 0, st>>>(partial, groups, n_tl, norms, nonfinite, slot_ctr,
                                                              slot_off, cap);
    return cudaGetLastError();
}

}  // namespace biot
