// Device-side per-node arithmetic shared by the sweep kernels (internal header).
// One row node i, the T time steps of one lane: residual with the fused
// previous-step coupling, P~2 / first half of P~1
// (L238-262), damped update, norm accumulation.
#pragma once
#include "sweep_kernels.cuh"

namespace biot {
namespace dev {

constexpr int kSlotUnroll = 1;   // slot loop kept rolled: bounded registers, no spills

template <int S, bool ELL>
__device__ __forceinline__ int64_t column(const int32_t *__restrict__ cols, const int64_t *off,
                                          int64_t i, int s) {
    if constexpr (ELL) return (int64_t)__ldg(cols + i * S + s);
    else return i + off[s];
}

template <int D>
__host__ __device__ constexpr int block_pitch() { return ((D + 1) * (D + 1) + 2) / 2 * 2; }

// Coefficient load: global (read-only path) or shared memory (staged by TMA).
template <bool SMEM>
__device__ __forceinline__ double cload(const double *p) {
    if constexpr (SMEM) return *p;
    else return __ldg(p);
}

// Arithmetic of the epilogue of one node over T consecutive steps (shared by every
// sweep kernel so the results are identical): r = s_t f + q(t-1) - acc, norms,
// z = P^-1 r (P~2, or the displacement half of P~1), x^{k+1} = x^k + omega z.
// MASK = false: the caller guarantees no Dirichlet row (interior stencil nodes).
// ZFULL: outz = z = P~2^{-1} r for every component (GMRES; zfull_rt = false: the first
// half (z_u, r_p) of P~1^{-1} r for GMRES with P~1); else outz = (z_u, r_p)
// (the P~1 first pass).
// The load of step t at one node: f_t = sum_j s_j(t) F_j.  The epilogue applies term 0
// (the traction load s_t F of R16, or the first term of R24); the kMaxLoads kernels
// subtract the further terms from the accumulators before it.
template <int NC, int T, int NL>
struct Loads {
    double F[NL][NC];
    double sv[NL][T];
    __device__ __forceinline__ double at(int c, int tt) const {
        double l = sv[0][tt] * F[0][c];
#pragma unroll
        for (int j = 1; j < NL; ++j) l = fma(sv[j][tt], F[j][c], l);
        return l;
    }
    // the load plus `add` with explicit fused multiply-adds (term 0 first): no rounding
    // left to the compiler's contraction choices, so a kernel that completes the update
    // later (the deferred first step of the overlapped halo) reproduces it bitwise
    __device__ __forceinline__ double at_plus(int c, int tt, double add) const {
        double l = __fma_rn(sv[0][tt], F[0][c], add);
#pragma unroll
        for (int j = 1; j < NL; ++j) l = __fma_rn(sv[j][tt], F[j][c], l);
        return l;
    }
};

template <int NC, int T>
__device__ __forceinline__ Loads<NC, T, 1> single_load(const double (&F)[NC], const double (&sv)[T]) {
    Loads<NC, T, 1> ld;
#pragma unroll
    for (int c = 0; c < NC; ++c) ld.F[0][c] = F[c];
#pragma unroll
    for (int tt = 0; tt < T; ++tt) ld.sv[0][tt] = sv[tt];
    return ld;
}

template <int D, int T, bool MASK, bool ZFULL = false, class LD>
__device__ __forceinline__ void epilogue_math(double omega, const double (&acc)[D + 1][T], const double (&q)[T],
                                              double qprev, const LD &ld,
                                              const double (&Dv)[D + 1], const double (&xs)[D + 1][T],
                                              double (&nu)[T], double (&npn)[T],
                                              double (&outx)[D + 1][T], double (&outz)[D + 1][T],
                                              bool zfull_rt = true) {
    constexpr int NC = D + 1;
#pragma unroll
    for (int tt = 0; tt < T; ++tt) {
        const double qp = (tt == 0) ? qprev : q[tt - 1];
        double r[NC];
#pragma unroll
        for (int c = 0; c < D; ++c) r[c] = ld.at(c, tt) - acc[c][tt];
        r[D] = __dsub_rn(ld.at_plus(D, tt, qp), acc[D][tt]);
        // Dirichlet rows (D^{-1} = 0) carry no residual: kernels that apply a shared
        // stencil to such rows (tile3d class templates) rely on this mask
        if constexpr (MASK) {
#pragma unroll
            for (int c = 0; c < NC; ++c) r[c] = (Dv[c] == 0.0) ? 0.0 : r[c];
        }
        double su = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) su = fma(r[c], r[c], su);
        nu[tt] += su;
        npn[tt] = fma(r[D], r[D], npn[tt]);
        double z[NC];
#pragma unroll
        for (int c = 0; c < D; ++c) z[c] = Dv[c] * r[c];
        z[D] = -(Dv[D] * r[D]);   // P~2 pressure part; P~1 finishes it in pass 2
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            outx[c][tt] = fma(omega, z[c], xs[c][tt]);
            outz[c][tt] = (c < D || (ZFULL && zfull_rt)) ? z[c] : r[D];
        }
    }
}

// Epilogue of one node over the lane's T steps: the shared arithmetic, then the
// stores (x^{k+1}, the P~1 Z panel, the send slice) by mode.
template <int D, int T, class A, bool MASK = true, class LD>
__device__ __forceinline__ void node_epilogue(const A &a, int64_t i, int t0,
                                              const double (&acc)[D + 1][T], const double (&q)[T],
                                              double qprev, const LD &ld,
                                              const double (&Dv)[D + 1], const double (&xs)[D + 1][T],
                                              double (&nu)[T], double (&npn)[T]) {
    constexpr int NC = D + 1;
    const int64_t P = a.pitch;
    const int mode = a.mode;
    double outx[NC][T], outz[NC][T];
    epilogue_math<D, T, MASK>(a.omega, acc, q, qprev, ld, Dv, xs, nu, npn, outx, outz);
    if (mode == MODE_RESIDUAL) return;

    const int n_tl = a.n_tl;
    const int ncw = (mode == MODE_UPDATE_P2) ? NC : D;   // P~1: pressure written by pass 2
    const bool full = (t0 + T <= n_tl);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c >= ncw) break;
        double *dst = a.xn + (i * NC + c) * P + t0;
        if (full) {
            if constexpr (T % 2 == 0) {
#pragma unroll
                for (int h = 0; h < T; h += 2)
                    *reinterpret_cast<double2 *>(dst + h) = make_double2(outx[c][h], outx[c][h + 1]);
            } else {
#pragma unroll
                for (int tt = 0; tt < T; ++tt) dst[tt] = outx[c][tt];
            }
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
                if constexpr (T % 2 == 0) {
#pragma unroll
                    for (int h = 0; h < T; h += 2)
                        *reinterpret_cast<double2 *>(dst + h) = make_double2(outz[c][h], outz[c][h + 1]);
                } else {
#pragma unroll
                    for (int tt = 0; tt < T; ++tt) dst[tt] = outz[c][tt];
                }
            } else {
#pragma unroll
                for (int tt = 0; tt < T; ++tt)
                    if (t0 + tt < n_tl) dst[tt] = outz[c][tt];
            }
        }
    }
    if (a.sendbuf) {
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

// One row node i over the lane's T steps.  bp -> the node's S coefficient blocks
// (global memory, or a shared-memory copy when SMEM_CF).  The FMA order (slots in
// storage order, components ascending) is the same for every kernel that calls it.
template <int D, int S, bool ELL, int T, bool SMEM_CF, int NL = 1>
__device__ __forceinline__ void node_update(const SweepArgs &a, int64_t i, const double *__restrict__ bp,
                                            int t0, int lane, const double (&sv)[NL][T], double (&nu)[T],
                                            double (&npn)[T]) {
    constexpr int NC = D + 1;
    constexpr int W = (NC * NC + 2) / 2 * 2;   // block pitch: (d+1)^2 + 1 padded to 16 B
    constexpr int UNR = SMEM_CF ? S : kSlotUnroll;
    const int64_t P = a.pitch;

    double acc[NC][T], q[T];
#pragma unroll
    for (int tt = 0; tt < T; ++tt) {
        q[tt] = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c][tt] = 0.0;
    }

#pragma unroll(UNR)
    for (int s = 0; s < S; ++s) {
        const int64_t j = column<S, ELL>(a.cols, a.off, i, s);
        const double *__restrict__ xj = a.x + j * NC * P + t0;
        double cf[W];
#pragma unroll
        for (int k = 0; k < W; ++k) cf[k] = cload<SMEM_CF>(bp + s * W + k);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
            double v[T];
#pragma unroll
            for (int h = 0; h < T; h += 2) {
                const double2 w2 = __ldg(reinterpret_cast<const double2 *>(xj + cc * P + h));
                v[h] = w2.x;
                v[h + 1] = w2.y;
            }
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
                for (int tt = 0; tt < T; ++tt) acc[c][tt] = fma(cf[c * NC + cc], v[tt], acc[c][tt]);
            const double qc = (cc < D) ? cf[D * NC + cc] : cf[NC * NC];
#pragma unroll
            for (int tt = 0; tt < T; ++tt) q[tt] = fma(qc, v[tt], q[tt]);
        }
    }

    // previous-step coupling for the lane's first step
    double qprev = __shfl_up_sync(0xffffffffu, q[T - 1], 1);
    if (lane == 0) {
        double qg = 0.0;
        const bool use_ghost = (t0 == 0);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int64_t j = column<S, ELL>(a.cols, a.off, i, s);
            const double *src = use_ghost ? (a.ghost + j * NC) : (a.x + j * NC * P + (t0 - 1));
            const int64_t stride = use_ghost ? 1 : P;
#pragma unroll
            for (int cc = 0; cc < NC; ++cc) {
                const double qc = (cc < D) ? cload<SMEM_CF>(bp + s * W + D * NC + cc)
                                           : cload<SMEM_CF>(bp + s * W + NC * NC);
                qg = fma(qc, __ldg(src + cc * stride), qg);
            }
        }
        qprev = qg;
    }

    // load terms j >= 1 folded into the accumulators (acc - sum_j s_j F_j); term 0 is
    // applied by the epilogue as in the single-load kernels
#pragma unroll
    for (int j = 1; j < NL; ++j)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const double fj = __ldg(a.loadx + ((j - 1) * a.n_nodes + i) * NC + c);
#pragma unroll
            for (int tt = 0; tt < T; ++tt) acc[c][tt] = fma(-sv[j][tt], fj, acc[c][tt]);
        }
    Loads<NC, T, 1> ld;
    double Dv[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        ld.F[0][c] = __ldg(a.load + i * NC + c);
        Dv[c] = __ldg(a.dinv + i * NC + c);
    }
#pragma unroll
    for (int tt = 0; tt < T; ++tt) ld.sv[0][tt] = sv[0][tt];
    double xs[NC][T];   // own x_i(t0..t0+3): reloaded (L1 hit) instead of held across the slot loop
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const double *src = a.x + (i * NC + c) * P + t0;
#pragma unroll
        for (int h = 0; h < T; h += 2) {
            const double2 w2 = __ldg(reinterpret_cast<const double2 *>(src + h));
            xs[c][h] = w2.x;
            xs[c][h + 1] = w2.y;
        }
    }
    node_epilogue<D, T>(a, i, t0, acc, q, qprev, ld, Dv, xs, nu, npn);
}


}  // namespace dev
}  // namespace biot
