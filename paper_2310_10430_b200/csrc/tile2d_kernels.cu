// TMA-pipelined 2D sweep kernel (structured n1 x n1 grid of right triangles,
// P1-P1, BDIA slot order [0, -W-1, -W, -1, +1, +W, +W+1]).  One outer
// iteration of the Jacobi-in-time inverted scheme (Alg. 2 as
// BASELINE.json reads it) with the block preconditioner (L238-262), the damped
// update and the per-step residual norms fused.
//
// The 2D path is HBM-bound (~88 FMAs per node and step against 48 bytes of x
// traffic), so the kernel is built to stream the space-time panel once with as
// few instructions per byte as possible:
//  * work tile = kSeg = 12 consecutive grid columns x a range of grid rows, for
//    every 128-step time chunk in turn (4 steps per lane: steps 2l, 2l+1 and
//    64+2l, 64+2l+1, so each 16-B shared-memory load of the warp is one contiguous
//    512-B run -- conflict-free; every coefficient and every loop/barrier
//    instruction serves 4 steps);
//  * one lane of a producer warpgroup streams each grid row's strip (14 nodes x 3
//    comps x 128 steps, one TMA tensor box, no time halo) and the 12 nodes' aux
//    records (kappa-dependent AA_pp per slot, load, preconditioner diagonals, path
//    flag) into a 5-stage ring (full/empty mbarriers); the producer warpgroup hands
//    its registers to the consumers (setmaxnreg 24 / 160);
//  * 12 consumer warps (one column each) march the rows holding only two rows:
//    at step m (rows m-1, m resident) a warp finishes its node of row m-1 (the
//    +W slots, then the epilogue) and starts its node of row m (-W and 0 slots);
//  * interior nodes share one stencil (kernel parameters, uniform-register
//    operands, structural zeros skipped); edge/corner nodes use the stencil of
//    their geometric class (9 classes, shared memory).
//  * P~1 in one pass (tile2d_p1_kernel below): 10 owned columns per tile, z_u
//    recomputed on a one-node halo, the pressure update lagged one row.
//
// Previous-step coupling (A' x_{n-1})_p: lane l uses q(t-1) of lane l-1 (one
// shuffle); lane 0 takes q(t0-1) from a shared-memory carry written by lane 31
// in the previous chunk, and in chunk 0 recomputes it from the ghost vector
// x_{first-1} in the same FMA order (iterates are bitwise independent of the
// time-slab split).  Per node the slots run in (row, column) order.
#include <cuda.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "node_update.cuh"
#include "sweep_kernels.cuh"
#include "tma_util.cuh"

namespace biot {

namespace {

using namespace dev;
using namespace tma;

constexpr int kSeg = 12;                    // grid columns per tile = consumer warps (3 warpgroups)
constexpr int kStrip = kSeg + 2;            // + halo columns
constexpr int kT2 = 4;                      // time steps per lane
constexpr int kCT = 32 * kT2;               // time steps per chunk
constexpr int kMaxRR = 32;                  // rows per tile (q carry capacity)
constexpr int kCW = Tile2dArgs::kClsW;      // doubles per class-stencil slot
constexpr uint32_t kXBytes = kStrip * 3 * kCT * 8;                                 // 43008

// Shared-memory layout by load-term count: single-load kernels stream 16-double aux
// records through a 5-stage ring and stage the class stencils in shared memory; the
// kMaxLoads kernels carry the further load vectors in 24-double records (F_j at
// [14 + 3 (j-1) + c]) through 5 stages and read the class stencils (boundary nodes only)
// from global memory, which frees the room for the longer records.
template <int NL>
struct Lay {
    static constexpr int kStages = 5;
    static constexpr int kAuxRec = NL == 1 ? Tile2dArgs::kAux : Tile2dArgs::kAuxML;
    static constexpr uint32_t kAuxBytes = kSeg * kAuxRec * 8;
    static constexpr uint32_t kStageBytes = (kXBytes + kAuxBytes + 127) / 128 * 128;
    static constexpr uint32_t kClsOff = kStages * kStageBytes;
    static constexpr uint32_t kCarryOff = kClsOff + (NL == 1 ? 9 * 7 * kCW * 8 : 0);
    static constexpr uint32_t kSmemBytes = kCarryOff + kMaxRR * kSeg * 8;
};

// (row delta, column delta) of the 7 BDIA slots in storage order
__host__ __device__ constexpr int sdr(int s) { return (s == 1 || s == 2) ? -1 : (s >= 5) ? 1 : 0; }
__host__ __device__ constexpr int sdc(int s) { return (s == 1 || s == 3) ? -1 : (s == 4 || s == 6) ? 1 : 0; }
__host__ __device__ constexpr int slot2(int dr, int dc) {
    int r = -1;
    for (int s = 0; s < 7; ++s)
        if (sdr(s) == dr && sdc(s) == dc) r = s;
    return r;
}

// Structural zeros of the interior right-triangle stencil, entry e = c*3+cc of the
// AA block (e < 9) or 9 = A'_pp: the self block has no displacement-pressure
// coupling, the diagonal (SW/NE) neighbours have no u_x-u_x / u_y-u_y coupling,
// and with S = 0 and uniform kappa no pressure-pressure coupling either (L is the
// 5-point stencil).  Host-verified.
__host__ __device__ constexpr bool tmpl_zero(int s, int e, bool s0) {
    return (s == 0) ? (e == 2 || e == 5 || e == 6 || e == 7)
                    : (s == 1 || s == 6) ? (e == 0 || e == 4 || (s0 && (e == 8 || e == 9))) : false;
}

// lane l holds steps t0 + {2l, 2l+1, 64+2l, 64+2l+1}: index tt -> (tt>>1)*64 + 2l + (tt&1)
__device__ __forceinline__ const double *col2(const double *row, int p, int c, int lane) {
    return row + (p * 3 + c) * kCT + lane * 2;
}

__device__ __forceinline__ void load_v(double (&v)[3][kT2], const double *row, int p, int lane) {
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const double *src = col2(row, p, cc, lane);
#pragma unroll
        for (int h = 0; h < kT2; h += 2) {
            const double2 w = *reinterpret_cast<const double2 *>(src + (h >> 1) * (kCT / 2));
            v[cc][h] = w.x;
            v[cc][h + 1] = w.y;
        }
    }
}

// acc/q of one interior node through slot s by the gathered column v
template <bool S0, class A>
__device__ __forceinline__ void fma_tmpl(double (&acc)[3][kT2], double (&q)[kT2], const A &a, int s,
                                         double pp, const double (&v)[3][kT2]) {
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int e = c * 3 + cc;
            if (tmpl_zero(s, e, S0)) continue;
            const double cf = (e == 8) ? pp : a.tmpl[s][e];
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) acc[c][tt] = fma(cf, v[cc][tt], acc[c][tt]);
        }
        const int eq = cc < 2 ? 6 + cc : 9;
        if (!tmpl_zero(s, eq, S0)) {
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) q[tt] = fma(a.tmpl[s][eq], v[cc][tt], q[tt]);
        }
    }
}

// same through a class stencil in shared memory (column-major per slot:
// T[cc*3 + c] = AA[c][cc], T[9] = A'_pp)
__device__ __forceinline__ void fma_cls(double (&acc)[3][kT2], double (&q)[kT2], const double *T, double pp,
                                        const double (&v)[3][kT2]) {
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const double c0 = T[cc * 3], c1 = T[cc * 3 + 1], c2 = cc == 2 ? pp : T[cc * 3 + 2];
        const double cq = cc < 2 ? T[cc * 3 + 2] : T[9];
#pragma unroll
        for (int tt = 0; tt < kT2; ++tt) {
            acc[0][tt] = fma(c0, v[cc][tt], acc[0][tt]);
            acc[1][tt] = fma(c1, v[cc][tt], acc[1][tt]);
            acc[2][tt] = fma(c2, v[cc][tt], acc[2][tt]);
            q[tt] = fma(cq, v[cc][tt], q[tt]);
        }
    }
}

// slots of row delta DR for the warp's node (strip position p), in column order
template <int DR, bool CLS, bool S0, class A>
__device__ __forceinline__ void accum_row(const A &a, const double *row, int p, int lane,
                                          const double *aux, const double *T, double (&acc)[3][kT2],
                                          double (&q)[kT2]) {
#pragma unroll
    for (int dc = -1; dc <= 1; ++dc) {
        const int s = slot2(DR, dc);
        if (s < 0) continue;
        double v[3][kT2];
        load_v(v, row, p + dc, lane);
        if constexpr (CLS) fma_cls(acc, q, T + s * kCW, aux[s], v);
        else fma_tmpl<S0, A>(acc, q, a, s, aux[s], v);
    }
}

// q(t0-1) from the ghost x_{first-1} in the accumulation order (lane 0, chunk 0)
template <bool CLS, bool S0, class A>
__device__ __forceinline__ double ghost_q(const A &a, int64_t i, const double *T) {
    double g = 0.0;
#pragma unroll
    for (int dr = -1; dr <= 1; ++dr)
#pragma unroll
        for (int dc = -1; dc <= 1; ++dc) {
            const int s = slot2(dr, dc);
            if (s < 0) continue;
            const int64_t j = i + a.off[s];
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const double xv = __ldg(a.ghost + (j * 3 + cc) * a.ghost_stride);
                if constexpr (CLS) {
                    g = fma(cc < 2 ? T[s * kCW + cc * 3 + 2] : T[s * kCW + 9], xv, g);
                } else {
                    const int eq = cc < 2 ? 6 + cc : 9;
                    if (!tmpl_zero(s, eq, S0)) g = fma(a.tmpl[s][eq], xv, g);
                }
            }
        }
    return g;
}

template <bool CLS, bool S0, class A>
__device__ __forceinline__ void start(const A &a, const double *pd, const double *pm, int p, int lane,
                                      const double *aux, const double *T, double (&acc)[3][kT2],
                                      double (&q)[kT2]) {
#pragma unroll
    for (int tt = 0; tt < kT2; ++tt) {
        q[tt] = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c][tt] = 0.0;
    }
    accum_row<-1, CLS, S0, A>(a, pd, p, lane, aux, T, acc, q);
    accum_row<0, CLS, S0, A>(a, pm, p, lane, aux, T, acc, q);
}

// The epilogue runs on each half (2 consecutive steps) of the lane's steps: the shared
// arithmetic (dev::epilogue_math), then stores through one row pointer per node (the
// mode is a compile-time parameter; `full`: the whole chunk lies inside the slab).
template <bool CLS, bool S0, int MODE, int NL, class A>
__device__ __forceinline__ void finish(const A &a, const double *po, const double *pu, int p, int lane,
                                       const double *aux, const double *T, int64_t i, int t0, bool ghost,
                                       bool full, double *carry, const double (&sv)[kT2], double (&acc)[3][kT2],
                                       double (&q)[kT2], double (&nu)[kT2], double (&npn)[kT2]) {
    accum_row<1, CLS, S0, A>(a, pu, p, lane, aux, T, acc, q);
    if constexpr (NL > 1) {
        // load terms j >= 1 folded into the accumulators now (acc - sum_j s_j F_j), while
        // only acc is live: the epilogue then applies term 0 as the single-load kernels do
#pragma unroll
        for (int j = 1; j < NL; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double2 s2 = __ldg(reinterpret_cast<const double2 *>(a.s + j * a.s_pitch + a.t_off + t0 +
                                                                           h * (kCT / 2)));
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double fj = aux[14 + 3 * (j - 1) + c];
                    acc[c][2 * h] = fma(-s2.x, fj, acc[c][2 * h]);
                    acc[c][2 * h + 1] = fma(-s2.y, fj, acc[c][2 * h + 1]);
                }
            }
    }
    // q(t-1) of each half's first step: lane l-1's matching step; lane 0 of the second
    // half takes lane 31's first-half step 63, lane 0 of the first half the carry
    double qp0 = __shfl_up_sync(0xffffffffu, q[1], 1);
    double qp1 = __shfl_sync(0xffffffffu, lane == 31 ? q[1] : q[3], (lane + 31) & 31);
    // ghost: q(t0-1) from the ghost column now (single-chunk windows); otherwise from the
    // carry, which the chunk loop prefilled from the ghost column for chunk 0
    if (lane == 0) qp0 = ghost ? (a.ghost_zero ? 0.0 : ghost_q<CLS, S0, A>(a, i, T)) : *carry;
    __syncwarp();
    if (lane == 31) *carry = q[3];
    double Dv[3], xs[3][kT2];
#pragma unroll
    for (int c = 0; c < 3; ++c) Dv[c] = aux[10 + c];
    load_v(xs, po, p, lane);
    const int64_t P = a.pitch;
    const int n_tl = a.n_tl;
    const int64_t row = i * 3 * P + a.t_off + t0;   // t0: step within the window
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double acc2[3][2], q2[2], xs2[3][2], nu2[2], np2[2], outx[3][2], outz[3][2];
        // load term 0 of the half's two steps (further terms are already in acc)
        Loads<3, 2, 1> ld;
        ld.sv[0][0] = sv[2 * h];
        ld.sv[0][1] = sv[2 * h + 1];
#pragma unroll
        for (int c = 0; c < 3; ++c) ld.F[0][c] = aux[7 + c];
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
            q2[tt] = q[2 * h + tt];
            nu2[tt] = nu[2 * h + tt];
            np2[tt] = npn[2 * h + tt];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                acc2[c][tt] = acc[c][2 * h + tt];
                xs2[c][tt] = xs[c][2 * h + tt];
            }
        }
        epilogue_math<2, 2, CLS, MODE == MODE_ZOUT>(a.omega, acc2, q2, h == 0 ? qp0 : qp1, ld, Dv, xs2, nu2, np2,
                                                    outx, outz, !a.p1_out);
        if (MODE == MODE_UPDATE_P2 && a.s0buf && h == 0 && t0 == 0) {   // deferred first step (lane 0)
            double *sb = a.s0buf + i * 8;
            sb[0] = acc2[2][0];
            sb[1] = aux[9];
            sb[2] = xs2[2][0];
            sb[4] = aux[12];
            sb[5] = aux[13];
        }
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
            nu[2 * h + tt] = nu2[tt];
            npn[2 * h + tt] = np2[tt];
        }
        if constexpr (MODE == MODE_ZOUT) {
            const int th = t0 + h * (kCT / 2);
            const bool st0 = th < n_tl && th >= a.t_lo, st1 = th + 1 < n_tl && th + 1 >= a.t_lo;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double *dst = a.zbuf + row + c * P + h * (kCT / 2);
                if (full) {
                    *reinterpret_cast<double2 *>(dst) = make_double2(outz[c][0], outz[c][1]);
                } else {
                    if (st0) dst[0] = outz[c][0];
                    if (st1) dst[1] = outz[c][1];
                }
            }
        } else if constexpr (MODE != MODE_RESIDUAL) {
            constexpr int ncw = MODE == MODE_UPDATE_P2 ? 3 : 2;   // P~1: pressure written by pass 2
            const int th = t0 + h * (kCT / 2);
            const bool st0 = th < n_tl && th >= a.t_lo, st1 = th + 1 < n_tl && th + 1 >= a.t_lo;
#pragma unroll
            for (int c = 0; c < ncw; ++c) {
                double *dst = a.xn + row + c * P + h * (kCT / 2);
                if (full) {
                    *reinterpret_cast<double2 *>(dst) = make_double2(outx[c][0], outx[c][1]);
                } else {
                    if (st0) dst[0] = outx[c][0];
                    if (st1) dst[1] = outx[c][1];
                }
            }
            if constexpr (MODE == MODE_P1_PASS1) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double *dst = a.zbuf + row + c * P + h * (kCT / 2);
                    if (full) {
                        *reinterpret_cast<double2 *>(dst) = make_double2(outz[c][0], outz[c][1]);
                    } else {
                        if (st0) dst[0] = outz[c][0];
                        if (st1) dst[1] = outz[c][1];
                    }
                }
            }
            if (a.sendbuf) {
                const int tl = n_tl - 1 - th;
                if (tl == 0 || tl == 1)
#pragma unroll
                    for (int c = 0; c < ncw; ++c) a.sendbuf[i * 3 + c] = tl == 0 ? outx[c][0] : outx[c][1];
            }
        }
    }
}

// ---- P~1 second pass (PAPER.md eq. p1: z_p = S~p^{-1} (B^T z_u - r_p)) on the Z panel
// staged like x: bt = (B^T z_u) over the slots in (row, column) order, interior
// coefficients AA[p][u_cc] from the template (zeros skipped) or the class stencil.
template <int DR, bool CLS, bool S0, class A>
__device__ __forceinline__ void accum_row_bt(const A &a, const double *row, int p, int lane, const double *T,
                                             double (&bt)[kT2]) {
#pragma unroll
    for (int dc = -1; dc <= 1; ++dc) {
        const int s = slot2(DR, dc);
        if (s < 0) continue;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            if constexpr (!CLS) {
                if (tmpl_zero(s, 6 + cc, S0)) continue;
            }
            const double cf = CLS ? T[s * kCW + cc * 3 + 2] : a.tmpl[s][6 + cc];
            const double *src = col2(row, p + dc, cc, lane);
#pragma unroll
            for (int h = 0; h < kT2; h += 2) {
                const double2 w = *reinterpret_cast<const double2 *>(src + (h >> 1) * (kCT / 2));
                bt[h] = fma(cf, w.x, bt[h]);
                bt[h + 1] = fma(cf, w.y, bt[h + 1]);
            }
        }
    }
}

template <bool CLS, bool S0, class A>
__device__ __forceinline__ void start_bt(const A &a, const double *pd, const double *pm, int p, int lane,
                                         const double *T, double (&bt)[kT2]) {
#pragma unroll
    for (int tt = 0; tt < kT2; ++tt) bt[tt] = 0.0;
    accum_row_bt<-1, CLS, S0, A>(a, pd, p, lane, T, bt);
    accum_row_bt<0, CLS, S0, A>(a, pm, p, lane, T, bt);
}

template <bool CLS, bool S0, class A>
__device__ __forceinline__ void finish_bt(const A &a, const double *po, const double *pu, int p, int lane,
                                          const double *aux, const double *T, int64_t i, int t0, bool whole,
                                          double (&bt)[kT2]) {
    accum_row_bt<1, CLS, S0, A>(a, pu, p, lane, T, bt);
    const double dv = aux[12];
    const int64_t P = a.pitch, row = i * 3 * P + 2 * P + a.t_off + t0;
    const double *rp = col2(po, p, 2, lane);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const double2 r2 = *reinterpret_cast<const double2 *>(rp + h * (kCT / 2));
        const double2 x2 = __ldg(reinterpret_cast<const double2 *>(a.x + row + h * (kCT / 2)));
        const double v0 = fma(a.omega, dv * (bt[2 * h] - r2.x), x2.x);
        const double v1 = fma(a.omega, dv * (bt[2 * h + 1] - r2.y), x2.y);
        double *dst = a.xn + row + h * (kCT / 2);
        const int th = t0 + h * (kCT / 2);
        if (whole) {
            *reinterpret_cast<double2 *>(dst) = make_double2(v0, v1);
        } else {
            if (th < a.n_tl && th >= a.t_lo) dst[0] = v0;
            if (th + 1 < a.n_tl && th + 1 >= a.t_lo) dst[1] = v1;
        }
        if (a.sendbuf) {
            if (th == a.n_tl - 1) a.sendbuf[i * 3 + 2] = v0;
            if (th + 1 == a.n_tl - 1) a.sendbuf[i * 3 + 2] = v1;
        }
    }
}

// ---- GMRES (Alg. 3 with K = GMRES, R23): w = P~2^{-1} (AA v) on the staged
// v panel; the slots as the residual's, no previous-step coupling.
template <bool CLS, bool S0, class A>
__device__ __forceinline__ void finish_mv(const A &a, const double *pu, int p, int lane, const double *aux,
                                          const double *T, int64_t i, int t0, bool whole, double (&acc)[3][kT2],
                                          double (&q)[kT2]) {
    accum_row<1, CLS, S0, A>(a, pu, p, lane, aux, T, acc, q);
    const int64_t P = a.pitch, row = i * 3 * P + a.t_off + t0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int th = t0 + h * (kCT / 2);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double dv = aux[10 + c];
            // P~2^{-1} AA v; P~1: its first half (D_A^{-1} (AA v)_u, (AA v)_p)
            const double w0 = c < 2 ? dv * acc[c][2 * h] : a.p1_out ? acc[c][2 * h] : -(dv * acc[c][2 * h]);
            const double w1 = c < 2 ? dv * acc[c][2 * h + 1] : a.p1_out ? acc[c][2 * h + 1] : -(dv * acc[c][2 * h + 1]);
            double *dst = a.xn + row + c * P + h * (kCT / 2);
            if (whole) {
                *reinterpret_cast<double2 *>(dst) = make_double2(w0, w1);
            } else {
                if (th < a.n_tl) dst[0] = w0;
                if (th + 1 < a.n_tl) dst[1] = w1;
            }
        }
    }
}

struct Geo2 {
    int W, nrows, nseg, nrr, ntiles, nchunks, rr;
    bool rb_even;                 // balanced row blocks (n_rblk)
    __device__ explicit Geo2(const Tile2dArgs &a) {
        W = (int)a.row_w;
        nrows = a.n_rows;
        rr = a.rows_per_tile;
        nseg = (W + kSeg - 1) / kSeg;
        rb_even = a.n_rblk > 0;
        nrr = rb_even ? a.n_rblk : (nrows + rr - 1) / rr;
        ntiles = nseg * nrr;
        nchunks = (a.n_tl + kCT - 1) / kCT;
    }
    __device__ void decode(int tile, int &i0, int &ja, int &jb) const {
        const int seg = tile % nseg, r = tile / nseg;
        i0 = seg * kSeg;
        if (rb_even) {
            ja = (int)((int64_t)r * nrows / nrr);
            jb = (int)((int64_t)(r + 1) * nrows / nrr);
        } else {
            ja = r * rr;
            jb = min(nrows, ja + rr);
        }
    }
};

__device__ __forceinline__ int axis_class(int v, int n) { return v == 0 ? 0 : (v == n - 1 ? 2 : 1); }

// the 12 aux records of grid row r from column c0 are all aux_u (see Tile2dArgs::aux_geo)
__device__ __forceinline__ bool seg_uniform(const Tile2dArgs &a, int r, int c0) {
    return a.aux_geo && r >= a.uy0 && r <= a.uy1 && c0 >= a.ux0 && c0 + kSeg - 1 <= a.ux1;
}

// Block = 3 consumer warpgroups + 1 producer warpgroup (only its first lane issues
// copies); the producer group hands its registers to the consumers (setmaxnreg:
// 4 x 32 x 24 + 12 x 32 x 160 <= 65536).
constexpr int kThreads2 = (kSeg + 4) * 32;
constexpr int kProducerRegs = 24, kConsumerRegs = 160;

template <bool S0, int MODE, int NL>
__global__ void __launch_bounds__(kThreads2, 1)
    tile2d_kernel(const __grid_constant__ CUtensorMap tmx, const Tile2dArgs a) {
    using L = Lay<NL>;
    constexpr int kStages = L::kStages, kAuxRec = L::kAuxRec;
    constexpr uint32_t kAuxBytes = L::kAuxBytes, kStageBytes = L::kStageBytes;
    constexpr uint32_t kClsOff = L::kClsOff, kCarryOff = L::kCarryOff;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    double *cls_sm = reinterpret_cast<double *>(smem + kClsOff);     // [9][7][kCW]
    double *qcarry = reinterpret_cast<double *>(smem + kCarryOff);   // [kMaxRR][kSeg]
    __shared__ __align__(16) double aux_u[kAuxRecU];                 // the aux-uniform record

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Geo2 g(a);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kSeg);
        }
        fence_barrier_init();
    }
    if constexpr (NL == 1)
        for (int k = threadIdx.x; k < 9 * 7 * kCW; k += blockDim.x) cls_sm[k] = a.cls[k];
    if (threadIdx.x < kAuxRecU) aux_u[threadIdx.x] = a.aux_u[threadIdx.x];
    __syncthreads();

    if (warp >= kSeg) {
        // ------------------------------- producer -------------------------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
        if (warp == kSeg && lane == 0) {
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
                int i0, ja, jb;
                g.decode(tile, i0, ja, jb);
                for (int chunk = 0; chunk < g.nchunks; ++chunk)
                    for (int r = ja - 1; r <= jb; ++r, ++it) {
                        const int st = it % kStages;
                        if (it >= (uint32_t)kStages) mbar_wait_suspend(&empty[st], ((it / kStages) - 1) & 1);
                        unsigned char *base = smem + (size_t)st * kStageBytes;
                        const bool real = (r >= 0 && r < g.nrows) && !(NL == 1 && seg_uniform(a, r, i0));
                        mbar_expect_tx(&full[st], kXBytes + (real ? kAuxBytes : 0u));
                        const int64_t node0 = (int64_t)r * g.W + i0 - 1;
                        load_2d(base, &tmx, a.t_off + chunk * kCT, (int)((node0 + a.pad_nodes) * 3), &full[st]);
                        if (real)
                            bulk_g2s(base + kXBytes, a.aux + ((int64_t)r * g.W + i0) * kAuxRec, kAuxBytes,
                                     &full[st]);
                    }
            }
        }
        return;
    }

    // ------------------------------- consumers ------------------------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));
    const int p = warp + 1;                   // strip position of the warp's column
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
        int i0, ja, jb;
        g.decode(tile, i0, ja, jb);
        const int col = i0 + warp;
        const bool valid = col < g.W;
        const int ccx = axis_class(min(col, g.W - 1), g.W);
        for (int chunk = 0; chunk < g.nchunks; ++chunk) {
            const int t0 = chunk * kCT + lane * 2;   // the lane's first half; second half at t0 + 64
            const bool ghost = chunk == 0;
            const bool whole = (chunk + 1) * kCT <= a.n_tl && (chunk > 0 || a.t_lo == 0);   // chunk inside the window
            double nu[kT2], npn[kT2], sv[kT2], prev[kT2][2];
            // load scales s_t of the lane's steps (zero past n_tl) and, issued now so its
            // latency hides behind the march, this (CTA, column)'s running norm sums
            const bool first = tile == (int)blockIdx.x;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double2 s2 = __ldg(reinterpret_cast<const double2 *>(a.s + a.t_off + t0 + h * (kCT / 2)));
                sv[2 * h] = s2.x;
                sv[2 * h + 1] = s2.y;
            }
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) {
                nu[tt] = 0.0;
                npn[tt] = 0.0;
                const int t = t0 + (tt >> 1) * (kCT / 2) + (tt & 1);
                prev[tt][0] = prev[tt][1] = 0.0;
                if (MODE != MODE_PASS2 && MODE != MODE_MATVEC && !first && t < a.n_tl) {
                    const double *src = a.partial + (((int64_t)blockIdx.x * kSeg + warp) * a.n_tl + t) * 2;
                    prev[tt][0] = src[0];
                    prev[tt][1] = src[1];
                }
            }
            double acc[3][kT2], q[kT2];
            int kindP = 0;                       // pending node (row m-1): 0 none, 1 interior, 2 class
            const double *const cls_base = NL == 1 ? static_cast<const double *>(cls_sm) : a.cls;
            const double *T = cls_base;
            if constexpr (MODE != MODE_PASS2 && MODE != MODE_MATVEC) {
                if (ghost && g.nchunks > 1 && valid && a.dry != 1) {
                    // q(t0-1) of chunk 0 from the ghost column, for every row of the tile at
                    // once (one row per lane, each in the march's FMA order), into the q
                    // carry that later chunks use: its global loads overlap instead of
                    // stalling lane 0 at every node.  Single-chunk passes (the Gauss-Seidel
                    // windows) keep the per-node path: there the prefill would stall every
                    // tile start while the ring is full
                    for (int mm = ja + lane; mm < jb; mm += 32) {
                        const int64_t i = (int64_t)mm * g.W + col;
                        const bool intr = __ldg(a.aux + i * kAuxRec + 13) == 1.0;
                        qcarry[(mm - ja) * kSeg + warp] =
                            a.ghost_zero ? 0.0
                            : intr ? ghost_q<false, S0, Tile2dArgs>(a, i, cls_base)
                                   : ghost_q<true, S0, Tile2dArgs>(
                                         a, i, cls_base + (ccx + 3 * axis_class(mm, g.nrows)) * 7 * kCW);
                    }
                    __syncwarp();
                }
            }
            int sd = it % kStages;               // stage of row m-1
            uint32_t phd = (it / kStages) & 1;
            mbar_wait_suspend(&full[sd], phd);
            for (int m = ja; m <= jb; ++m) {
                const int sm_ = sd + 1 == kStages ? 0 : sd + 1;
                const uint32_t phm = sm_ == 0 ? phd ^ 1u : phd;
                mbar_wait_suspend(&full[sm_], phm);
                const double *pd = reinterpret_cast<const double *>(smem + (size_t)sd * kStageBytes);
                const double *pm = reinterpret_cast<const double *>(smem + (size_t)sm_ * kStageBytes);
                if (a.dry != 1) {
                    if (kindP != 0) {            // finish row m-1
                        const double *aux = (NL == 1 && seg_uniform(a, m - 1, i0)) ? aux_u
                                            : reinterpret_cast<const double *>(
                                                  reinterpret_cast<const unsigned char *>(pd) + kXBytes) + warp * kAuxRec;
                        const int64_t i = (int64_t)(m - 1) * g.W + col;
                        double *carry = qcarry + (m - 1 - ja) * kSeg + warp;
                        if constexpr (MODE == MODE_PASS2) {
                            if (kindP == 1) finish_bt<false, S0, Tile2dArgs>(a, pd, pm, p, lane, aux, T, i, t0, whole, q);
                            else finish_bt<true, S0, Tile2dArgs>(a, pd, pm, p, lane, aux, T, i, t0, whole, q);
                        } else if constexpr (MODE == MODE_MATVEC) {
                            if (kindP == 1) finish_mv<false, S0, Tile2dArgs>(a, pm, p, lane, aux, T, i, t0, whole, acc, q);
                            else finish_mv<true, S0, Tile2dArgs>(a, pm, p, lane, aux, T, i, t0, whole, acc, q);
                        } else {
                            if (kindP == 1)
                                finish<false, S0, MODE, NL, Tile2dArgs>(a, pd, pm, p, lane, aux, T, i, t0, ghost && g.nchunks == 1, whole,
                                                                    carry, sv, acc, q, nu, npn);
                            else
                                finish<true, S0, MODE, NL, Tile2dArgs>(a, pd, pm, p, lane, aux, T, i, t0, ghost && g.nchunks == 1, whole,
                                                                   carry, sv, acc, q, nu, npn);
                        }
                    }
                    kindP = 0;
                    if (m < jb && valid) {       // start row m
                        const double *aux = (NL == 1 && seg_uniform(a, m, i0)) ? aux_u
                                            : reinterpret_cast<const double *>(
                                                  reinterpret_cast<const unsigned char *>(pm) + kXBytes) + warp * kAuxRec;
                        kindP = aux[13] == 1.0 ? 1 : 2;
                        if (kindP == 2) T = cls_base + (ccx + 3 * axis_class(m, g.nrows)) * 7 * kCW;
                        if constexpr (MODE == MODE_PASS2) {   // bt rides in q
                            if (kindP == 1) start_bt<false, S0, Tile2dArgs>(a, pd, pm, p, lane, T, q);
                            else start_bt<true, S0, Tile2dArgs>(a, pd, pm, p, lane, T, q);
                        } else {
                            if (kindP == 1) start<false, S0, Tile2dArgs>(a, pd, pm, p, lane, aux, T, acc, q);
                            else start<true, S0, Tile2dArgs>(a, pd, pm, p, lane, aux, T, acc, q);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[sd]);   // row m-1 no longer needed
                sd = sm_;
                phd = phm;
            }
            if (lane == 0) mbar_arrive(&empty[sd]);       // row jb
            it += (uint32_t)(jb - ja + 2);
            // per-step norm partials of this (CTA, column), summed over the rows and, in
            // the CTA's fixed tile order, over its tiles (the lane re-reads its own sums)
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) {
                if constexpr (MODE == MODE_PASS2 || MODE == MODE_MATVEC) break;   // no norms in these passes
                const int t = t0 + (tt >> 1) * (kCT / 2) + (tt & 1);
                if (t < a.n_tl) {
                    double *dst = a.partial + (((int64_t)blockIdx.x * kSeg + warp) * a.n_tl + t) * 2;
                    const double u = t >= a.t_lo ? nu[tt] : 0.0, v = t >= a.t_lo ? npn[tt] : 0.0;
                    dst[0] = first ? u : prev[tt][0] + u;
                    dst[1] = first ? v : prev[tt][1] + v;
                }
            }
        }
    }
}


// ============================================================================
// P~1 in one pass (PAPER.md eq. p1: P~1 = [[A, 0], [B^T, -S~p]], so
// z_u = A^{-1} r_u and z_p = S~p^{-1} (B^T z_u - r_p); inner inverses by their
// diagonals, reading R2).  z_p of a node needs z_u of its 7 neighbours, and z_u of a
// neighbour needs that neighbour's residual, so a tile computes z_u on a one-node
// halo around the nodes it owns: of the 12 consumer columns (strip positions 1..12)
// positions 2..11 are owned and 1, 12 only produce z_u; the rows march from ja-1 to
// jb (ja-1 and jb produce z_u only), reading x rows ja-2..jb+1.  The pressure update
// is lagged one row: at row step m a warp finishes node m-1 (residual, norms, x_u,
// z_u published in shared memory), then -- after a CTA-wide named barrier -- adds
// the B^T contributions of row m-1's z_u to the nodes of rows m-2, m-1 and m of its
// column (push form: the node's own coefficients, slot order (row, column) as the
// two-pass kernel's pull), which completes node m-2: x_p += omega D_S^{-1} (bt - r_p).
// The Z panel round trip of the two-pass form (8 + 5 panel accesses per DoF instead
// of 6) is gone; the halo costs 14/10 x reads and 12/10 x residual work.
// ============================================================================
constexpr int kSegP1 = kSeg - 2;            // owned grid columns per tile

template <int NL>
struct LayP1 {
    static constexpr int kStages = NL == 1 ? 4 : 3;
    static constexpr int kAuxRec = NL == 1 ? Tile2dArgs::kAux : Tile2dArgs::kAuxML;
    static constexpr uint32_t kAuxBytes = kSeg * kAuxRec * 8;
    static constexpr uint32_t kStageBytes = (kXBytes + kAuxBytes + 127) / 128 * 128;
    static constexpr uint32_t kZBytes = kSeg * 2 * kCT * 8;                 // z_u of one row: 12 positions x 2 comps
    static constexpr uint32_t kZOff = kStages * kStageBytes;
    static constexpr uint32_t kCarryOff = kZOff + 2 * kZBytes;              // z_u double-buffered by row parity
    static constexpr uint32_t kSmemBytes = kCarryOff + (kMaxRR + 1) * kSeg * 8;   // + dummy carry row (halo rows)
};
static_assert(LayP1<1>::kSmemBytes <= 232448 - 128 && LayP1<kMaxLoads>::kSmemBytes <= 232448 - 128,
              "fused P~1 tile exceeds 227 KB");

constexpr uint32_t cmax(uint32_t x, uint32_t y) { return x > y ? x : y; }
// one dynamic shared-memory size for every tile2d kernel (the largest layout)
constexpr uint32_t kSmemBytes = cmax(cmax(Lay<1>::kSmemBytes, Lay<kMaxLoads>::kSmemBytes),
                                     cmax(LayP1<1>::kSmemBytes, LayP1<kMaxLoads>::kSmemBytes));
static_assert(kSmemBytes <= 232448 - 128, "tile2d shared memory exceeds 227 KB");

// B^T contribution of the z_u column at position p + DC of a published row to a node
// whose row delta to that row is DR (its slot (DR, DC)), both displacement components.
template <int DR, int DC, bool CLS, bool S0, class A>
__device__ __forceinline__ void bt_col(const A &a, const double (&z)[2][kT2], const double *T, double (&bt)[kT2]) {
    constexpr int s = slot2(DR, DC);
    if constexpr (s >= 0) {
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            if constexpr (!CLS) {
                if (tmpl_zero(s, 6 + cc, S0)) continue;
            }
            const double cf = CLS ? T[s * kCW + cc * 3 + 2] : a.tmpl[s][6 + cc];
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) bt[tt] = fma(cf, z[cc][tt], bt[tt]);
        }
    }
}

template <int DR, int DC, bool S0, class A>
__device__ __forceinline__ void bt_col_any(const A &a, int kind, const double (&z)[2][kT2], const double *T,
                                           double (&bt)[kT2]) {
    if (kind == 1) bt_col<DR, DC, false, S0, A>(a, z, T, bt);
    else if (kind == 2) bt_col<DR, DC, true, S0, A>(a, z, T, bt);
}

__device__ __forceinline__ void load_z(double (&z)[2][kT2], const double *zrow, int pos, int lane) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double2 w = *reinterpret_cast<const double2 *>(zrow + ((pos - 1) * 2 + c) * kCT + lane * 2 +
                                                                 h * (kCT / 2));
            z[c][2 * h] = w.x;
            z[c][2 * h + 1] = w.y;
        }
}

// Finish node (m-1) of the fused pass: the +W slots, the residual epilogue (norms of
// owned nodes), x_u^{k+1} of owned nodes; returns z_u (published by the caller),
// r_p and x_p^k of the lane's steps.
template <bool CLS, bool S0, int NL, class A>
__device__ __forceinline__ void finish_p1(const A &a, const double *po, const double *pu, int p, int lane,
                                          const double *aux, const double *T, int64_t i, int t0, bool ghost,
                                          bool whole, bool own, double *carry, double (&acc)[3][kT2], double (&q)[kT2], double (&nu)[kT2],
                                          double (&npn)[kT2], double *zd, double wdv, double (&y)[kT2]) {
    accum_row<1, CLS, S0, A>(a, pu, p, lane, aux, T, acc, q);
    if constexpr (NL > 1) {
#pragma unroll
        for (int j = 1; j < NL; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double2 s2 = __ldg(reinterpret_cast<const double2 *>(a.s + j * a.s_pitch + a.t_off + t0 +
                                                                           h * (kCT / 2)));
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double fj = aux[14 + 3 * (j - 1) + c];
                    acc[c][2 * h] = fma(-s2.x, fj, acc[c][2 * h]);
                    acc[c][2 * h + 1] = fma(-s2.y, fj, acc[c][2 * h + 1]);
                }
            }
    }
    double qp0 = __shfl_up_sync(0xffffffffu, q[1], 1);
    double qp1 = __shfl_sync(0xffffffffu, lane == 31 ? q[1] : q[3], (lane + 31) & 31);
    if (lane == 0) qp0 = ghost ? (a.ghost_zero ? 0.0 : ghost_q<CLS, S0, A>(a, i, T)) : *carry;
    __syncwarp();
    if (lane == 31) *carry = q[3];
    double Dv[3], xs[3][kT2];
#pragma unroll
    for (int c = 0; c < 3; ++c) Dv[c] = aux[10 + c];
    load_v(xs, po, p, lane);
    const int64_t P = a.pitch;
    const int n_tl = a.n_tl;
    const int64_t row = i * 3 * P + a.t_off + t0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        double acc2[3][2], q2[2], xs2[3][2], nu2[2] = {0.0, 0.0}, np2[2] = {0.0, 0.0}, outx[3][2], outz[3][2];
        Loads<3, 2, 1> ld;
        {   // the load scales from L1 at the point of use: 8 registers fewer across the march
            const double2 s2 = __ldg(reinterpret_cast<const double2 *>(a.s + a.t_off + t0 + h * (kCT / 2)));
            ld.sv[0][0] = s2.x;
            ld.sv[0][1] = s2.y;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) ld.F[0][c] = aux[7 + c];
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
            q2[tt] = q[2 * h + tt];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                acc2[c][tt] = acc[c][2 * h + tt];
                xs2[c][tt] = xs[c][2 * h + tt];
            }
        }
        epilogue_math<2, 2, CLS, false>(a.omega, acc2, q2, h == 0 ? qp0 : qp1, ld, Dv, xs2, nu2, np2, outx, outz);
        if (a.s0buf && own && h == 0 && t0 == 0) {   // deferred first step (lane 0)
            double *sb = a.s0buf + i * 8;
            sb[0] = acc2[2][0];
            sb[1] = aux[9];
            sb[2] = xs2[2][0];
            sb[4] = aux[12];
            sb[5] = aux[13];
        }
        const int th = t0 + h * (kCT / 2);
        // z_u published for the neighbours; the pressure part waits for B^T z_u:
        // x_p^{k+1} = x_p + omega D_S^{-1} (bt - r_p) = y + (omega D_S^{-1}) bt
#pragma unroll
        for (int c = 0; c < 2; ++c)
            *reinterpret_cast<double2 *>(zd + c * kCT + h * (kCT / 2)) = make_double2(outz[c][0], outz[c][1]);
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) y[2 * h + tt] = fma(-wdv, outz[2][tt], xs2[2][tt]);
        if (own) {
#pragma unroll
            for (int tt = 0; tt < 2; ++tt) {
                nu[2 * h + tt] += nu2[tt];       // = the in-place accumulation: nu + (0 + su)
                npn[2 * h + tt] += np2[tt];
            }
            const bool st0 = th < n_tl && th >= a.t_lo, st1 = th + 1 < n_tl && th + 1 >= a.t_lo;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                double *dst = a.xn + row + c * P + h * (kCT / 2);
                if (whole) {
                    *reinterpret_cast<double2 *>(dst) = make_double2(outx[c][0], outx[c][1]);
                } else {
                    if (st0) dst[0] = outx[c][0];
                    if (st1) dst[1] = outx[c][1];
                }
            }
            if (a.sendbuf) {
                const int tl = n_tl - 1 - th;
                if (tl == 0 || tl == 1)
#pragma unroll
                    for (int c = 0; c < 2; ++c) a.sendbuf[i * 3 + c] = tl == 0 ? outx[c][0] : outx[c][1];
            }
        }
    }
}

// x_p^{k+1} of an owned node whose B^T z_u is complete (as finish_bt of the two-pass form)
template <class A>
__device__ __forceinline__ void finish_zp(const A &a, int64_t i, int t0, bool whole, double wdv,
                                          const double (&bt)[kT2], const double (&y)[kT2]) {
    const int64_t P = a.pitch, row = i * 3 * P + 2 * P + a.t_off + t0;
    if (a.s0buf && t0 == 0) a.s0buf[i * 8 + 3] = bt[0];   // deferred first step (lane 0)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const double v0 = fma(wdv, bt[2 * h], y[2 * h]);
        const double v1 = fma(wdv, bt[2 * h + 1], y[2 * h + 1]);
        double *dst = a.xn + row + h * (kCT / 2);
        const int th = t0 + h * (kCT / 2);
        if (whole) {
            *reinterpret_cast<double2 *>(dst) = make_double2(v0, v1);
        } else {
            if (th < a.n_tl && th >= a.t_lo) dst[0] = v0;
            if (th + 1 < a.n_tl && th + 1 >= a.t_lo) dst[1] = v1;
        }
        if (a.sendbuf) {
            if (th == a.n_tl - 1) a.sendbuf[i * 3 + 2] = v0;
            if (th + 1 == a.n_tl - 1) a.sendbuf[i * 3 + 2] = v1;
        }
    }
}

__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <bool S0, int NL>
__global__ void __launch_bounds__(kThreads2, 1)
    tile2d_p1_kernel(const __grid_constant__ CUtensorMap tmx, const Tile2dArgs a) {
    using L = LayP1<NL>;
    constexpr int kStages = L::kStages, kAuxRec = L::kAuxRec;
    constexpr uint32_t kAuxBytes = L::kAuxBytes, kStageBytes = L::kStageBytes;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    __shared__ __align__(16) double aux_u[kAuxRecU];                     // the aux-uniform record
    double *zbuf = reinterpret_cast<double *>(smem + L::kZOff);          // [2][12][2][kCT]
    double *qcarry = reinterpret_cast<double *>(smem + L::kCarryOff);    // [kMaxRR + 1][kSeg]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = (int)a.row_w, nrows = a.n_rows, rr = a.rows_per_tile;
    const int nseg = (W + kSegP1 - 1) / kSegP1, nrr = (nrows + rr - 1) / rr;
    const int ntiles = nseg * nrr, nchunks = (a.n_tl + kCT - 1) / kCT;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kSeg);
        }
        fence_barrier_init();
    }
    if (threadIdx.x < kAuxRecU) aux_u[threadIdx.x] = a.aux_u[threadIdx.x];
    __syncthreads();

    if (warp >= kSeg) {
        // ------------------------------- producer -------------------------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
        if (warp == kSeg && lane == 0) {
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int i0 = (tile % nseg) * kSegP1, ja = (tile / nseg) * rr, jb = min(nrows, ja + rr);
                for (int chunk = 0; chunk < nchunks; ++chunk)
                    for (int r = ja - 2; r <= jb + 1; ++r, ++it) {
                        const int st = it % kStages;
                        if (it >= (uint32_t)kStages) mbar_wait_suspend(&empty[st], ((it / kStages) - 1) & 1);
                        unsigned char *base = smem + (size_t)st * kStageBytes;
                        const bool real = (r >= 0 && r < nrows) && !(NL == 1 && seg_uniform(a, r, i0 - 1));
                        mbar_expect_tx(&full[st], kXBytes + (real ? kAuxBytes : 0u));
                        const int64_t node0 = (int64_t)r * W + i0 - 2;
                        load_2d(base, &tmx, a.t_off + chunk * kCT, (int)((node0 + a.pad_nodes) * 3), &full[st]);
                        if (real)
                            bulk_g2s(base + kXBytes, a.aux + ((int64_t)r * W + i0 - 1) * kAuxRec, kAuxBytes,
                                     &full[st]);
                    }
            }
        }
        return;
    }

    // ------------------------------- consumers ------------------------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));
    const int p = warp + 1;                   // strip position: 1..12, owned 2..11
    const double *const cls_base = a.cls;     // class stencils (boundary nodes) from global memory
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int i0 = (tile % nseg) * kSegP1, ja = (tile / nseg) * rr, jb = min(nrows, ja + rr);
        const int col = i0 + p - 2;
        const bool valid = col >= 0 && col < W;
        const bool ocol = valid && p >= 2 && p <= kSegP1 + 1;
        const int ccx = axis_class(min(max(col, 0), W - 1), W);
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            const int t0 = chunk * kCT + lane * 2;
            const bool ghost = chunk == 0;
            const bool whole = (chunk + 1) * kCT <= a.n_tl && (chunk > 0 || a.t_lo == 0);
            double nu[kT2], npn[kT2];
            const bool first = tile == (int)blockIdx.x;
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) nu[tt] = npn[tt] = 0.0;
            if (ghost && nchunks > 1 && ocol) {
                // q(t0-1) of chunk 0 for the tile's owned rows, as the P~2 kernel does
                for (int mm = ja + lane; mm < jb; mm += 32) {
                    const int64_t i = (int64_t)mm * W + col;
                    const bool intr = __ldg(a.aux + i * kAuxRec + 13) == 1.0;
                    qcarry[(mm - ja) * kSeg + warp] =
                        a.ghost_zero ? 0.0
                        : intr ? ghost_q<false, S0, Tile2dArgs>(a, i, cls_base)
                               : ghost_q<true, S0, Tile2dArgs>(a, i, cls_base + (ccx + 3 * axis_class(mm, nrows)) * 7 * kCW);
                }
                __syncwarp();
            }
            double acc[3][kT2], q[kT2];
            double btA[kT2], btB[kT2], btC[kT2];          // B^T z_u of the nodes of rows m-2, m-1, m
            double yA[kT2], yB[kT2];                      // x_p - omega D_S^{-1} r_p of rows m-2, m-1
            double wA = 0.0, wB = 0.0;                    // omega D_S^{-1} of rows m-2, m-1
            int kindP = 0, kindA = 0, kindB = 0;          // node m-1 (pending finish); rows m-2, m-1 (pending z_p)
            const double *T = cls_base;
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) btA[tt] = btB[tt] = btC[tt] = yA[tt] = yB[tt] = 0.0;
            int sd = it % kStages;                        // stage of row m-1
            uint32_t phd = (it / kStages) & 1;
            mbar_wait_suspend(&full[sd], phd);
            for (int m = ja - 1; m <= jb + 1; ++m) {
                const int sm_ = sd + 1 == kStages ? 0 : sd + 1;
                const uint32_t phm = sm_ == 0 ? phd ^ 1u : phd;
                mbar_wait_suspend(&full[sm_], phm);
                const double *pd = reinterpret_cast<const double *>(smem + (size_t)sd * kStageBytes);
                const double *pm = reinterpret_cast<const double *>(smem + (size_t)sm_ * kStageBytes);
                double *zrow = zbuf + (size_t)((m - 1) & 1) * (kSeg * 2 * kCT);
                const bool orow1 = m - 1 >= ja && m - 1 < jb;       // node m-1 owned (row)
                // (1) finish node m-1 and publish its z_u (zero off the mesh)
                if (m >= ja) {
                    double *zd = zrow + (p - 1) * 2 * kCT + lane * 2;
                    if (kindP != 0) {
                        const double *aux = (NL == 1 && seg_uniform(a, m - 1, i0 - 1)) ? aux_u
                                            : reinterpret_cast<const double *>(
                                                  reinterpret_cast<const unsigned char *>(pd) + kXBytes) + warp * kAuxRec;
                        const int64_t i = (int64_t)(m - 1) * W + col;
                        double *carry = qcarry + (orow1 ? (m - 1 - ja) : kMaxRR) * kSeg + warp;
                        const bool own = orow1 && ocol;
                        wB = a.omega * aux[12];
                        if (kindP == 1)
                            finish_p1<false, S0, NL, Tile2dArgs>(a, pd, pm, p, lane, aux, T, i, t0, ghost && nchunks == 1,
                                                                 whole, own, carry, acc, q, nu, npn, zd, wB, yB);
                        else
                            finish_p1<true, S0, NL, Tile2dArgs>(a, pd, pm, p, lane, aux, T, i, t0, ghost && nchunks == 1,
                                                                whole, own, carry, acc, q, nu, npn, zd, wB, yB);
                    } else {
#pragma unroll
                        for (int c = 0; c < 2; ++c)
#pragma unroll
                            for (int h = 0; h < 2; ++h)
                                *reinterpret_cast<double2 *>(zd + c * kCT + h * (kCT / 2)) = make_double2(0.0, 0.0);
                    }
                }
                kindB = (orow1 && ocol) ? kindP : 0;
                kindP = 0;
                // (2) the chunk's first row step fences the z buffers against the previous
                // chunk's last reads
                if (m < ja) named_barrier_sync(1, kSeg * 32);
                // (3) start node m (z rows ja-1..jb on the mesh): independent of the z_u
                // exchange, so it runs before the barrier
                int kindC = 0;
                if (m <= jb && valid && m >= 0 && m < nrows) {
                    const double *aux = (NL == 1 && seg_uniform(a, m, i0 - 1)) ? aux_u
                                        : reinterpret_cast<const double *>(
                                              reinterpret_cast<const unsigned char *>(pm) + kXBytes) + warp * kAuxRec;
                    kindC = aux[13] == 1.0 ? 1 : 2;
                    kindP = kindC;
                    if (kindP == 2) T = cls_base + (ccx + 3 * axis_class(m, nrows)) * 7 * kCW;
                    if (kindP == 1) start<false, S0, Tile2dArgs>(a, pd, pm, p, lane, aux, T, acc, q);
                    else start<true, S0, Tile2dArgs>(a, pd, pm, p, lane, aux, T, acc, q);
                }
                // (4) every z_u of row m-1 published (a hardware barrier: waiting warps issue
                // nothing, where an mbarrier wait re-polled at every barrier event of the CTA,
                // ~24 polls per row step measured; it also orders the buffer's reuse two row
                // steps later): B^T contributions of row m-1's z_u to node m-2 (its +W slots;
                // then complete), node m-1 (0 slots), node m (-W slots)
                if (m >= ja) named_barrier_sync(2, kSeg * 32);
                if (m >= ja && ocol) {
                    // the z_u columns p-1, p (registers), p+1, each read once and applied to
                    // every node of this column that uses it, in ascending column order per node
                    // (node m-2: slots (+1, 0), (+1, +1); node m-1: (0, -1), (0, 0), (0, +1);
                    // node m: (-1, -1), (-1, 0))
                    const int kC = (kindC != 0 && m < jb) ? kindC : 0;
                    // the own column re-read too: holding it in registers across the barrier
                    // spills (4.84 -> 4.68 ms measured)
                    double zn[2][kT2], zo[2][kT2];
                    load_z(zo, zrow, p, lane);
                    if (kindA == 1 && kindB == 1 && kC == 1) {
                        // interior rows (the common case): one template path, no per-node branches
                        load_z(zn, zrow, p - 1, lane);
                        bt_col<0, -1, false, S0, Tile2dArgs>(a, zn, cls_base, btB);
                        bt_col<-1, -1, false, S0, Tile2dArgs>(a, zn, cls_base, btC);
                        bt_col<1, 0, false, S0, Tile2dArgs>(a, zo, cls_base, btA);
                        bt_col<0, 0, false, S0, Tile2dArgs>(a, zo, cls_base, btB);
                        bt_col<-1, 0, false, S0, Tile2dArgs>(a, zo, cls_base, btC);
                        load_z(zn, zrow, p + 1, lane);
                        bt_col<1, 1, false, S0, Tile2dArgs>(a, zn, cls_base, btA);
                        bt_col<0, 1, false, S0, Tile2dArgs>(a, zn, cls_base, btB);
                    } else {
                        const double *TA = cls_base + (ccx + 3 * axis_class(m - 2, nrows)) * 7 * kCW;
                        const double *TB = cls_base + (ccx + 3 * axis_class(m - 1, nrows)) * 7 * kCW;
                        const double *TC = cls_base + (ccx + 3 * axis_class(m, nrows)) * 7 * kCW;
                        load_z(zn, zrow, p - 1, lane);
                        bt_col_any<0, -1, S0, Tile2dArgs>(a, kindB, zn, TB, btB);
                        bt_col_any<-1, -1, S0, Tile2dArgs>(a, kC, zn, TC, btC);
                        bt_col_any<1, 0, S0, Tile2dArgs>(a, kindA, zo, TA, btA);
                        bt_col_any<0, 0, S0, Tile2dArgs>(a, kindB, zo, TB, btB);
                        bt_col_any<-1, 0, S0, Tile2dArgs>(a, kC, zo, TC, btC);
                        load_z(zn, zrow, p + 1, lane);
                        bt_col_any<1, 1, S0, Tile2dArgs>(a, kindA, zn, TA, btA);
                        bt_col_any<0, 1, S0, Tile2dArgs>(a, kindB, zn, TB, btB);
                    }
                    if (kindA != 0) finish_zp<Tile2dArgs>(a, (int64_t)(m - 2) * W + col, t0, whole, wA, btA, yA);
                }
                // rotate the pending rows: m-1 -> A, m -> B
                kindA = kindB;
                wA = wB;
#pragma unroll
                for (int tt = 0; tt < kT2; ++tt) {
                    btA[tt] = btB[tt];
                    yA[tt] = yB[tt];
                    btB[tt] = btC[tt];
                    btC[tt] = 0.0;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[sd]);   // row m-1 no longer needed
                sd = sm_;
                phd = phm;
            }
            if (lane == 0) mbar_arrive(&empty[sd]);       // row jb+1
            it += (uint32_t)(jb - ja + 4);
            // per-(CTA, column) norm partials, summed over this CTA's tiles in order (the
            // halo columns contribute zeros)
#pragma unroll
            for (int tt = 0; tt < kT2; ++tt) {
                const int t = t0 + (tt >> 1) * (kCT / 2) + (tt & 1);
                if (t < a.n_tl) {
                    double *dst = a.partial + (((int64_t)blockIdx.x * kSeg + warp) * a.n_tl + t) * 2;
                    const double u = t >= a.t_lo ? nu[tt] : 0.0, v = t >= a.t_lo ? npn[tt] : 0.0;
                    if (first) {
                        dst[0] = u;
                        dst[1] = v;
                    } else {
                        dst[0] = dst[0] + u;
                        dst[1] = dst[1] + v;
                    }
                }
            }
        }
    }
}


// ============================================================================
// Deferred first step (overlapped time-slab halo): the sweep of a rank
// r > 0 runs while the ghost x^k_{first-1} is still in flight, with a zero ghost, so
// only the pressure update of the slab's first local step is wrong (A' enters through
// q(t0-1) alone).  The sweep saves, per node, the pieces of that update the ghost does
// not touch (a.s0buf: acc_p, load_p, x_p^k and, for the fused P~1, B^T z_u); once the
// ghost has arrived this kernel (one thread per node) forms q(t0-1) in the sweep's order,
// r_p = (load_p + q) - acc_p and the sweep's update formula, so x^{k+1} is bitwise the
// undeferred value, and reduces the step's pressure-norm contributions per block.
// ============================================================================
template <bool S0, int MODE, int NL>
__global__ void __launch_bounds__(256) tile2d_step0_kernel(const Tile2dArgs a, double *part) {
    const int64_t N = a.n_nodes, P = a.pitch;
    const int W = (int)a.row_w;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double sp = 0.0;
    if (i < N) {
        const double *sv = a.s0buf + i * 8;   // acc_p, f_p, x_p^k, B^T z_u, D_S^{-1}, path flag
        const bool intr = sv[5] == 1.0;
        const double *T = a.cls + (axis_class((int)(i % W), W) + 3 * axis_class((int)(i / W), a.n_rows)) * 7 * kCW;
        const double qp = intr ? ghost_q<false, S0, Tile2dArgs>(a, i, T) : ghost_q<true, S0, Tile2dArgs>(a, i, T);
        const double dv = sv[4];
        double r = __dsub_rn(__fma_rn(a.s[a.t_off], sv[1], qp), sv[0]);   // epilogue_math's r_p
        if (dv == 0.0) r = 0.0;                 // Dirichlet pressure row (the epilogue's mask)
        sp = r * r;
        double xn;
        if constexpr (MODE == MODE_P1_FUSED) {   // finish_p1 / finish_zp
            const double wdv = a.omega * dv;
            const double y = fma(-wdv, r, sv[2]);
            xn = fma(wdv, sv[3], y);
        } else {                                 // P~2: z_p = -D_S^{-1} r_p
            xn = fma(a.omega, -(dv * r), sv[2]);
        }
        a.xn[(i * 3 + 2) * P + a.t_off] = xn;
        if (a.sendbuf && a.n_tl == 1) a.sendbuf[i * 3 + 2] = xn;
    }
    __shared__ double red[256];
    red[threadIdx.x] = sp;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

}  // namespace

int tile2d_seg() { return kSeg; }
int tile2d_seg_p1() { return kSegP1; }
int tile2d_chunk() { return kCT; }
int tile2d_max_rows() { return kMaxRR; }

int64_t tile2d_tiles(const Tile2dArgs &a) {
    const int seg = a.mode == MODE_P1_FUSED ? kSegP1 : kSeg;
    const int64_t n_seg = (a.row_w + seg - 1) / seg;
    const int64_t n_rr = (a.mode != MODE_P1_FUSED && a.n_rblk > 0) ? a.n_rblk
                                                                      : (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
    return n_seg * n_rr;
}

int64_t tile2d_groups(const Tile2dArgs &a, int grid) {
    const int64_t tiles = tile2d_tiles(a);
    return (tiles < grid ? tiles : grid) * kSeg;
}

cudaError_t tile2d_shape(int device, LaunchShape *out) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    constexpr int ML = kMaxLoads;
    for (auto fn : {tile2d_kernel<false, MODE_UPDATE_P2, 1>, tile2d_kernel<true, MODE_UPDATE_P2, 1>,
                    tile2d_kernel<false, MODE_P1_PASS1, 1>, tile2d_kernel<true, MODE_P1_PASS1, 1>,
                    tile2d_kernel<false, MODE_RESIDUAL, 1>, tile2d_kernel<true, MODE_RESIDUAL, 1>,
                    tile2d_kernel<false, MODE_PASS2, 1>, tile2d_kernel<true, MODE_PASS2, 1>,
                    tile2d_kernel<false, MODE_ZOUT, 1>, tile2d_kernel<true, MODE_ZOUT, 1>,
                    tile2d_kernel<false, MODE_MATVEC, 1>, tile2d_kernel<true, MODE_MATVEC, 1>,
                    tile2d_kernel<false, MODE_UPDATE_P2, ML>, tile2d_kernel<true, MODE_UPDATE_P2, ML>,
                    tile2d_kernel<false, MODE_P1_PASS1, ML>, tile2d_kernel<true, MODE_P1_PASS1, ML>,
                    tile2d_kernel<false, MODE_RESIDUAL, ML>, tile2d_kernel<true, MODE_RESIDUAL, ML>,
                    tile2d_kernel<false, MODE_ZOUT, ML>, tile2d_kernel<true, MODE_ZOUT, ML>,
                    tile2d_kernel<false, MODE_PASS2, ML>, tile2d_kernel<true, MODE_PASS2, ML>,
                    tile2d_kernel<false, MODE_MATVEC, ML>, tile2d_kernel<true, MODE_MATVEC, ML>,
                    tile2d_p1_kernel<false, 1>, tile2d_p1_kernel<true, 1>, tile2d_p1_kernel<false, ML>,
                    tile2d_p1_kernel<true, ML>}) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile2d_kernel<false, MODE_UPDATE_P2, 1>, kThreads2,
                                                      kSmemBytes);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    out->smem = kSmemBytes;
    return cudaSuccess;
}

cudaError_t launch_tile2d(const CUtensorMap &tmx, const Tile2dArgs &a, const LaunchShape &sh,
                          cudaStream_t st) {
    if (a.rows_per_tile < 1 || a.rows_per_tile > kMaxRR) return cudaErrorInvalidValue;
    const int64_t tiles = tile2d_tiles(a);
    const int grid = (int)(tiles < sh.grid ? tiles : sh.grid);   // = tile2d_groups / kSeg
    const dim3 block(kThreads2);
#define BIOT_T2(S0_, M_, NL_) tile2d_kernel<S0_, M_, NL_><<<grid, block, sh.smem, st>>>(tmx, a)
// NL = kMaxLoads also selects the aux-record layout (Lay), so every mode follows n_load
#define BIOT_T2L(S0_, M_) { if (a.n_load > 1) BIOT_T2(S0_, M_, kMaxLoads); else BIOT_T2(S0_, M_, 1); }
    if (a.mode == MODE_P1_FUSED) {
#define BIOT_T2P(S0_, NL_) tile2d_p1_kernel<S0_, NL_><<<grid, block, sh.smem, st>>>(tmx, a)
        if (a.n_load > 1) { if (a.s0) BIOT_T2P(true, kMaxLoads); else BIOT_T2P(false, kMaxLoads); }
        else { if (a.s0) BIOT_T2P(true, 1); else BIOT_T2P(false, 1); }
#undef BIOT_T2P
    } else if (a.mode == MODE_UPDATE_P2) { if (a.s0) BIOT_T2L(true, MODE_UPDATE_P2) else BIOT_T2L(false, MODE_UPDATE_P2) }
    else if (a.mode == MODE_P1_PASS1) { if (a.s0) BIOT_T2L(true, MODE_P1_PASS1) else BIOT_T2L(false, MODE_P1_PASS1) }
    else if (a.mode == MODE_PASS2) { if (a.s0) BIOT_T2L(true, MODE_PASS2) else BIOT_T2L(false, MODE_PASS2) }
    else if (a.mode == MODE_ZOUT) { if (a.s0) BIOT_T2L(true, MODE_ZOUT) else BIOT_T2L(false, MODE_ZOUT) }
    else if (a.mode == MODE_MATVEC) { if (a.s0) BIOT_T2L(true, MODE_MATVEC) else BIOT_T2L(false, MODE_MATVEC) }
    else { if (a.s0) BIOT_T2L(true, MODE_RESIDUAL) else BIOT_T2L(false, MODE_RESIDUAL) }
#undef BIOT_T2L
#undef BIOT_T2
    return cudaGetLastError();
}

int tile2d_step0_blocks(int64_t n_nodes) { return (int)((n_nodes + 255) / 256); }

cudaError_t launch_tile2d_step0(const Tile2dArgs &a, double *part, cudaStream_t st) {
    const int nb = tile2d_step0_blocks(a.n_nodes);
#define BIOT_S0(S0_, M_, NL_) tile2d_step0_kernel<S0_, M_, NL_><<<nb, 256, 0, st>>>(a, part)
#define BIOT_S0M(M_)                                                                                     \
    {                                                                                                    \
        if (a.n_load > 1) { if (a.s0) BIOT_S0(true, M_, kMaxLoads); else BIOT_S0(false, M_, kMaxLoads); } \
        else { if (a.s0) BIOT_S0(true, M_, 1); else BIOT_S0(false, M_, 1); }                              \
    }
    if (a.mode == MODE_P1_FUSED) BIOT_S0M(MODE_P1_FUSED)
    else if (a.mode == MODE_UPDATE_P2) BIOT_S0M(MODE_UPDATE_P2)
    else return cudaErrorInvalidValue;
#undef BIOT_S0M
#undef BIOT_S0
    return cudaGetLastError();
}

// box of the x tensor map: {time steps, tensor rows}
void tile2d_box(uint32_t *box) {
    box[0] = kCT;
    box[1] = (uint32_t)(kStrip * 3);
}

}  // namespace biot
