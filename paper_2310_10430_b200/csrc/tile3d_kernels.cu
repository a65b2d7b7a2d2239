// TMA-pipelined 3D sweep kernel (structured n1^3 cube split into Kuhn
// tetrahedra, P1-P1, 15-slot BDIA stencil).  One outer iteration of the
// Jacobi-in-time inverted scheme (Alg. 2 as BASELINE.json
// reads it) with the block preconditioner (L238-262), the damped update and the
// per-step residual norms fused.
//
// The 3D path is fp64-bound (~267 FMAs per node and step against 64 bytes of
// x traffic), so the design goal is to keep the FP64 pipe busy: the operator is
// not streamed per node but held as stencils -- the interior one in the kernel
// parameters (uniform-register operands, structural zeros skipped), the face /
// edge / corner ones (geometric classes) in shared memory -- and the x values come
// from shared memory staged by TMA.
//
// Work tile = a 4x4 (x, y) node patch x a z range, for every 32-step time chunk
// (lane = one step).  One lane of a producer warpgroup streams, per z plane, one
// 4D TMA box {32 steps, 6 x-nodes x 4 comps, 6 y-rows, 1 plane} (patch + halo;
// out-of-mesh positions are zero-filled) and the 16 patch nodes' aux records
// (kappa-dependent AA_pp per slot, load, preconditioner diagonals, path flag) into
// a 5-stage ring.  16 consumer warps (one node each, R = 1) march z holding only
// two planes: at step m (planes m-1, m resident) a warp finishes its node of plane
// m-1 (the z+1 columns, from plane m, then the epilogue) and starts its node of
// plane m (z-1 and z columns); the partial sums ride in registers.  Every node's
// FMAs run in the fixed (dz, dy, dx) column order.  (R = 2, two x-adjacent nodes
// per warp, is kept as a template option; measured slower, see kConsumersOf.)
//
// Previous-step coupling (A' x_{n-1})_p: lane l uses q(t-1) of lane l-1 (one
// shuffle); lane 0 takes q(t0-1) from a shared-memory carry written by lane 31
// when the same warp computed the node's previous chunk, and in chunk 0 recomputes
// it from the ghost vector x_{first-1} in the same FMA order (so iterates are
// bitwise independent of the time-slab split).
#include <cuda.h>
#include <cstdint>
#include <cstdlib>

#include "node_update.cuh"
#include "sweep_kernels.cuh"
#include "tma_util.cuh"

namespace biot {

namespace {

using namespace dev;
using namespace tma;

constexpr int kB = 4;                      // patch edge (nodes)
constexpr int kSE = kB + 2;                // staged edge incl. halo
constexpr int kTc = 32;                    // time steps per chunk (one per lane)
// R = x-adjacent nodes per consumer warp (1 or 2); consumers = 16 / R.  R = 1 (16
// warps, 4 per scheduler) measured faster than R = 2 (8 warps, more operand reuse):
// config 4 5.23 vs 5.29 ms; R = 4 (4 warps) 8.5 ms, a 6x4 patch with R = 2 (12 warps,
// 3 stages) 5.93 ms.  The kernel is latency-bound at IPC ~2.5.
template <int R> constexpr int kConsumersOf = kB * kB / R;
template <int R> constexpr int kStagesOf = 5;
constexpr int kMaxZ = 24;                  // planes per tile (q carry capacity)
constexpr int kCW = Tile3dArgs::kClsW;     // doubles per class-stencil slot
constexpr int kClsD = 272;                 // doubles per class stencil in shared memory (15*18 padded)
constexpr int kClsLocal = 8;               // classes a tile can touch: 2 (x) x 2 (y) x 2 (z; one z face per tile)
constexpr int kRowD = kSE * 4 * kTc;       // doubles per staged y-row
constexpr uint32_t kXBytes = kSE * kRowD * 8;                                  // 36864
constexpr uint32_t kAuxRec = Tile3dArgs::kAux;                                 // doubles per record
constexpr uint32_t kAuxBytes = kB * kB * kAuxRec * 8;                          // 3072
constexpr uint32_t kStageBytes = (kXBytes + kAuxBytes + 127) / 128 * 128;      // 39936
template <int R> constexpr uint32_t kClsOffOf = kStagesOf<R> * kStageBytes;
template <int R> constexpr uint32_t kCarryOffOf = kClsOffOf<R> + kClsLocal * kClsD * 8;
template <int R> constexpr uint32_t kSmemBytesOf = kCarryOffOf<R> + kMaxZ * kB * kB * 8;

// (dx, dy, dz) of the 15 BDIA slots in storage order (offsets sorted ascending,
// self first): 0, -V-W-1, -V-W, -V-1, -V, -W-1, -W, -1, 1, W, W+1, V, V+1, V+W, V+W+1
__host__ __device__ constexpr int sdx(int s) {
    return (s == 1 || s == 3 || s == 5 || s == 7) ? -1 : (s == 8 || s == 10 || s == 12 || s == 14) ? 1 : 0;
}
__host__ __device__ constexpr int sdy(int s) {
    return (s == 1 || s == 2 || s == 5 || s == 6) ? -1 : (s == 9 || s == 10 || s == 13 || s == 14) ? 1 : 0;
}
__host__ __device__ constexpr int sdz(int s) { return (s >= 1 && s <= 4) ? -1 : (s >= 11) ? 1 : 0; }
__host__ __device__ constexpr int slot_of(int dx, int dy, int dz) {
    int r = -1;
    for (int s = 0; s < 15; ++s)
        if (sdx(s) == dx && sdy(s) == dy && sdz(s) == dz) r = s;
    return r;
}
// slots whose node pair shares only "diagonal" edges of the Kuhn split
__host__ __device__ constexpr bool diag_slot(int s) {
    return s == 1 || s == 2 || s == 3 || s == 5 || s == 10 || s == 12 || s == 13 || s == 14;
}
// Structural zeros of the interior stencil, entry e of the 17 (AA block 0..15,
// A'_pp = 16; A' u-entries are AA entries 12..14): the self block has no
// displacement-pressure coupling, diagonal neighbours no u_c-u_c coupling, and with
// S = 0 and uniform kappa no pressure-pressure coupling either.  Host-verified.
__host__ __device__ constexpr bool tmpl3_zero(int s, int e, bool s0) {
    return (s == 0) ? (e == 3 || e == 7 || e == 11 || e == 12 || e == 13 || e == 14)
                    : diag_slot(s) ? (e == 0 || e == 5 || e == 10 || (s0 && (e == 15 || e == 16))) : false;
}

__device__ __forceinline__ const double *col_ptr(const double *plane, int sx, int sy, int lane) {
    return plane + (sy * kSE + sx) * 4 * kTc + lane;
}

// acc/q update of one interior node through slot s by the gathered column v
// (interior stencil in the kernel parameters, structural zeros skipped)
template <bool S0>
__device__ __forceinline__ void fma_tmpl(double (&acc)[4], double &q, const Tile3dArgs &a, int s, double pp,
                                         const double (&v)[4]) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int e = c * 4 + cc;
            if (tmpl3_zero(s, e, S0)) continue;
            const double cf = (e == 15) ? pp : a.tmpl[s][e];
            acc[c] = fma(cf, v[cc], acc[c]);
        }
        const int eq = cc < 3 ? 12 + cc : 16;
        if (!tmpl3_zero(s, eq, S0)) q = fma(a.tmpl[s][eq], v[cc], q);
    }
}

// same through a class stencil in shared memory, stored column-major per slot
// (T[cc*4 + c] = AA[c][cc], T[16] = A'_pp): two 16-B loads per column feed 5 FMAs
__device__ __forceinline__ void fma_cls(double (&acc)[4], double &q, const double *T, double pp,
                                        const double (&v)[4]) {
    const double2 *T2 = reinterpret_cast<const double2 *>(T);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const double2 w0 = T2[cc * 2], w1 = T2[cc * 2 + 1];
        acc[0] = fma(w0.x, v[cc], acc[0]);
        acc[1] = fma(w0.y, v[cc], acc[1]);
        acc[2] = fma(w1.x, v[cc], acc[2]);
        acc[3] = fma(cc == 3 ? pp : w1.y, v[cc], acc[3]);
        q = fma(cc < 3 ? w1.y : T[16], v[cc], q);
    }
}

// Columns of plane offset DZ (stage pl) for the NN x-adjacent nodes A, B = A+1
// of one warp, in (dy, dx) order.  CLS: stencils TA/TB in shared memory, else the
// interior template.  aux: node A's record in its own plane's stage.
template <int DZ, int NN, bool CLS, bool S0>
__device__ __forceinline__ void accum_plane(const Tile3dArgs &a, const double *pl, int sx, int sy, int lane,
                                            const double *aux, const double *TA, const double *TB,
                                            double (&acc)[2][4], double (&q)[2]) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dxc = -1; dxc <= 2; ++dxc) {
            const int sA = slot_of(dxc, dy, DZ), sB = NN == 2 ? slot_of(dxc - 1, dy, DZ) : -1;
            if (sA < 0 && sB < 0) continue;
            const double *cp = col_ptr(pl, sx + dxc, sy + dy, lane);
            double v[4];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) v[cc] = cp[cc * kTc];
            if (sA >= 0) {
                if constexpr (CLS) fma_cls(acc[0], q[0], TA + sA * kCW, aux[sA], v);
                else fma_tmpl<S0>(acc[0], q[0], a, sA, aux[sA], v);
            }
            if (sB >= 0) {
                if constexpr (CLS) fma_cls(acc[1], q[1], TB + sB * kCW, aux[kAuxRec + sB], v);
                else fma_tmpl<S0>(acc[1], q[1], a, sB, aux[kAuxRec + sB], v);
            }
        }
}

// q(t0-1) of the NN nodes from the ghost x_{first-1}: the same walk and FMA order as
// the q accumulation (lane 0, chunk 0 only)
template <int NN, bool CLS, bool S0>
__device__ __forceinline__ void ghost_q(const double *ghost, int64_t n1, int64_t iA, const Tile3dArgs &a,
                                        const double *TA, const double *TB, double (&g)[2]) {
    g[0] = 0.0;
    g[1] = 0.0;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dxc = -1; dxc <= 2; ++dxc) {
                const int sA = slot_of(dxc, dy, dz), sB = NN == 2 ? slot_of(dxc - 1, dy, dz) : -1;
                if (sA < 0 && sB < 0) continue;
                const int64_t j = iA + ((int64_t)dz * n1 + dy) * n1 + dxc;
                double xv[4];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) xv[cc] = __ldg(ghost + (j * 4 + cc) * a.ghost_stride);
#pragma unroll
                for (int n = 0; n < NN; ++n) {
                    const int s = n == 0 ? sA : sB;
                    if (s < 0) continue;
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        const int eq = cc < 3 ? 12 + cc : 16;
                        if constexpr (CLS) {
                            const double *T = (n == 0 ? TA : TB) + s * kCW;
                            g[n] = fma(cc < 3 ? T[cc * 4 + 3] : T[16], xv[cc], g[n]);
                        } else {
                            if (!tmpl3_zero(s, eq, S0)) g[n] = fma(a.tmpl[s][eq], xv[cc], g[n]);
                        }
                    }
                }
            }
}

// Finish the NN nodes of plane m-1 at step m: z+1 columns from plane m (pu), the
// previous-step coupling, the epilogue with their own x and aux (plane m-1, po).
template <int NN, bool CLS, bool S0, int MODE>
__device__ __forceinline__ void finish(const Tile3dArgs &a, const double *po, const double *pu, const double *aux,
                                       int64_t iA, int sx, int sy, int lane, int t, bool ghost, double *carry,
                                       double sv, const double *TA, const double *TB, double (&acc)[2][4],
                                       double (&q)[2], double &nu, double &npn) {
    accum_plane<1, NN, CLS, S0>(a, pu, sx, sy, lane, aux, TA, TB, acc, q);
    if constexpr (MODE == MODE_MATVEC) {
        // GMRES Arnoldi (R23): w = P~2^{-1} AA v, no time coupling, no load, no norms
        if (t < a.n_tl && t >= a.t_lo) {
            const int64_t P = a.pitch;
#pragma unroll
            for (int n = 0; n < NN; ++n) {
                const double *ax = aux + n * kAuxRec;
                const int64_t row = (iA + n) * 4 * P + a.t_off + t;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const double dv = ax[19 + c];
                    a.xn[row + c * P] = c < 3 ? dv * acc[n][c] : -(dv * acc[n][c]);
                }
            }
        }
        return;
    }
    double qp[2];
#pragma unroll
    for (int n = 0; n < NN; ++n) qp[n] = __shfl_up_sync(0xffffffffu, q[n], 1);
    if (lane == 0) {
        if (ghost) {
            double gq[2];
            ghost_q<NN, CLS, S0>(a.ghost, a.n1, iA, a, TA, TB, gq);
#pragma unroll
            for (int n = 0; n < NN; ++n) qp[n] = gq[n];
        } else {
#pragma unroll
            for (int n = 0; n < NN; ++n) qp[n] = carry[n];
        }
    }
    __syncwarp();
    if (lane == kTc - 1) {
#pragma unroll
        for (int n = 0; n < NN; ++n) carry[n] = q[n];
    }
#pragma unroll
    for (int n = 0; n < NN; ++n) {
        const double *ax = aux + n * kAuxRec;
        double F[4], Dv[4], xs[4][1], acc1[4][1], q1[1] = {q[n]}, sv1[1] = {sv}, nu1[1] = {0.0}, np1[1] = {0.0};
        const double *cp = col_ptr(po, sx + n, sy, lane);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            F[c] = ax[15 + c];
            Dv[c] = ax[19 + c];
            xs[c][0] = cp[c * kTc];
            acc1[c][0] = acc[n][c];
        }
        double outx[4][1], outz[4][1];
        epilogue_math<3, 1, CLS, MODE == MODE_ZOUT>(a.omega, acc1, q1, qp[n], single_load(F, sv1), Dv, xs, nu1, np1,
                                                    outx, outz);
        nu += nu1[0];
        npn += np1[0];
        if constexpr (MODE == MODE_ZOUT) {       // GMRES start: z = P~2^{-1} r, x untouched
            if (t < a.n_tl && t >= a.t_lo) {
                const int64_t P = a.pitch, row = (iA + n) * 4 * P + a.t_off + t;
#pragma unroll
                for (int c = 0; c < 4; ++c) a.zbuf[row + c * P] = outz[c][0];
            }
        } else if constexpr (MODE != MODE_RESIDUAL) {   // stores through one row pointer per node
            constexpr int ncw = MODE == MODE_UPDATE_P2 ? 4 : 3;   // P~1: pressure written by pass 2
            if (t < a.n_tl && t >= a.t_lo) {
                const int64_t P = a.pitch, row = (iA + n) * 4 * P + a.t_off + t;
#pragma unroll
                for (int c = 0; c < ncw; ++c) a.xn[row + c * P] = outx[c][0];
                if constexpr (MODE == MODE_P1_PASS1) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) a.zbuf[row + c * P] = outz[c][0];
                }
                if (a.sendbuf && t == a.n_tl - 1) {
#pragma unroll
                    for (int c = 0; c < ncw; ++c) a.sendbuf[(iA + n) * 4 + c] = outx[c][0];
                }
            }
        }
    }
}

// Start the NN nodes of plane m at step m: z-1 columns (plane m-1, pd), z columns (pm).
template <int NN, bool CLS, bool S0>
__device__ __forceinline__ void start(const Tile3dArgs &a, const double *pd, const double *pm, const double *aux,
                                      int sx, int sy, int lane, const double *TA, const double *TB,
                                      double (&acc)[2][4], double (&q)[2]) {
#pragma unroll
    for (int n = 0; n < 2; ++n) {
        q[n] = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[n][c] = 0.0;
    }
    accum_plane<-1, NN, CLS, S0>(a, pd, sx, sy, lane, aux, TA, TB, acc, q);
    accum_plane<0, NN, CLS, S0>(a, pm, sx, sy, lane, aux, TA, TB, acc, q);
}

// ---- P~1 second pass (PAPER.md eq. p1: z_p = S~p^{-1} (B^T z_u - r_p)) on the Z panel
// staged like x: bt = (B^T z_u) over the slots in (dz, dy, dx) order, one node per warp
// (R = 1), coefficients AA[p][u_cc] from the interior template (zeros skipped) or the
// class stencil (column-major: T[cc*4 + 3]).
template <int DZ, bool CLS, bool S0>
__device__ __forceinline__ void accum_plane_bt(const Tile3dArgs &a, const double *pl, int sx, int sy, int lane,
                                               const double *T, double &bt) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const int s = slot_of(dx, dy, DZ);
            if (s < 0) continue;
            const double *cp = col_ptr(pl, sx + dx, sy + dy, lane);
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                if constexpr (!CLS) {
                    if (tmpl3_zero(s, 12 + cc, S0)) continue;
                }
                const double cf = CLS ? T[s * kCW + cc * 4 + 3] : a.tmpl[s][12 + cc];
                bt = fma(cf, cp[cc * kTc], bt);
            }
        }
}

template <bool CLS, bool S0>
__device__ __forceinline__ void finish_bt(const Tile3dArgs &a, const double *po, const double *pu,
                                          const double *aux, int64_t i, int sx, int sy, int lane, int t,
                                          const double *T, double bt) {
    accum_plane_bt<1, CLS, S0>(a, pu, sx, sy, lane, T, bt);
    if (t < a.n_tl && t >= a.t_lo) {
        const int64_t P = a.pitch, row = i * 4 * P + 3 * P + a.t_off + t;
        const double rp = col_ptr(po, sx, sy, lane)[3 * kTc];
        const double v = fma(a.omega, aux[22] * (bt - rp), __ldg(a.x + row));
        a.xn[row] = v;
        if (a.sendbuf && t == a.n_tl - 1) a.sendbuf[i * 4 + 3] = v;
    }
}

struct Geo3 {
    int n1, np, nzr, ntiles, nchunks;
    __device__ explicit Geo3(const Tile3dArgs &a) {
        n1 = a.n1;
        np = (n1 + kB - 1) / kB;
        nzr = (n1 + a.z_rows - 1) / a.z_rows;
        ntiles = np * np * nzr;
        nchunks = (a.n_tl + kTc - 1) / kTc;
    }
    __device__ void decode(int tile, int zrows, int &x0, int &y0, int &za, int &zb) const {
        const int px = tile % np, py = (tile / np) % np, zr = tile / (np * np);
        x0 = px * kB;
        y0 = py * kB;
        za = zr * zrows;
        zb = min(n1, za + zrows);
    }
};

__device__ __forceinline__ int axis_class(int v, int n1) { return v == 0 ? 0 : (v == n1 - 1 ? 2 : 1); }

// Kind of a warp's nodes in one plane: 0 nothing, 1 interior template, 2 class stencils
__device__ __forceinline__ int group_kind(bool vA, bool vB, const double *aux) {
    if (!vA) return 0;
    return (aux[23] == 1.0 && (!vB || aux[kAuxRec + 23] == 1.0)) ? 1 : 2;
}

template <int NN, bool S0, int MODE>
__device__ __forceinline__ void finish_any(int kind, const Tile3dArgs &a, const double *po, const double *pu,
                                           const double *aux, int64_t iA, int sx, int sy, int lane, int t,
                                           bool ghost, double *carry, double sv, const double *TA,
                                           const double *TB, double (&acc)[2][4], double (&q)[2], double &nu,
                                           double &npn) {
    if (kind == 1)
        finish<NN, false, S0, MODE>(a, po, pu, aux, iA, sx, sy, lane, t, ghost, carry, sv, TA, TB, acc, q, nu, npn);
    else if (a.dry != 2)
        finish<NN, true, S0, MODE>(a, po, pu, aux, iA, sx, sy, lane, t, ghost, carry, sv, TA, TB, acc, q, nu, npn);
}

template <int NN, bool S0>
__device__ __forceinline__ void start_any(int kind, const Tile3dArgs &a, const double *pd, const double *pm,
                                          const double *aux, int sx, int sy, int lane, const double *TA,
                                          const double *TB, double (&acc)[2][4], double (&q)[2]) {
    if (kind == 1)
        start<NN, false, S0>(a, pd, pm, aux, sx, sy, lane, TA, TB, acc, q);
    else if (a.dry != 2)
        start<NN, true, S0>(a, pd, pm, aux, sx, sy, lane, TA, TB, acc, q);
}

// Block = the consumer warpgroups + one producer warpgroup (only its first lane issues
// copies): the producer group hands its registers to the consumers (setmaxnreg), which
// run at 112 registers instead of the 96 an even split of 20 warps would leave them.
template <int R> constexpr int kThreadsOf = (kConsumersOf<R> + 4) * 32;
constexpr int kProducerRegs = 24, kConsumerRegs = 112;

template <bool S0, int R, int MODE>
__global__ void __launch_bounds__(kThreadsOf<R>, 1)
    tile3d_kernel(const __grid_constant__ CUtensorMap tmx, const Tile3dArgs a) {
    constexpr int kConsumers = kConsumersOf<R>, kStages = kStagesOf<R>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    __shared__ double red[kConsumers][kTc][2];
    double *cls_sm = reinterpret_cast<double *>(smem + kClsOffOf<R>);      // [kClsLocal][kClsD]
    double *qcarry = reinterpret_cast<double *>(smem + kCarryOffOf<R>);    // [kMaxZ][16]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Geo3 g(a);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp >= kConsumers) {
        // ------------------------------- producer -------------------------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
        if (warp == kConsumers && lane == 0) {
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
                int x0, y0, za, zb;
                g.decode(tile, a.z_rows, x0, y0, za, zb);
                const int ny = min(kB, g.n1 - y0);
                for (int chunk = 0; chunk < g.nchunks; ++chunk)
                    for (int z = za - 1; z <= zb; ++z, ++it) {
                        const int st = it % kStages;
                        if (it >= (uint32_t)kStages) mbar_wait_suspend(&empty[st], ((it / kStages) - 1) & 1);
                        unsigned char *base = smem + (size_t)st * kStageBytes;
                        const bool real = (z >= 0 && z < g.n1);
                        mbar_expect_tx(&full[st], kXBytes + (real ? (uint32_t)ny * kB * kAuxRec * 8 : 0u));
                        load_4d(base, &tmx, a.t_off + chunk * kTc, (x0 - 1) * 4, y0 - 1, z, &full[st]);
                        if (real)
                            for (int yy = 0; yy < ny; ++yy)
                                bulk_g2s(base + kXBytes + yy * kB * kAuxRec * 8,
                                         a.aux + (((int64_t)z * g.n1 + y0 + yy) * g.n1 + x0) * kAuxRec,
                                         kB * kAuxRec * 8, &full[st]);
                    }
            }
        }
        return;
    }

    // ------------------------------- consumers ------------------------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));
    const int px = (warp % (kB / R)) * R, py = warp / (kB / R);
    const int sx = px + 1, sy = py + 1;
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
        int x0, y0, za, zb;
        g.decode(tile, a.z_rows, x0, y0, za, zb);
        // class stencils this tile can touch: x class in {cxl, cxl+1}, y in {cyl, cyl+1}, z in
        // {interior, the one z face the tile's plane range reaches (z_rows < n1)}
        const int cxl = x0 == 0 ? 0 : 1, cyl = y0 == 0 ? 0 : 1, czf = za == 0 ? 0 : 2;
        // every consumer is done with the previous tile's class stencils before they are
        // overwritten (the norm-reduction barriers order this in the residual modes, but
        // the PASS2 / MATVEC modes have none: without this barrier a fast warp reloaded
        // the stencils under a slow one -- found by the full-K parity test of P~1, config 4)
        if (tile != (int)blockIdx.x) asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
        for (int k = threadIdx.x; k < kClsLocal * kClsD; k += kConsumers * 32) {
            const int L = k / kClsD, w = k - L * kClsD;
            const int cz = (L >> 2) ? czf : 1, cy = cyl + ((L >> 1) & 1), cx = cxl + (L & 1);
            if (cy <= 2 && cx <= 2 && w < 15 * kCW) cls_sm[k] = a.cls[(size_t)(cx + 3 * cy + 9 * cz) * (15 * kCW) + w];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
        const int xA = x0 + px, y = y0 + py;
        const bool vA = xA < g.n1 && y < g.n1, vB = R == 2 && xA + 1 < g.n1 && y < g.n1;
        const int ccxA = axis_class(xA, g.n1), ccxB = axis_class(xA + 1, g.n1), ccy = axis_class(y, g.n1);
        for (int chunk = 0; chunk < g.nchunks; ++chunk) {
            const int t = chunk * kTc + lane;
            const double sv = t < a.n_tl ? a.s[a.t_off + t] : 0.0;
            const bool ghost = chunk == 0;
            double nu = 0.0, npn = 0.0;
            double acc[2][4], q[2];
            int kindP = 0;                       // pending nodes (plane m-1)
            const double *TAp = cls_sm, *TBp = cls_sm;
            int sd = it % kStages;               // stage of plane m-1
            uint32_t phd = (it / kStages) & 1;
            mbar_wait_suspend(&full[sd], phd);
            for (int m = za; m <= zb; ++m) {
                const int sm_ = sd + 1 == kStages ? 0 : sd + 1;
                const uint32_t phm = sm_ == 0 ? phd ^ 1u : phd;
                mbar_wait_suspend(&full[sm_], phm);
                const double *pd = reinterpret_cast<const double *>(smem + (size_t)sd * kStageBytes);
                const double *pm = reinterpret_cast<const double *>(smem + (size_t)sm_ * kStageBytes);
                if (a.dry != 1) {
                    if (kindP != 0) {            // finish plane m-1
                        const double *aux = reinterpret_cast<const double *>(
                                                reinterpret_cast<const unsigned char *>(pd) + kXBytes) +
                                            (py * kB + px) * kAuxRec;
                        const int64_t iA = ((int64_t)(m - 1) * g.n1 + y) * g.n1 + xA;
                        double *carry = qcarry + (m - 1 - za) * (kB * kB) + py * kB + px;
                        if constexpr (MODE == MODE_PASS2) {   // bt rides in q[0]
                            if (kindP == 1) finish_bt<false, S0>(a, pd, pm, aux, iA, sx, sy, lane, t, TAp, q[0]);
                            else finish_bt<true, S0>(a, pd, pm, aux, iA, sx, sy, lane, t, TAp, q[0]);
                        } else if (vB) {
                            finish_any<2, S0, MODE>(kindP, a, pd, pm, aux, iA, sx, sy, lane, t, ghost, carry, sv, TAp,
                                              TBp, acc, q, nu, npn);
                        } else {
                            finish_any<1, S0, MODE>(kindP, a, pd, pm, aux, iA, sx, sy, lane, t, ghost, carry, sv, TAp,
                                              TBp, acc, q, nu, npn);
                        }
                    }
                    kindP = 0;
                    if (m < zb) {                // start plane m
                        const double *aux = reinterpret_cast<const double *>(
                                                reinterpret_cast<const unsigned char *>(pm) + kXBytes) +
                                            (py * kB + px) * kAuxRec;
                        kindP = group_kind(vA, vB, aux);
                        if (kindP == 2) {
                            const int base = (axis_class(m, g.n1) != 1) * 4 + (ccy - cyl) * 2;
                            TAp = cls_sm + (base + ccxA - cxl) * kClsD;
                            TBp = cls_sm + (base + (vB ? ccxB : ccxA) - cxl) * kClsD;
                        }
                        if constexpr (MODE == MODE_PASS2) {
                            if (kindP != 0) {
                                q[0] = 0.0;
                                if (kindP == 1) {
                                    accum_plane_bt<-1, false, S0>(a, pd, sx, sy, lane, TAp, q[0]);
                                    accum_plane_bt<0, false, S0>(a, pm, sx, sy, lane, TAp, q[0]);
                                } else {
                                    accum_plane_bt<-1, true, S0>(a, pd, sx, sy, lane, TAp, q[0]);
                                    accum_plane_bt<0, true, S0>(a, pm, sx, sy, lane, TAp, q[0]);
                                }
                            }
                        } else if (kindP != 0) {
                            if (vB)
                                start_any<2, S0>(kindP, a, pd, pm, aux, sx, sy, lane, TAp, TBp, acc, q);
                            else
                                start_any<1, S0>(kindP, a, pd, pm, aux, sx, sy, lane, TAp, TBp, acc, q);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[sd]);   // plane m-1 no longer needed
                sd = sm_;
                phd = phm;
            }
            if (lane == 0) mbar_arrive(&empty[sd]);       // plane zb
            it += (uint32_t)(zb - za + 2);
            // per-step norm partials of this (tile, chunk), fixed reduction order over warps
            if constexpr (MODE == MODE_PASS2 || MODE == MODE_MATVEC) continue;   // no norms in these passes
            red[warp][lane][0] = t >= a.t_lo ? nu : 0.0;
            red[warp][lane][1] = t >= a.t_lo ? npn : 0.0;
            asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
            if (threadIdx.x < kTc * 2) {
                const int tl = threadIdx.x >> 1, part = threadIdx.x & 1;
                const int tt = chunk * kTc + tl;
                if (tt < a.n_tl) {
                    double sum = 0.0;
#pragma unroll
                    for (int w = 0; w < kConsumers; ++w) sum += red[w][tl][part];
                    a.partial[((int64_t)tile * a.n_tl + tt) * 2 + part] = sum;
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
        }
    }
}

}  // namespace

int64_t tile3d_groups(const Tile3dArgs &a) {
    const int64_t np = (a.n1 + kB - 1) / kB;
    const int64_t nzr = (a.n1 + a.z_rows - 1) / a.z_rows;
    return np * np * nzr;
}

int tile3d_chunk() { return kTc; }
int tile3d_max_zrows() { return kMaxZ; }   // and < n1: a tile reaches at most one z face
int tile3d_min_n1() { return kB + 1; }

void tile3d_box(uint32_t *box) {
    box[0] = kTc;
    box[1] = kSE * 4;
    box[2] = kSE;
    box[3] = 1;
}

// One node per consumer warp (R = 1) is the configuration in use (see kConsumersOf).
constexpr int kR = 1;

cudaError_t tile3d_shape(int device, LaunchShape *out) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    for (auto fn : {tile3d_kernel<false, kR, MODE_UPDATE_P2>, tile3d_kernel<true, kR, MODE_UPDATE_P2>,
                    tile3d_kernel<false, kR, MODE_P1_PASS1>, tile3d_kernel<true, kR, MODE_P1_PASS1>,
                    tile3d_kernel<false, kR, MODE_RESIDUAL>, tile3d_kernel<true, kR, MODE_RESIDUAL>,
                    tile3d_kernel<false, kR, MODE_PASS2>, tile3d_kernel<true, kR, MODE_PASS2>,
                    tile3d_kernel<false, kR, MODE_ZOUT>, tile3d_kernel<true, kR, MODE_ZOUT>,
                    tile3d_kernel<false, kR, MODE_MATVEC>, tile3d_kernel<true, kR, MODE_MATVEC>}) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytesOf<kR>);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile3d_kernel<false, kR, MODE_UPDATE_P2>,
                                                      kThreadsOf<kR>, kSmemBytesOf<kR>);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    out->smem = kSmemBytesOf<kR>;
    return cudaSuccess;
}

cudaError_t launch_tile3d(const CUtensorMap &tmx, const Tile3dArgs &a, const LaunchShape &sh,
                          cudaStream_t st) {
    if (a.z_rows < 1 || a.z_rows > kMaxZ || a.z_rows >= a.n1 || a.n1 < kB + 1) return cudaErrorInvalidValue;
    const int64_t tiles = tile3d_groups(a);
    const int grid = (int)(tiles < sh.grid ? tiles : sh.grid);
    const dim3 block(kThreadsOf<kR>);
#define BIOT_T3(S0_, M_) tile3d_kernel<S0_, kR, M_><<<grid, block, sh.smem, st>>>(tmx, a)
    if (a.mode == MODE_UPDATE_P2) { if (a.s0) BIOT_T3(true, MODE_UPDATE_P2); else BIOT_T3(false, MODE_UPDATE_P2); }
    else if (a.mode == MODE_P1_PASS1) { if (a.s0) BIOT_T3(true, MODE_P1_PASS1); else BIOT_T3(false, MODE_P1_PASS1); }
    else if (a.mode == MODE_PASS2) { if (a.s0) BIOT_T3(true, MODE_PASS2); else BIOT_T3(false, MODE_PASS2); }
    else if (a.mode == MODE_ZOUT) { if (a.s0) BIOT_T3(true, MODE_ZOUT); else BIOT_T3(false, MODE_ZOUT); }
    else if (a.mode == MODE_MATVEC) { if (a.s0) BIOT_T3(true, MODE_MATVEC); else BIOT_T3(false, MODE_MATVEC); }
    else { if (a.s0) BIOT_T3(true, MODE_RESIDUAL); else BIOT_T3(false, MODE_RESIDUAL); }
#undef BIOT_T3
    return cudaGetLastError();
}

}  // namespace biot
