// TMA-pipelined 3D sweep kernel (structured n1^3 cube split into Kuhn
// tetrahedra, P1-P1, 15-slot BDIA stencil).  One outer iteration of the
// Jacobi-in-time inverted scheme (Alg. 2 as BASELINE.json
// reads it) with the block preconditioner (L238-262), the damped update and the
// per-step residual norms fused.
//
// The 3D path is fp64-bound (~267 FMAs per node and step against 64 bytes of
// x traffic), so the design goal is to keep the FP64 pipe busy with as few other
// instructions per DFMA as possible: the operator is not streamed per node but held
// as stencils -- the interior one in the kernel parameters (uniform-register
// operands, structural zeros skipped), the face / edge / corner ones (geometric
// classes) in shared memory -- and the x values come from shared memory staged by TMA.
//
// Work tile = a 4x3 (x, y) node patch x a z range, for every 64-step time chunk;
// every lane carries TWO consecutive steps (2l, 2l+1), so one 16-B shared-memory load
// brings both steps of a column component and every coefficient (an LDCU into a
// uniform register: DFMA takes no constant-bank operand on sm_100a) feeds two DFMAs.
// One lane of a producer warpgroup streams, per z plane, one 4D TMA box {64 steps,
// 6 x-nodes x 4 comps, 5 y-rows, 1 plane} (patch + halo; out-of-mesh positions are
// zero-filled) and the 12 patch nodes' aux records (kappa-dependent AA_pp per slot,
// load, preconditioner diagonals, path flag) into a 3-stage ring.  12 consumer warps
// (one node each) march z holding only two planes: at step m (planes m-1, m resident)
// a warp finishes its node of plane m-1 (the z+1 columns, from plane m, then the
// epilogue) and starts its node of plane m (z-1 and z columns); the partial sums ride
// in registers (setmaxnreg: 160 per consumer thread).  Measured (config 4): 4x4 patch,
// one step per lane, 32-step chunks: 4.87 ms; 4x2 patch, 8 warps, 4 stages: 4.18 ms; 4x3,
// 12 warps, 3 stages: 3.90 ms (the largest patch whose 3 stages fit 227 KB).  Every node's FMAs run in the
// fixed (dz, dy, dx) column order.
//
// Previous-step coupling (A' x_{n-1})_p: step 2l+1 uses the lane's own q(2l); step
// 2l uses lane l-1's q(2l-1) (one shuffle); lane 0 takes q(t0-1) from a shared-memory
// carry written by lane 31 when the same warp computed the node's previous chunk, and
// in chunk 0 recomputes it from the ghost vector x_{first-1} in the same FMA order (so
// iterates are bitwise independent of the time-slab split).
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

constexpr int kBX = 4, kBY = 3;            // patch (nodes): x, y (4x3: 12 consumer warps)
constexpr int kSX = kBX + 2, kSY = kBY + 2;   // staged incl. halo
constexpr int kNodes = kBX * kBY;          // consumer warps (one node each)
constexpr int kT3 = 2;                     // time steps per lane
constexpr int kTc = 32 * kT3;              // time steps per chunk
constexpr int kMaxZ = 24;                  // planes per tile (q carry capacity)
constexpr int kCW = Tile3dArgs::kClsW;     // doubles per class-stencil slot
constexpr int kClsD = 272;                 // doubles per class stencil in shared memory (15*18 padded)
constexpr int kClsLocal = 8;               // classes a tile can touch: 2 (x) x 2 (y) x 2 (z; one z face per tile)
constexpr uint32_t kAuxRec = Tile3dArgs::kAux;                                 // doubles per record
constexpr uint32_t kAuxRowBytes = kBX * kAuxRec * 8;                           // 768
constexpr uint32_t kAuxBytes = kBY * kAuxRowBytes;                             // 2304
// Shared-memory layout by mode.  The sweep modes stage all 4 components of every column
// of a plane (61 KB) in a 3-stage ring, one plane of lookahead.  The P~1 second pass
// (B^T z_u, memory-bound: ~45 FMAs per node and step) stages only z_u's 3 components
// through a 5D box {steps, comps 0-2, x, y, z} of the Z panel (46 KB; r_p, the fourth,
// is read per node from global memory) in a 4-stage ring: two planes in flight.
template <int MODE>
struct Lay3 {
    static constexpr int kNC = MODE == MODE_PASS2 ? 3 : 4;                              // staged components
    static constexpr int kStages = MODE == MODE_PASS2 ? 4 : 3;
    static constexpr uint32_t kXBytes = kSX * kSY * kNC * kTc * 8;                      // 61440 / 46080
    static constexpr uint32_t kStageBytes = (kXBytes + kAuxBytes + 127) / 128 * 128;  // 63744 / 48384
    static constexpr uint32_t kClsOff = kStages * kStageBytes;
    static constexpr uint32_t kCarryOff = kClsOff + kClsLocal * kClsD * 8;
    static constexpr uint32_t kSmemBytes = kCarryOff + kMaxZ * kNodes * 8;
};
constexpr uint32_t kSmemBytes = Lay3<MODE_UPDATE_P2>::kSmemBytes > Lay3<MODE_PASS2>::kSmemBytes
                                    ? Lay3<MODE_UPDATE_P2>::kSmemBytes : Lay3<MODE_PASS2>::kSmemBytes;
constexpr int kStagesMax = 4;
constexpr int kThreads3 = (kNodes + 4) * 32;
constexpr int kProducerRegs = 24, kConsumerRegs = 160;   // 4*32*24 + 12*32*160 <= 65536
static_assert(kSmemBytes + kNodes * kTc * 2 * 8 + 2 * kStagesMax * 8 <= 232448, "tile3d shared memory exceeds 227 KB");

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

// acc/q update of one interior node through slot s by the gathered column v, T steps
// (interior stencil in the kernel parameters, structural zeros skipped)
template <bool S0, int T>
__device__ __forceinline__ void fma_tmpl(double (&acc)[4][T], double (&q)[T], const Tile3dArgs &a, int s, double pp,
                                         const double (&v)[4][T]) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int e = c * 4 + cc;
            if (tmpl3_zero(s, e, S0)) continue;
            const double cf = (e == 15) ? pp : a.tmpl[s][e];
#pragma unroll
            for (int tt = 0; tt < T; ++tt) acc[c][tt] = fma(cf, v[cc][tt], acc[c][tt]);
        }
        const int eq = cc < 3 ? 12 + cc : 16;
        if (!tmpl3_zero(s, eq, S0)) {
#pragma unroll
            for (int tt = 0; tt < T; ++tt) q[tt] = fma(a.tmpl[s][eq], v[cc][tt], q[tt]);
        }
    }
}

// same through a class stencil (shared or global memory), stored column-major per slot
// (T[cc*4 + c] = AA[c][cc], T[16] = A'_pp)
template <int T>
__device__ __forceinline__ void fma_cls(double (&acc)[4][T], double (&q)[T], const double *Ts, double pp,
                                        const double (&v)[4][T]) {
    const double2 *T2 = reinterpret_cast<const double2 *>(Ts);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const double2 w0 = T2[cc * 2], w1 = T2[cc * 2 + 1];
        const double c3 = cc == 3 ? pp : w1.y, cq = cc < 3 ? w1.y : Ts[16];
#pragma unroll
        for (int tt = 0; tt < T; ++tt) {
            acc[0][tt] = fma(w0.x, v[cc][tt], acc[0][tt]);
            acc[1][tt] = fma(w0.y, v[cc][tt], acc[1][tt]);
            acc[2][tt] = fma(w1.x, v[cc][tt], acc[2][tt]);
            acc[3][tt] = fma(c3, v[cc][tt], acc[3][tt]);
            q[tt] = fma(cq, v[cc][tt], q[tt]);
        }
    }
}

// staged column (sx, sy) of a plane: component cc at + cc * kTc, the lane's two steps at + 2 lane
// (NC components staged per column)
template <int NC = 4>
__device__ __forceinline__ const double *col_ptr(const double *plane, int sx, int sy, int lane) {
    return plane + (sy * kSX + sx) * NC * kTc + 2 * lane;
}

__device__ __forceinline__ void load_col(double (&v)[4][kT3], const double *cp) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const double2 w = *reinterpret_cast<const double2 *>(cp + cc * kTc);
        v[cc][0] = w.x;
        v[cc][1] = w.y;
    }
}

// Columns of plane offset DZ (stage pl) for the warp's node, in (dy, dx) order.
template <int DZ, bool CLS, bool S0>
__device__ __forceinline__ void accum_plane(const Tile3dArgs &a, const double *pl, int sx, int sy, int lane,
                                            const double *aux, const double *TA, double (&acc)[4][kT3],
                                            double (&q)[kT3]) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const int s = slot_of(dx, dy, DZ);
            if (s < 0) continue;
            double v[4][kT3];
            load_col(v, col_ptr(pl, sx + dx, sy + dy, lane));
            if constexpr (CLS) fma_cls<kT3>(acc, q, TA + s * kCW, aux[s], v);
            else fma_tmpl<S0, kT3>(acc, q, a, s, aux[s], v);
        }
}

// scalar (one step) forms for the ghost and the deferred first step
template <bool S0>
__device__ __forceinline__ void fma_tmpl1(double (&acc)[4], double &q, const Tile3dArgs &a, int s, double pp,
                                          const double (&v)[4]) {
    double acc1[4][1] = {{acc[0]}, {acc[1]}, {acc[2]}, {acc[3]}}, q1[1] = {q}, v1[4][1] = {{v[0]}, {v[1]}, {v[2]}, {v[3]}};
    fma_tmpl<S0, 1>(acc1, q1, a, s, pp, v1);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = acc1[c][0];
    q = q1[0];
}
__device__ __forceinline__ void fma_cls1(double (&acc)[4], double &q, const double *Ts, double pp,
                                         const double (&v)[4]) {
    double acc1[4][1] = {{acc[0]}, {acc[1]}, {acc[2]}, {acc[3]}}, q1[1] = {q}, v1[4][1] = {{v[0]}, {v[1]}, {v[2]}, {v[3]}};
    fma_cls<1>(acc1, q1, Ts, pp, v1);
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = acc1[c][0];
    q = q1[0];
}

// q(t0-1) of node iA from the ghost x_{first-1} (stride: 1 for a vector, pitch for a
// panel column): the same walk and FMA order as the q accumulation
template <bool CLS, bool S0>
__device__ __forceinline__ double ghost_q(const double *ghost, int64_t n1, int64_t iA, const Tile3dArgs &a,
                                          const double *TA) {
    double g = 0.0;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
                const int s = slot_of(dx, dy, dz);
                if (s < 0) continue;
                const int64_t j = iA + ((int64_t)dz * n1 + dy) * n1 + dx;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const double xv = __ldg(ghost + (j * 4 + cc) * a.ghost_stride);
                    const int eq = cc < 3 ? 12 + cc : 16;
                    if constexpr (CLS) {
                        g = fma(cc < 3 ? TA[s * kCW + cc * 4 + 3] : TA[s * kCW + 16], xv, g);
                    } else {
                        if (!tmpl3_zero(s, eq, S0)) g = fma(a.tmpl[s][eq], xv, g);
                    }
                }
            }
    return g;
}

// 16-B store of the lane's two steps (t even), or the steps inside [t_lo, n_tl)
__device__ __forceinline__ void store2(double *dst, double v0, double v1, int t, int t_lo, int n_tl) {
    if (t >= t_lo && t + 1 < n_tl) {
        *reinterpret_cast<double2 *>(dst) = make_double2(v0, v1);
    } else {
        if (t < n_tl && t >= t_lo) dst[0] = v0;
        if (t + 1 < n_tl && t + 1 >= t_lo) dst[1] = v1;
    }
}

// Finish the node of plane m-1 at step m: z+1 columns from plane m (pu), the
// previous-step coupling, the epilogue with its own x and aux (plane m-1, po).
template <bool CLS, bool S0, int MODE>
__device__ __forceinline__ void finish(const Tile3dArgs &a, const double *po, const double *pu, const double *aux,
                                       int64_t iA, int sx, int sy, int lane, int t, bool ghost, double *carry,
                                       const double (&sv)[kT3], const double *TA, double (&acc)[4][kT3],
                                       double (&q)[kT3], double (&nu)[kT3], double (&npn)[kT3]) {
    accum_plane<1, CLS, S0>(a, pu, sx, sy, lane, aux, TA, acc, q);
    const int64_t P = a.pitch, row = iA * 4 * P + a.t_off + t;
    if constexpr (MODE == MODE_MATVEC) {
        // GMRES Arnoldi (R23): w = P~2^{-1} AA v, no time coupling, no load, no norms
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const double dv = aux[19 + c];
            const double w0 = c < 3 ? dv * acc[c][0] : a.p1_out ? acc[c][0] : -(dv * acc[c][0]);
            const double w1 = c < 3 ? dv * acc[c][1] : a.p1_out ? acc[c][1] : -(dv * acc[c][1]);
            store2(a.xn + row + c * P, w0, w1, t, a.t_lo, a.n_tl);
        }
        return;
    }
    // q(t-1): step t+1 uses q[0]; step t lane l-1's q[1]; lane 0 the carry / ghost
    double qp = __shfl_up_sync(0xffffffffu, q[1], 1);
    if (lane == 0) qp = ghost ? (a.ghost_zero ? 0.0 : ghost_q<CLS, S0>(a.ghost, a.n1, iA, a, TA)) : *carry;
    __syncwarp();
    if (lane == 31) *carry = q[1];
    double F[4], Dv[4], xs[4][kT3], outx[4][kT3], outz[4][kT3];
    const double *cp = col_ptr(po, sx, sy, lane);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        F[c] = aux[15 + c];
        Dv[c] = aux[19 + c];
        const double2 w = *reinterpret_cast<const double2 *>(cp + c * kTc);
        xs[c][0] = w.x;
        xs[c][1] = w.y;
    }
    epilogue_math<3, kT3, CLS, MODE == MODE_ZOUT>(a.omega, acc, q, qp, single_load(F, sv), Dv, xs, nu, npn, outx, outz,
                                                  !a.p1_out);
    if ((MODE == MODE_UPDATE_P2 || MODE == MODE_P1_PASS1) && a.s0buf && t == 0) {   // deferred first step
        double *sb = a.s0buf + iA * 8;
        sb[0] = acc[3][0];
        sb[1] = F[3];
        sb[2] = xs[3][0];
        sb[4] = Dv[3];
        sb[5] = aux[23];
    }
    if constexpr (MODE == MODE_ZOUT) {       // GMRES start: z = P~2^{-1} r, x untouched
#pragma unroll
        for (int c = 0; c < 4; ++c) store2(a.zbuf + row + c * P, outz[c][0], outz[c][1], t, a.t_lo, a.n_tl);
    } else if constexpr (MODE != MODE_RESIDUAL) {
        constexpr int ncw = MODE == MODE_UPDATE_P2 ? 4 : 3;   // P~1: pressure written by pass 2
#pragma unroll
        for (int c = 0; c < ncw; ++c) store2(a.xn + row + c * P, outx[c][0], outx[c][1], t, a.t_lo, a.n_tl);
        if constexpr (MODE == MODE_P1_PASS1) {
#pragma unroll
            for (int c = 0; c < 4; ++c) store2(a.zbuf + row + c * P, outz[c][0], outz[c][1], t, a.t_lo, a.n_tl);
        }
        if (a.sendbuf) {
            const int tl = a.n_tl - 1 - t;
            if (tl == 0 || tl == 1)
#pragma unroll
                for (int c = 0; c < ncw; ++c) a.sendbuf[iA * 4 + c] = tl == 0 ? outx[c][0] : outx[c][1];
        }
    }
}

// Start the node of plane m at step m: z-1 columns (plane m-1, pd), z columns (pm).
template <bool CLS, bool S0>
__device__ __forceinline__ void start(const Tile3dArgs &a, const double *pd, const double *pm, const double *aux,
                                      int sx, int sy, int lane, const double *TA, double (&acc)[4][kT3],
                                      double (&q)[kT3]) {
#pragma unroll
    for (int tt = 0; tt < kT3; ++tt) {
        q[tt] = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c][tt] = 0.0;
    }
    accum_plane<-1, CLS, S0>(a, pd, sx, sy, lane, aux, TA, acc, q);
    accum_plane<0, CLS, S0>(a, pm, sx, sy, lane, aux, TA, acc, q);
}

// ---- P~1 second pass (PAPER.md eq. p1: z_p = S~p^{-1} (B^T z_u - r_p)) on the Z panel
// staged like x: bt = (B^T z_u) over the slots in (dz, dy, dx) order, coefficients
// AA[p][u_cc] from the interior template (zeros skipped) or the class stencil
// (column-major: T[cc*4 + 3]).
template <int DZ, bool CLS, bool S0>
__device__ __forceinline__ void accum_plane_bt(const Tile3dArgs &a, const double *pl, int sx, int sy, int lane,
                                               const double *T, double (&bt)[kT3]) {
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const int s = slot_of(dx, dy, DZ);
            if (s < 0) continue;
            const double *cp = col_ptr<3>(pl, sx + dx, sy + dy, lane);
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                if constexpr (!CLS) {
                    if (tmpl3_zero(s, 12 + cc, S0)) continue;
                }
                const double cf = CLS ? T[s * kCW + cc * 4 + 3] : a.tmpl[s][12 + cc];
                const double2 w = *reinterpret_cast<const double2 *>(cp + cc * kTc);
                bt[0] = fma(cf, w.x, bt[0]);
                bt[1] = fma(cf, w.y, bt[1]);
            }
        }
}

template <bool CLS, bool S0>
__device__ __forceinline__ void finish_bt(const Tile3dArgs &a, const double *po, const double *pu,
                                          const double *aux, int64_t i, int sx, int sy, int lane, int t,
                                          const double *T, double (&bt)[kT3], const double (&xpre)[kT3],
                                          const double (&rpre)[kT3]) {
    accum_plane_bt<1, CLS, S0>(a, pu, sx, sy, lane, T, bt);
    const int64_t P = a.pitch, row = i * 4 * P + 3 * P + a.t_off + t;
    const double2 rp = make_double2(rpre[0], rpre[1]);   // r_p and x_p^k, prefetched when the
    const double x0 = xpre[0], x1 = xpre[1];              // node was started
    if (a.s0buf && t == 0) a.s0buf[i * 8 + 3] = bt[0];   // deferred first step
    const double v0 = fma(a.omega, aux[22] * (bt[0] - rp.x), x0);
    const double v1 = fma(a.omega, aux[22] * (bt[1] - rp.y), x1);
    store2(a.xn + row, v0, v1, t, a.t_lo, a.n_tl);
    if (a.sendbuf) {
        if (t == a.n_tl - 1) a.sendbuf[i * 4 + 3] = v0;
        if (t + 1 == a.n_tl - 1) a.sendbuf[i * 4 + 3] = v1;
    }
}

struct Geo3 {
    int n1, npx, npy, nzr, ntiles, nchunks;
    __device__ explicit Geo3(const Tile3dArgs &a) {
        n1 = a.n1;
        npx = (n1 + kBX - 1) / kBX;
        npy = (n1 + kBY - 1) / kBY;
        nzr = (n1 + a.z_rows - 1) / a.z_rows;
        ntiles = npx * npy * nzr;
        nchunks = (a.n_tl + kTc - 1) / kTc;
    }
    __device__ void decode(int tile, int zrows, int &x0, int &y0, int &za, int &zb) const {
        const int px = tile % npx, py = (tile / npx) % npy, zr = tile / (npx * npy);
        x0 = px * kBX;
        y0 = py * kBY;
        za = zr * zrows;
        zb = min(n1, za + zrows);
    }
};

__device__ __forceinline__ int axis_class(int v, int n1) { return v == 0 ? 0 : (v == n1 - 1 ? 2 : 1); }

template <bool S0, int MODE>
__global__ void __launch_bounds__(kThreads3, 1)
    tile3d_kernel(const __grid_constant__ CUtensorMap tmx, const Tile3dArgs a) {
    using L = Lay3<MODE>;
    constexpr int kStages = L::kStages;
    constexpr uint32_t kXBytes = L::kXBytes, kStageBytes = L::kStageBytes;
    constexpr uint32_t kClsOff = L::kClsOff, kCarryOff = L::kCarryOff;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[kStages], empty[kStages];
    __shared__ double red[kNodes][kTc][2];
    double *cls_sm = reinterpret_cast<double *>(smem + kClsOff);      // [kClsLocal][kClsD]
    double *qcarry = reinterpret_cast<double *>(smem + kCarryOff);    // [kMaxZ][kNodes]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Geo3 g(a);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNodes);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp >= kNodes) {
        // ------------------------------- producer -------------------------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
        if (warp == kNodes && lane == 0) {
            uint32_t it = 0;
            for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
                int x0, y0, za, zb;
                g.decode(tile, a.z_rows, x0, y0, za, zb);
                const int ny = min(kBY, g.n1 - y0);
                for (int chunk = 0; chunk < g.nchunks; ++chunk)
                    for (int z = za - 1; z <= zb; ++z, ++it) {
                        const int st = it % kStages;
                        if (it >= (uint32_t)kStages) mbar_wait_suspend(&empty[st], ((it / kStages) - 1) & 1);
                        unsigned char *base = smem + (size_t)st * kStageBytes;
                        const bool real = (z >= 0 && z < g.n1);
                        mbar_expect_tx(&full[st], kXBytes + (real ? (uint32_t)ny * kAuxRowBytes : 0u));
                        if constexpr (MODE == MODE_PASS2)
                            load_5d(base, &tmx, a.t_off + chunk * kTc, 0, x0 - 1, y0 - 1, z, &full[st]);
                        else
                            load_4d(base, &tmx, a.t_off + chunk * kTc, (x0 - 1) * 4, y0 - 1, z, &full[st]);
                        if (real)
                            for (int yy = 0; yy < ny; ++yy)
                                bulk_g2s(base + kXBytes + yy * kAuxRowBytes,
                                         a.aux + (((int64_t)z * g.n1 + y0 + yy) * g.n1 + x0) * kAuxRec,
                                         kAuxRowBytes, &full[st]);
                    }
            }
        }
        return;
    }

    // ------------------------------- consumers ------------------------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));
    const int px = warp % kBX, py = warp / kBX;
    const int sx = px + 1, sy = py + 1;
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
        int x0, y0, za, zb;
        g.decode(tile, a.z_rows, x0, y0, za, zb);
        // class stencils this tile can touch: x class in {cxl, cxl+1}, y in {cyl, cyl+1}, z in
        // {interior, the one z face the tile's plane range reaches (z_rows < n1)}; every
        // consumer is done with the previous tile's copy first
        const int cxl = x0 == 0 ? 0 : 1, cyl = y0 == 0 ? 0 : 1, czf = za == 0 ? 0 : 2;
        if (tile != (int)blockIdx.x) asm volatile("bar.sync 1, %0;" ::"r"(kNodes * 32) : "memory");
        for (int k = threadIdx.x; k < kClsLocal * kClsD; k += kNodes * 32) {
            const int L = k / kClsD, w = k - L * kClsD;
            const int cz = (L >> 2) ? czf : 1, cy = cyl + ((L >> 1) & 1), cx = cxl + (L & 1);
            if (cy <= 2 && cx <= 2 && w < 15 * kCW) cls_sm[k] = a.cls[(size_t)(cx + 3 * cy + 9 * cz) * (15 * kCW) + w];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kNodes * 32) : "memory");
        const int xA = x0 + px, y = y0 + py;
        const bool vA = xA < g.n1 && y < g.n1;
        const int ccxA = axis_class(min(xA, g.n1 - 1), g.n1), ccy = axis_class(min(y, g.n1 - 1), g.n1);
        for (int chunk = 0; chunk < g.nchunks; ++chunk) {
            const int t = chunk * kTc + 2 * lane;          // the lane's first step; second at t + 1
            double sv[kT3];
            sv[0] = t < a.n_tl ? a.s[a.t_off + t] : 0.0;
            sv[1] = t + 1 < a.n_tl ? a.s[a.t_off + t + 1] : 0.0;
            const bool ghost = chunk == 0;
            double nu[kT3] = {0.0, 0.0}, npn[kT3] = {0.0, 0.0};
            double acc[4][kT3], q[kT3];
            int kindP = 0;                       // pending node (plane m-1): 0 none, 1 interior, 2 class
            const double *TAp = cls_sm;
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
                                            (py * kBX + px) * kAuxRec;
                        const int64_t iA = ((int64_t)(m - 1) * g.n1 + y) * g.n1 + xA;
                        double *carry = qcarry + (m - 1 - za) * kNodes + warp;
                        if constexpr (MODE == MODE_PASS2) {   // bt rides in q
                            if (kindP == 1) finish_bt<false, S0>(a, pd, pm, aux, iA, sx, sy, lane, t, TAp, q, acc[3], acc[2]);
                            else finish_bt<true, S0>(a, pd, pm, aux, iA, sx, sy, lane, t, TAp, q, acc[3], acc[2]);
                        } else {
                            if (kindP == 1)
                                finish<false, S0, MODE>(a, pd, pm, aux, iA, sx, sy, lane, t, ghost, carry, sv, TAp, acc, q,
                                                        nu, npn);
                            else
                                finish<true, S0, MODE>(a, pd, pm, aux, iA, sx, sy, lane, t, ghost, carry, sv, TAp, acc, q,
                                                       nu, npn);
                        }
                    }
                    kindP = 0;
                    if (m < zb && vA) {          // start plane m
                        const double *aux = reinterpret_cast<const double *>(
                                                reinterpret_cast<const unsigned char *>(pm) + kXBytes) +
                                            (py * kBX + px) * kAuxRec;
                        kindP = aux[23] == 1.0 ? 1 : 2;
                        if (kindP == 2)
                            TAp = cls_sm + ((axis_class(m, g.n1) != 1) * 4 + (ccy - cyl) * 2 + ccxA - cxl) * kClsD;
                        if constexpr (MODE == MODE_PASS2) {
                            q[0] = q[1] = 0.0;
                            // prefetch x_p^k of the node (used at its finish, one plane later): its
                            // global-load latency then overlaps the plane march instead of stalling it
                            const int64_t rowp = (((int64_t)m * g.n1 + y) * g.n1 + xA) * 4 * a.pitch + 3 * a.pitch + a.t_off + t;
                            // (and r_p from the Z panel's fourth component, which the box does not stage)
                            acc[3][0] = acc[3][1] = acc[2][0] = acc[2][1] = 0.0;
                            if (t + 1 < a.n_tl) {
                                const double2 xv = __ldg(reinterpret_cast<const double2 *>(a.x + rowp));
                                const double2 rv = __ldg(reinterpret_cast<const double2 *>(a.zbuf + rowp));
                                acc[3][0] = xv.x;
                                acc[3][1] = xv.y;
                                acc[2][0] = rv.x;
                                acc[2][1] = rv.y;
                            } else if (t < a.n_tl) {
                                acc[3][0] = __ldg(a.x + rowp);
                                acc[2][0] = __ldg(a.zbuf + rowp);
                            }
                            if (kindP == 1) {
                                accum_plane_bt<-1, false, S0>(a, pd, sx, sy, lane, TAp, q);
                                accum_plane_bt<0, false, S0>(a, pm, sx, sy, lane, TAp, q);
                            } else {
                                accum_plane_bt<-1, true, S0>(a, pd, sx, sy, lane, TAp, q);
                                accum_plane_bt<0, true, S0>(a, pm, sx, sy, lane, TAp, q);
                            }
                        } else {
                            if (kindP == 1) start<false, S0>(a, pd, pm, aux, sx, sy, lane, TAp, acc, q);
                            else start<true, S0>(a, pd, pm, aux, sx, sy, lane, TAp, acc, q);
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
#pragma unroll
            for (int tt = 0; tt < kT3; ++tt) {
                red[warp][2 * lane + tt][0] = t + tt >= a.t_lo ? nu[tt] : 0.0;
                red[warp][2 * lane + tt][1] = t + tt >= a.t_lo ? npn[tt] : 0.0;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kNodes * 32) : "memory");
            for (int k = threadIdx.x; k < kTc * 2; k += kNodes * 32) {
                const int tl = k >> 1, part = k & 1;
                const int tt = chunk * kTc + tl;
                if (tt < a.n_tl) {
                    double sum = 0.0;
#pragma unroll
                    for (int w = 0; w < kNodes; ++w) sum += red[w][tl][part];
                    a.partial[((int64_t)tile * a.n_tl + tt) * 2 + part] = sum;
                }
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kNodes * 32) : "memory");
        }
    }
}

// Deferred first local step (overlapped time-slab halo; see tile2d_step0_kernel): the
// pressure update of the first local step completed from the ghost and the pieces the
// sweep saved (P~1 here is two-pass: pass 1 saves acc_p, load_p, x_p^k, pass 2 B^T z_u).
template <bool S0, int MODE>
__global__ void __launch_bounds__(256) tile3d_step0_kernel(const Tile3dArgs a, double *part) {
    const int64_t n1 = a.n1, N = a.n_nodes, P = a.pitch;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double sp = 0.0;
    if (i < N) {
        const double *sv = a.s0buf + i * 8;   // acc_p, f_p, x_p^k, B^T z_u, D_S^{-1}, path flag
        const bool intr = sv[5] == 1.0;
        const int x = (int)(i % n1), y = (int)((i / n1) % n1), z = (int)(i / (n1 * n1));
        const double *T = a.cls + (size_t)(axis_class(x, (int)n1) + 3 * axis_class(y, (int)n1) +
                                           9 * axis_class(z, (int)n1)) * (15 * kCW);
        const double qp = intr ? ghost_q<false, S0>(a.ghost, n1, i, a, T) : ghost_q<true, S0>(a.ghost, n1, i, a, T);
        const double dv = sv[4];
        double r = __dsub_rn(__fma_rn(a.s[a.t_off], sv[1], qp), sv[0]);   // epilogue_math's r_p
        if (dv == 0.0) r = 0.0;
        sp = r * r;
        const double xn = MODE == MODE_P1_PASS1 ? fma(a.omega, dv * (sv[3] - r), sv[2])   // finish_bt
                                                : fma(a.omega, -(dv * r), sv[2]);         // P~2
        a.xn[(i * 4 + 3) * P + a.t_off] = xn;
        if (a.sendbuf && a.n_tl == 1) a.sendbuf[i * 4 + 3] = xn;
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

int64_t tile3d_groups(const Tile3dArgs &a) {
    const int64_t npx = (a.n1 + kBX - 1) / kBX, npy = (a.n1 + kBY - 1) / kBY;
    const int64_t nzr = (a.n1 + a.z_rows - 1) / a.z_rows;
    return npx * npy * nzr;
}

int64_t tile3d_patches(int64_t n1) { return ((n1 + kBX - 1) / kBX) * ((n1 + kBY - 1) / kBY); }
int tile3d_chunk() { return kTc; }
int tile3d_max_zrows() { return kMaxZ; }   // and < n1: a tile reaches at most one z face
int tile3d_min_n1() { return kBX + 1; }

void tile3d_box(uint32_t *box) {
    box[0] = kTc;
    box[1] = kSX * 4;
    box[2] = kSY;
    box[3] = 1;
}

// box of the 5D Z-panel map {steps, component, x, y, z} the P~1 second pass stages
void tile3d_box_z(uint32_t *box) {
    box[0] = kTc;
    box[1] = Lay3<MODE_PASS2>::kNC;
    box[2] = kSX;
    box[3] = kSY;
    box[4] = 1;
}

cudaError_t tile3d_shape(int device, LaunchShape *out) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    for (auto fn : {tile3d_kernel<false, MODE_UPDATE_P2>, tile3d_kernel<true, MODE_UPDATE_P2>,
                    tile3d_kernel<false, MODE_P1_PASS1>, tile3d_kernel<true, MODE_P1_PASS1>,
                    tile3d_kernel<false, MODE_RESIDUAL>, tile3d_kernel<true, MODE_RESIDUAL>,
                    tile3d_kernel<false, MODE_PASS2>, tile3d_kernel<true, MODE_PASS2>,
                    tile3d_kernel<false, MODE_ZOUT>, tile3d_kernel<true, MODE_ZOUT>,
                    tile3d_kernel<false, MODE_MATVEC>, tile3d_kernel<true, MODE_MATVEC>}) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
        if (e != cudaSuccess) return e;
    }
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile3d_kernel<false, MODE_UPDATE_P2>, kThreads3,
                                                      kSmemBytes);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    out->smem = kSmemBytes;
    return cudaSuccess;
}

int tile3d_step0_blocks(int64_t n_nodes) { return (int)((n_nodes + 255) / 256); }

cudaError_t launch_tile3d_step0(const Tile3dArgs &a, double *part, cudaStream_t st) {
    const int nb = tile3d_step0_blocks(a.n_nodes);
    if (a.mode == MODE_UPDATE_P2) {
        if (a.s0) tile3d_step0_kernel<true, MODE_UPDATE_P2><<<nb, 256, 0, st>>>(a, part);
        else tile3d_step0_kernel<false, MODE_UPDATE_P2><<<nb, 256, 0, st>>>(a, part);
    } else if (a.mode == MODE_P1_PASS1) {
        if (a.s0) tile3d_step0_kernel<true, MODE_P1_PASS1><<<nb, 256, 0, st>>>(a, part);
        else tile3d_step0_kernel<false, MODE_P1_PASS1><<<nb, 256, 0, st>>>(a, part);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_tile3d(const CUtensorMap &tmx, const Tile3dArgs &a, const LaunchShape &sh,
                          cudaStream_t st) {
    if (a.z_rows < 1 || a.z_rows > kMaxZ || a.z_rows >= a.n1 || a.n1 < kBX + 1) return cudaErrorInvalidValue;
    const int64_t tiles = tile3d_groups(a);
    const int grid = (int)(tiles < sh.grid ? tiles : sh.grid);
    const dim3 block(kThreads3);
#define BIOT_T3(S0_, M_) tile3d_kernel<S0_, M_><<<grid, block, sh.smem, st>>>(tmx, a)
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
