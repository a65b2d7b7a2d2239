// TMA-pipelined 2D sweep kernel (structured right-triangle meshes, BDIA slot
// order [0, -W-1, -W, -1, +1, +W, +W+1]).  One outer iteration of the
// Jacobi-in-time inverted scheme with the block
// preconditioner (L238-262), the damped update and the per-step norms fused.
//
// Work tile = SEG = 8R consecutive grid columns x 64 time steps x a range of
// grid rows, marched upward.  A producer warp streams, for every grid row r of
// the tile (plus the two halo rows), one TMA tensor box -- the (SEG+2)-node strip
// x 3 components x 66 time steps (t0-2 .. t0+63) of the space-time panel -- and
// one bulk copy of the SEG row nodes' aux records (kappa-dependent pressure
// entries, load, preconditioner diagonals) into a shared-memory ring
// (full/empty mbarriers).  Consumer warp w computes R horizontally adjacent
// nodes (r, i0 + R w + k) from shared memory only; for R = 2 their 14
// (node, neighbour) products need 10 distinct columns of rows r-1, r, r+1,
// walked once in a fixed order.  Every x value is read from HBM/L2 once per
// tile (+2/SEG halo from L2); compute warps issue no global loads except for
// boundary-class nodes.
//
// Interior nodes share one stencil (uniform lambda, mu, alpha, S and mesh):
// their blocks are kernel parameters (constant-bank operands); only the
// kappa-dependent pressure-pressure entry of AA varies per node (aux record).
// Structural zeros of that stencil are skipped at compile time (host-verified;
// fma(0, x, acc) == acc).  Nodes whose blocks differ from the template
// (boundary rows/columns, Dirichlet masking) read full blocks from global
// memory.  The epilogue is dev::node_epilogue, shared with every kernel; the
// neighbour order is the fixed column order below (deterministic, independent
// of the time-slab split; equal to the generic kernel to rounding).
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

constexpr int kT = 2;                       // time steps per lane
constexpr int kCh = 32 * kT;                // time steps per tile
constexpr int kChp = kCh + 2;               // + halo steps t0-2, t0-1
template <int R, int NC>
struct Geo {
    static constexpr int kSeg = NC * R;                               // row nodes per tile
    static constexpr int kStrip = kSeg + 2;                           // + halo columns
    static constexpr int kXRows = kStrip * 3;                         // tensor rows per stage
    static constexpr uint32_t kXBytes = kXRows * kChp * 8;
    static constexpr uint32_t kAuxOff = (kXBytes + 127) / 128 * 128;
    static constexpr uint32_t kAuxBytes = kSeg * Tile2dArgs::kAux * 8;
    static constexpr uint32_t kStageBytes = (kAuxOff + kAuxBytes + 127) / 128 * 128;
};

// (row delta, column delta) of the 7 BDIA slots in storage order
__device__ constexpr int kDr[7] = {0, -1, -1, 0, 0, 1, 1};
__device__ constexpr int kDc[7] = {0, -1, 0, -1, 1, 0, 1};

// Column walk of an R-node horizontal group A = (r, c), B = (r, c+1):
// row delta, column delta (from A), slot of A served, slot of B served (-1: none).
template <int R>
struct Walk;
template <>
struct Walk<1> {
    static constexpr int N = 7;
    __host__ __device__ static constexpr int dr(int k) { return k == 0 ? 0 : k <= 2 ? -1 : k <= 4 ? 0 : 1; }
    __host__ __device__ static constexpr int dc(int k) {
        return k == 0 ? 0 : k == 1 ? -1 : k == 2 ? 0 : k == 3 ? -1 : k == 4 ? 1 : k == 5 ? 0 : 1;
    }
    __host__ __device__ static constexpr int slot(int k, int node) { return node == 0 ? k : -1; }
};
template <>
struct Walk<2> {
    static constexpr int N = 10;
    __host__ __device__ static constexpr int dr(int k) { return k <= 2 ? -1 : k <= 6 ? 0 : 1; }
    __host__ __device__ static constexpr int dc(int k) {
        return k == 0 ? -1 : k == 1 ? 0 : k == 2 ? 1 : k == 3 ? -1 : k == 4 ? 0 : k == 5 ? 1 : k == 6 ? 2
               : k == 7 ? 0 : k == 8 ? 1 : 2;
    }
    __host__ __device__ static constexpr int slot(int k, int node) {
        // A: k -> 1 2 - 3 0 4 - 5 6 - ;  B: k -> - 1 2 - 3 0 4 - 5 6
        return node == 0 ? (k == 0 ? 1 : k == 1 ? 2 : k == 2 ? -1 : k == 3 ? 3 : k == 4 ? 0 : k == 5 ? 4
                            : k == 6 ? -1 : k == 7 ? 5 : k == 8 ? 6 : -1)
                         : (k == 0 ? -1 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? -1 : k == 4 ? 3 : k == 5 ? 0
                            : k == 6 ? 4 : k == 7 ? -1 : k == 8 ? 5 : 6);
    }
};

// Structural zeros of the interior right-triangle stencil, entry e = c*3+cc of the
// AA block (e < 9) or 9 = A'_pp: the self block has no displacement-pressure
// coupling, the diagonal (SW/NE) neighbours have no u_x-u_x / u_y-u_y coupling,
// and with S = 0 no pressure-pressure coupling either (L is the 5-point stencil).
__host__ __device__ constexpr bool tmpl_zero(int s, int e, bool s0) {
    return (s == 0) ? (e == 2 || e == 5 || e == 6 || e == 7)
                    : (s == 1 || s == 6) ? (e == 0 || e == 4 || (s0 && (e == 8 || e == 9))) : false;
}

using namespace tma;

template <int SEG>
struct TileGeom {
    int64_t n_seg, n_jr, n_chunks, n_tiles;
    __device__ explicit TileGeom(const Tile2dArgs &a) {
        n_seg = (a.row_w + SEG - 1) / SEG;
        n_jr = (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
        n_chunks = (a.n_tl + kCh - 1) / kCh;
        n_tiles = n_seg * n_jr * n_chunks;
    }
};

// x of one column (3 components x kT steps) from a ring stage
__device__ __forceinline__ void load_col(double (&v)[3][kT], const double *colp) {
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const double2 w2 = *reinterpret_cast<const double2 *>(colp + cc * kChp);
        v[cc][0] = w2.x;
        v[cc][1] = w2.y;
    }
}

// interior block coefficient (template, with the per-node pp entry)
__device__ __forceinline__ double tcoef(const Tile2dArgs &a, int s, int e, double pp) {
    return (e == 8) ? pp : a.tmpl[s][e];
}

// acc/q update of one interior node by gathered column v through slot s
template <bool S0>
__device__ __forceinline__ void fma_interior(double (&acc)[3][kT], double (&q)[kT], const Tile2dArgs &a, int s,
                                             double pp, const double (&v)[3][kT]) {
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int e = c * 3 + cc;
            if (tmpl_zero(s, e, S0)) continue;
            const double cf = tcoef(a, s, e, pp);
#pragma unroll
            for (int tt = 0; tt < kT; ++tt) acc[c][tt] = fma(cf, v[cc][tt], acc[c][tt]);
        }
        const int eq = (cc < 2) ? 6 + cc : 9;
        if (!tmpl_zero(s, eq, S0)) {
#pragma unroll
            for (int tt = 0; tt < kT; ++tt) q[tt] = fma(a.tmpl[s][eq], v[cc][tt], q[tt]);
        }
    }
}

// R interior nodes of one row (warp group): walk the union columns once.
template <int R, bool GHOST, bool S0>
__device__ __forceinline__ void group_interior(const Tile2dArgs &a, const double *r0, const double *r1,
                                               const double *r2, const double *aux0, int j,
                                               int64_t col0, int p0, int lane, int t0, const double (&sv)[kT],
                                               double (&nu)[kT], double (&npn)[kT]) {
    using Wk = Walk<R>;
    const double *rows[3] = {r0, r1, r2};
    const int64_t W = a.row_w;
    double acc[R][3][kT], q[R][kT];
#pragma unroll
    for (int n = 0; n < R; ++n)
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
            q[n][tt] = 0.0;
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[n][c][tt] = 0.0;
        }
#pragma unroll
    for (int k = 0; k < Wk::N; ++k) {
        double v[3][kT];
        load_col(v, rows[1 + Wk::dr(k)] + ((p0 + Wk::dc(k)) * 3) * kChp + 2 + lane * kT);
#pragma unroll
        for (int n = 0; n < R; ++n) {
            const int s = Wk::slot(k, n);
            if (s < 0) continue;
            fma_interior<S0>(acc[n], q[n], a, s, aux0[n * Tile2dArgs::kAux + s], v);
        }
    }
    double qp[R];
#pragma unroll
    for (int n = 0; n < R; ++n) qp[n] = __shfl_up_sync(0xffffffffu, q[n][kT - 1], 1);
    if (lane == 0) {                 // q(t0-1): same order, x at t0-1 (ring) or the ghost
        double g[R];
#pragma unroll
        for (int n = 0; n < R; ++n) g[n] = 0.0;
#pragma unroll
        for (int k = 0; k < Wk::N; ++k) {
            double xv[3];
            if constexpr (GHOST) {
                const int64_t jn = (int64_t)(j + Wk::dr(k)) * W + col0 + Wk::dc(k);
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) xv[cc] = __ldg(a.ghost + jn * 3 + cc);
            } else {
                const double *colp = rows[1 + Wk::dr(k)] + ((p0 + Wk::dc(k)) * 3) * kChp + 1;
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) xv[cc] = colp[cc * kChp];
            }
#pragma unroll
            for (int n = 0; n < R; ++n) {
                const int s = Wk::slot(k, n);
                if (s < 0) continue;
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    const int eq = (cc < 2) ? 6 + cc : 9;
                    if (!tmpl_zero(s, eq, S0)) g[n] = fma(a.tmpl[s][eq], xv[cc], g[n]);
                }
            }
        }
#pragma unroll
        for (int n = 0; n < R; ++n) qp[n] = g[n];
    }
#pragma unroll
    for (int n = 0; n < R; ++n) {
        const double *aux = aux0 + n * Tile2dArgs::kAux;
        double F[3], Dv[3], xs[3][kT];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            F[c] = aux[7 + c];
            Dv[c] = aux[10 + c];
        }
        load_col(xs, rows[1] + ((p0 + n) * 3) * kChp + 2 + lane * kT);
        node_epilogue<2, kT>(a, (int64_t)j * W + col0 + n, t0, acc[n], q[n], qp[n], F, Dv, xs, sv, nu, npn);
    }
}

// Everything the boundary path reads from the kernel parameters (so the
// out-of-line function does not force the whole parameter block into local
// memory); also what node_epilogue needs.
struct BArgs {
    double *xn, *zbuf, *sendbuf;
    const double *blk, *ghost;
    int64_t pitch, row_w;
    int64_t off[7];
    int32_t n_tl, mode;
    double omega;
};

struct Norms2 {
    double nu[kT], npn[kT];
};

// Boundary-class node at strip position p of row j: full blocks from global
// memory, slot order.  Rare (domain edges, Dirichlet neighbourhoods): kept out of
// line so its register footprint does not burden the interior path.
__device__ __noinline__ Norms2 node_boundary(const BArgs &a, const double *r0, const double *r1,
                                             const double *r2, const double *aux, int j, int64_t col, int p,
                                             int lane, int t0, double sv0, double sv1) {
    const double *rows[3] = {r0, r1, r2};
    const double sv[kT] = {sv0, sv1};
    double nu[kT] = {0.0, 0.0}, npn[kT] = {0.0, 0.0};
    const int64_t i = (int64_t)j * a.row_w + col;
    const double *gb = a.blk + i * (7 * 10);
    double acc[3][kT], q[kT];
#pragma unroll
    for (int tt = 0; tt < kT; ++tt) {
        q[tt] = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c][tt] = 0.0;
    }
#pragma unroll 1
    for (int s = 0; s < 7; ++s) {
        double v[3][kT];
        load_col(v, rows[1 + kDr[s]] + ((p + kDc[s]) * 3) * kChp + 2 + lane * kT);
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double cf = __ldg(gb + s * 10 + c * 3 + cc);
#pragma unroll
                for (int tt = 0; tt < kT; ++tt) acc[c][tt] = fma(cf, v[cc][tt], acc[c][tt]);
            }
            const double qc = __ldg(gb + s * 10 + ((cc < 2) ? 6 + cc : 9));
#pragma unroll
            for (int tt = 0; tt < kT; ++tt) q[tt] = fma(qc, v[cc][tt], q[tt]);
        }
    }
    double qp = __shfl_up_sync(0xffffffffu, q[kT - 1], 1);
    if (lane == 0) {
        double g = 0.0;
        for (int s = 0; s < 7; ++s) {
            const int64_t jn = i + a.off[s];
            const double *colp = rows[1 + kDr[s]] + ((p + kDc[s]) * 3) * kChp + 1;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) {
                const double qc = __ldg(gb + s * 10 + ((cc < 2) ? 6 + cc : 9));
                const double xv = (t0 == 0) ? __ldg(a.ghost + jn * 3 + cc) : colp[cc * kChp];
                g = fma(qc, xv, g);
            }
        }
        qp = g;
    }
    double F[3], Dv[3], xs[3][kT];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        F[c] = aux[7 + c];
        Dv[c] = aux[10 + c];
    }
    load_col(xs, rows[1] + (p * 3) * kChp + 2 + lane * kT);
    node_epilogue<2, kT>(a, i, t0, acc, q, qp, F, Dv, xs, sv, nu, npn);
    Norms2 o;
#pragma unroll
    for (int tt = 0; tt < kT; ++tt) {
        o.nu[tt] = nu[tt];
        o.npn[tt] = npn[tt];
    }
    return o;
}

template <int R, int NC, int STAGES, int MAXREG>
__global__ void __launch_bounds__((NC + 1) * 32) __maxnreg__(MAXREG)
    tile2d_kernel(const __grid_constant__ CUtensorMap tmx, const Tile2dArgs a) {
    using G = Geo<R, NC>;
    constexpr int kConsumers = NC;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[STAGES], empty[STAGES];
    __shared__ double red[kConsumers][kCh][2];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TileGeom<G::kSeg> g(a);
    const int64_t W = a.row_w;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kConsumers) {
        // ------------------------------- producer -------------------------------
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t tile = blockIdx.x; tile < g.n_tiles; tile += gridDim.x) {
                const int chunk = (int)(tile % g.n_chunks);
                const int64_t grp = tile / g.n_chunks;
                const int64_t seg = grp % g.n_seg, jr = grp / g.n_seg;
                const int ja = (int)(jr * a.rows_per_tile);
                const int jb = min(a.n_rows, ja + a.rows_per_tile);
                const int64_t i0 = seg * G::kSeg;
                for (int r = ja - 1; r <= jb; ++r, ++it) {
                    const int st = it % STAGES;
                    if (it >= (uint32_t)STAGES) mbar_wait_sleep(&empty[st], ((it / STAGES) - 1) & 1);
                    unsigned char *base = smem + (size_t)st * G::kStageBytes;
                    const bool real = (r >= 0 && r < a.n_rows);
                    mbar_expect_tx(&full[st], G::kXBytes + (real ? G::kAuxBytes : 0u));
                    const int64_t node0 = (int64_t)r * W + i0 - 1;
                    load_2d(base, &tmx, chunk * kCh - 2, (int)((node0 + a.pad_nodes) * 3), &full[st]);
                    if (real)
                        bulk_g2s(base + G::kAuxOff, a.aux + ((int64_t)r * W + i0) * Tile2dArgs::kAux, G::kAuxBytes,
                                 &full[st]);
                }
            }
        }
        return;
    }

    // ------------------------------- consumers ------------------------------
    uint32_t it = 0;
    const int p0 = 1 + R * warp;              // strip position of the warp's first node
    for (int64_t tile = blockIdx.x; tile < g.n_tiles; tile += gridDim.x) {
        const int chunk = (int)(tile % g.n_chunks);
        const int64_t grp = tile / g.n_chunks;
        const int64_t seg = grp % g.n_seg, jr = grp / g.n_seg;
        const int ja = (int)(jr * a.rows_per_tile);
        const int jb = min(a.n_rows, ja + a.rows_per_tile);
        const int64_t col0 = seg * G::kSeg + R * warp;
        const int64_t rem = W - col0;
        const int nvalid = rem <= 0 ? 0 : (rem >= R ? R : (int)rem);
        const int t0 = chunk * kCh + lane * kT;
        double nu[kT], npn[kT], sv[kT];
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
            nu[tt] = 0.0;
            npn[tt] = 0.0;
            sv[tt] = (t0 + tt < a.n_tl) ? a.s[t0 + tt] : 0.0;
        }
        // ring positions (stage index, phase parity) of rows j-1, j, j+1, advanced
        // incrementally (no division by the stage count in the row loop)
        int s0i = it % STAGES;
        uint32_t ph0 = (it / STAGES) & 1;
        int s1i = s0i + 1 == STAGES ? 0 : s0i + 1;
        uint32_t ph1 = s1i == 0 ? ph0 ^ 1u : ph0;
        mbar_wait(&full[s0i], ph0);
        mbar_wait(&full[s1i], ph1);
        for (int j = ja; j < jb; ++j) {
            const int s2i = s1i + 1 == STAGES ? 0 : s1i + 1;
            const uint32_t ph2 = s2i == 0 ? ph1 ^ 1u : ph1;
            mbar_wait(&full[s2i], ph2);
            if (nvalid > 0 && !a.dry) {
                const double *r0 = reinterpret_cast<const double *>(smem + (size_t)s0i * G::kStageBytes);
                const double *r1 = reinterpret_cast<const double *>(smem + (size_t)s1i * G::kStageBytes);
                const double *r2 = reinterpret_cast<const double *>(smem + (size_t)s2i * G::kStageBytes);
                const double *aux0 = reinterpret_cast<const double *>(
                                         reinterpret_cast<const unsigned char *>(r1) + G::kAuxOff) +
                                     (R * warp) * Tile2dArgs::kAux;
                bool interior = (nvalid == R);   // partial groups (last segment) take the generic path
#pragma unroll
                for (int n = 0; n < R; ++n) interior &= aux0[n * Tile2dArgs::kAux + 13] != 0.0;
                if (interior) {
                    if (chunk == 0) {
                        if (a.s0)
                            group_interior<R, true, true>(a, r0, r1, r2, aux0, j, col0, p0, lane, t0, sv, nu, npn);
                        else
                            group_interior<R, true, false>(a, r0, r1, r2, aux0, j, col0, p0, lane, t0, sv, nu, npn);
                    } else {
                        if (a.s0)
                            group_interior<R, false, true>(a, r0, r1, r2, aux0, j, col0, p0, lane, t0, sv, nu, npn);
                        else
                            group_interior<R, false, false>(a, r0, r1, r2, aux0, j, col0, p0, lane, t0, sv, nu, npn);
                    }
                } else {
                    BArgs b;
                    b.xn = a.xn; b.zbuf = a.zbuf; b.sendbuf = a.sendbuf; b.blk = a.blk; b.ghost = a.ghost;
                    b.pitch = a.pitch; b.row_w = a.row_w; b.n_tl = a.n_tl; b.mode = a.mode; b.omega = a.omega;
#pragma unroll
                    for (int q = 0; q < 7; ++q) b.off[q] = a.off[q];
                    for (int n = 0; n < nvalid; ++n) {
                        const Norms2 o = node_boundary(b, r0, r1, r2, aux0 + n * Tile2dArgs::kAux, j, col0 + n,
                                                       p0 + n, lane, t0, sv[0], sv[1]);
#pragma unroll
                        for (int tt = 0; tt < kT; ++tt) {
                            nu[tt] += o.nu[tt];
                            npn[tt] += o.npn[tt];
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s0i]);   // row j-1 no longer needed
            s0i = s1i;
            ph0 = ph1;
            s1i = s2i;
            ph1 = ph2;
        }
        if (lane == 0) {                        // rows jb-1 and jb
            mbar_arrive(&empty[s0i]);
            mbar_arrive(&empty[s1i]);
        }
        it += (uint32_t)(jb - ja + 2);
        // per-step norm partials of this tile (fixed reduction order over warps)
#pragma unroll
        for (int tt = 0; tt < kT; ++tt) {
            red[warp][lane * kT + tt][0] = nu[tt];
            red[warp][lane * kT + tt][1] = npn[tt];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
        for (int k = threadIdx.x; k < kCh * 2; k += kConsumers * 32) {
            const int tl = k >> 1, part = k & 1;
            const int t = chunk * kCh + tl;
            if (t < a.n_tl) {
                double sum = 0.0;
#pragma unroll
                for (int w = 0; w < kConsumers; ++w) sum += red[w][tl][part];
                a.partial[(grp * a.n_tl + t) * 2 + part] = sum;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers * 32) : "memory");
    }
}

struct TileCfg {
    int r, nc, stages, maxreg;
};

TileCfg tile_cfg() {
    TileCfg c{1, 15, 6, 128};
    if (const char *e = std::getenv("BIOT_TILE_CFG")) {   // "r,consumers,stages,maxreg"
        int r = 0, nc = 0, st = 0, mr = 0;
        if (std::sscanf(e, "%d,%d,%d,%d", &r, &nc, &st, &mr) == 4) c = TileCfg{r, nc, st, mr};
    }
    return c;
}

using TileFn = void (*)(const CUtensorMap, const Tile2dArgs);

TileFn tile_fn(TileCfg c) {
#define BIOT_TCFG(R_, NC_, ST_, MR_) \
    if (c.r == R_ && c.nc == NC_ && c.stages == ST_ && c.maxreg == MR_) return tile2d_kernel<R_, NC_, ST_, MR_>;
    BIOT_TCFG(2, 8, 6, 168)
    BIOT_TCFG(1, 8, 6, 168)
    BIOT_TCFG(1, 12, 6, 128)
    BIOT_TCFG(1, 15, 6, 128)
    BIOT_TCFG(1, 15, 7, 128)
    BIOT_TCFG(1, 15, 6, 120)
    BIOT_TCFG(1, 19, 5, 96)
    BIOT_TCFG(1, 11, 6, 168)
    BIOT_TCFG(2, 7, 6, 168)
    BIOT_TCFG(2, 11, 5, 128)
#undef BIOT_TCFG
    return nullptr;
}

uint32_t stage_bytes(TileCfg c) {
    const uint32_t seg = c.r * c.nc;
    const uint32_t xb = (seg + 2) * 3 * kChp * 8;
    const uint32_t off = (xb + 127) / 128 * 128;
    return (off + seg * Tile2dArgs::kAux * 8 + 127) / 128 * 128;
}

}  // namespace

int tile2d_seg() { return tile_cfg().nc * tile_cfg().r; }

int64_t tile2d_groups(const Tile2dArgs &a) {
    const int64_t seg = tile2d_seg();
    const int64_t n_seg = (a.row_w + seg - 1) / seg;
    const int64_t n_jr = (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
    return n_seg * n_jr;
}

int tile2d_chunk() { return kCh; }

cudaError_t tile2d_shape(int device, LaunchShape *out) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return e;
    const TileCfg c = tile_cfg();
    TileFn fn = tile_fn(c);
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = (size_t)c.stages * stage_bytes(c);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (c.nc + 1) * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    out->grid = sms * per_sm;
    out->smem = smem;
    return cudaSuccess;
}

cudaError_t launch_tile2d(const CUtensorMap &tmx, const Tile2dArgs &a, const LaunchShape &sh,
                          cudaStream_t st) {
    const TileCfg c = tile_cfg();
    TileFn fn = tile_fn(c);
    if (!fn) return cudaErrorInvalidValue;
    fn<<<sh.grid, (c.nc + 1) * 32, sh.smem, st>>>(tmx, a);
    return cudaGetLastError();
}

// box of the x tensor map: {time steps incl. halo, tensor rows}
void tile2d_box(uint32_t *box) {
    box[0] = kChp;
    box[1] = (uint32_t)((tile2d_seg() + 2) * 3);
}

}  // namespace biot
