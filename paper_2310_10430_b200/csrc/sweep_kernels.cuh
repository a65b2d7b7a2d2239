// Hot-path kernels of the B200 Biot solver (sm_100a, fp64, no tensor cores).
// Internal header shared by sweep_kernels.cu and biot_api.cu.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace biot {

constexpr int kThreads = 256;   // 8 warps per CTA
constexpr int kT = 4;           // consecutive time steps per lane (2 x 16-B loads)
constexpr int kChunk = 32 * kT; // time steps per warp chunk
constexpr int kMaxLoads = 4;    // load terms of the multi-load kernels (R24)

enum SweepMode : int {
    MODE_UPDATE_P2 = 0,   // fused residual + P~2 + update + norms
    MODE_P1_PASS1 = 1,    // residual, x_u update, Z = (z_u, r_p), norms
    MODE_RESIDUAL = 2,    // residual norms only (no writes)
    MODE_PASS2 = 3,       // P~1 second pass (tile kernels): x_p += omega DSinv (B^T z_u - r_p)
    MODE_ZOUT = 4,        // GMRES start (2D tile): zbuf = P~2^{-1} r, norms of r, x untouched
    MODE_MATVEC = 5,      // GMRES Arnoldi (2D tile): xn = P~2^{-1} AA x, no time coupling
    MODE_P1_FUSED = 6,    // P~1 in one pass (2D tile): residual, z_u, z_p = D_S^{-1}(B^T z_u - r_p) from
                          // the neighbours' z_u (recomputed on the tile's halo), update, norms
};

struct SweepArgs {
    const double *x;        // panel of x^k at node 0: x[(i*nc + c)*pitch + t]; padded nodes around
    double *xn;             // panel of x^{k+1} (same layout)
    const double *ghost;    // x_{first-1}^k, [i*nc + c] at node 0 (padded)
    const double *blk;      // operator blocks [i][slot][W]
    const int32_t *cols;    // ELL columns [i][slot] (null for BDIA)
    const double *load;     // f [i*nc + c]
    const double *dinv;     // inverse preconditioner diagonals [i*nc + c]
    const double *s;        // load coefficients of the local steps: term j at s[j * s_pitch + t]
    const double *loadx;    // load vectors of terms j = 1..kMaxLoads-1: [(j-1) * n_nodes + i][nc]
    int64_t s_pitch;        // doubles between the coefficient rows of s
    int32_t n_load;         // load terms (1: s_t f; > 1: the kMaxLoads-term kernels, unused terms zero)
    double *zbuf;           // P~1: Z panel (z_u in u rows, r_p in p row)
    double *sendbuf;        // x^{k+1} of the last local step [i*nc + c] (null: not needed)
    double *partial;        // per-CTA norm partials [gridDim.x][n_tl][2]
    int64_t n_nodes;
    int64_t pitch;          // doubles per (node, component) row; multiple of kChunk
    int32_t n_tl;           // local time steps
    int32_t tw;             // chunk-warps per CTA (power of two dividing 8)
    int32_t node_block;     // consecutive nodes per CTA work block
    int32_t mode;
    double omega;
    int64_t off[32];        // BDIA column offsets (slot 0 = self)
    // 2D march kernel (structured right-triangle mesh): node = j * row_w + i
    int64_t row_w;          // nodes per grid row (n+1)
    int32_t n_rows;         // grid rows (n+1)
    int32_t rows_per_tile;  // rows marched by one tile
    int32_t ghost_zero;     // tile kernels: the ghost is identically zero (x_0 = 0 on rank 0, or the
                            // deferred sweep of the overlapped halo): q(t0-1) = A' 0 = +0 without loads
    int32_t p1_out;         // GMRES modes (ZOUT / MATVEC) with P~1: write the first half (z_u, r_p) of
                            // P~1^{-1} r; pass2 (pure) then completes z_p in place
    double *s0buf;          // deferred sweep (overlapped halo): per node, the pieces of the first local
                            // step's pressure update that do not depend on the ghost:
                            // [acc_p, f_p, x_p^k, (B^T z_u)_p, D_S^{-1}, path flag, -, -] (tile
                            // kernels), else null
};

struct Pass2Args {          // P~1 second pass: x_p += omega DSinv (B^T z_u - r_p)
    int32_t t_off, t_lo;    // time window (Gauss-Seidel waves): columns t_off.., stores from t_lo
    const double *x;
    double *xn;
    const double *zbuf;
    const double *blk;
    const int32_t *cols;
    const double *dinv;
    double *sendbuf;
    int64_t n_nodes, pitch;
    int32_t n_tl, tw, node_block;
    double omega;
    int64_t off[32];
    int32_t pure;           // 1: xn_p = D_S^{-1} (B^T z_u - r_p) itself (GMRES with P~1, in place on
                            // a Krylov panel: zbuf = xn), not x_p + omega times it
};


// Arguments of the TMA-pipelined 2D tile kernel (tile2d_kernels.cu).
constexpr int kAuxRecU = 16;
struct Tile2dArgs : SweepArgs {
    static constexpr int kAux = 16;   // per-node record: AA_pp per slot [7], f [3], dinv [3], path flag
    static constexpr int kAuxML = 24; // kMaxLoads kernels: + the further load vectors F_j at [14 + 3 (j-1) + c]
    double tmpl[7][10];               // interior stencil blocks (slot order), pp entry unused
    const double *aux;                // [n_alloc][kAux]
    const double *cls;                // geometric-class stencils [9][7][kClsW], column-major blocks
    static constexpr int kClsW = 10;  // 9 AA entries + A'_pp
    int64_t pad_nodes;                // panel rows start at node -pad_nodes
    int64_t ghost_stride;             // doubles between ghost entries (1: a vector; pitch: a panel column)
    int32_t t_off;                    // first panel column of the time window (Gauss-Seidel waves; even)
    int32_t t_lo;                     // window steps below t_lo are computed but not stored or counted
    int32_t s0;                       // zero-storage variant: extra structural zeros (see tile2d)
    int32_t dry;                      // dev/measurement only: stream the ring without computing
    // aux-uniform rectangle (single-load problems with uniform coefficients, e.g. config 3):
    // every node with ux0 <= column <= ux1 and uy0 <= row <= uy1 has the aux record aux_u
    // (pp entries against fixed pressure columns may differ: they multiply x = 0), so row
    // strips inside it skip the aux bulk copy and read aux_u (staged once in shared memory)
    int32_t aux_geo, ux0, ux1, uy0, uy1;
    // P~2-family tile kernels: the grid rows split into n_rblk blocks of floor/ceil(n_rows /
    // n_rblk) rows (block r: rows [r n_rows / n_rblk, (r+1) n_rows / n_rblk)); rows_per_tile
    // is then the largest block. 0: uniform blocks of rows_per_tile rows (the fused P~1)
    int32_t n_rblk;
    double aux_u[kAuxRecU];
};

// Arguments of the TMA-pipelined 3D tile kernel (tile3d_kernels.cu): structured
// n1^3 Kuhn cube, node = (z*n1 + y)*n1 + x, BDIA slot order of host_assembly.
struct Tile3dArgs : SweepArgs {
    static constexpr int kAux = 24;   // per-node record: AA_pp per slot [15], f [4], dinv [4], path flag
    double tmpl[15][17];              // interior stencil: AA block [16] (pp entry unused) + A'_pp
    const double *aux;                // [n_alloc][kAux]
    const double *cls;                // geometric-class stencils [27][15][kClsW], column-major blocks
    static constexpr int kClsW = 18;  // 17 entries padded to 16 B
    int64_t ghost_stride;             // doubles between ghost entries (1: a vector; pitch: a panel column)
    int32_t t_off;                    // first panel column of the time window (Gauss-Seidel waves)
    int32_t t_lo;                     // window steps below t_lo are computed but not stored or counted
    int32_t n1;                      // nodes per axis
    int32_t z_rows;                   // planes marched per tile
    int32_t s0;                       // zero-storage structural-zero variant
    int32_t dry;                      // dev/measurement only: stream the ring without computing
};

struct LaunchShape {
    int grid;
    size_t smem;
};

// dim in {2,3}; path 1 = BDIA, 2 = ELL; n_slots must match the instantiations.
cudaError_t sweep_shape(int dim, int path, int n_slots, bool ml, int device, LaunchShape *out);
cudaError_t launch_sweep(int dim, int path, int n_slots, const SweepArgs &a, const LaunchShape &sh,
                         cudaStream_t st);
cudaError_t launch_pass2(int dim, int path, int n_slots, const Pass2Args &a, int grid,
                         cudaStream_t st);
// norms[t][k] = sqrt(sum_g partial[g][t][k]) in fixed g order; flags non-finite values
// 2D march kernel: CTA = 8-node row segment x (32*T)-step chunk, marching rows.
cudaError_t march_shape(int T, int device, LaunchShape *out);
cudaError_t launch_march(int T, const SweepArgs &a, const LaunchShape &sh, cudaStream_t st);
// norm-partial groups of the march kernel (segments x row ranges)
inline int64_t march_groups(const SweepArgs &a) {
    const int64_t n_seg = (a.row_w + 7) / 8;
    const int64_t n_jr = (a.n_rows + a.rows_per_tile - 1) / a.rows_per_tile;
    return n_seg * n_jr;
}

// 2D TMA tile kernel: x boxes {time, rows} of the panel tensor map
int64_t tile2d_tiles(const Tile2dArgs &a);
int64_t tile2d_groups(const Tile2dArgs &a, int grid);   // norm-partial groups: CTAs x columns
int tile2d_chunk();
int tile2d_seg();         // grid columns per tile
int tile2d_max_rows();    // rows per tile (q carry capacity)
int tile2d_seg_p1();      // own grid columns per tile of the fused P~1 mode
void tile2d_box(uint32_t *box);
cudaError_t tile2d_shape(int device, LaunchShape *out);
cudaError_t launch_tile2d(const CUtensorMap &tmx, const Tile2dArgs &a, const LaunchShape &sh,
                          cudaStream_t st);
// Deferred first local step (overlapped halo): complete step t_off of every node from the
// ghost and the pieces the sweep saved in a.s0buf (bitwise the undeferred update),
// overwrite x_p^{k+1} there; the step's pressure-norm partials per block -> part[blocks].
// Modes MODE_UPDATE_P2 and MODE_P1_FUSED.
int tile2d_step0_blocks(int64_t n_nodes);
cudaError_t launch_tile2d_step0(const Tile2dArgs &a, double *part, cudaStream_t st);

// 3D TMA tile kernel: 4x2 (x,y) node patches x 64-step chunks, marching z
int64_t tile3d_groups(const Tile3dArgs &a);
int64_t tile3d_patches(int64_t n1);   // (x, y) patches of an n1^3 mesh
int tile3d_chunk();
int tile3d_max_zrows();
int tile3d_min_n1();
void tile3d_box(uint32_t *box);      // {time, x*4+c, y, z}
void tile3d_box_z(uint32_t *box);    // {time, c, x, y, z}: the P~1 second pass's Z-panel box
cudaError_t tile3d_shape(int device, LaunchShape *out);
cudaError_t launch_tile3d(const CUtensorMap &tmx, const Tile3dArgs &a, const LaunchShape &sh,
                          cudaStream_t st);
// deferred first local step (see launch_tile2d_step0): MODE_UPDATE_P2 or MODE_P1_PASS1
int tile3d_step0_blocks(int64_t n_nodes);
cudaError_t launch_tile3d_step0(const Tile3dArgs &a, double *part, cudaStream_t st);


// Per-step GMRES panel kernels (gmres_kernels.cu): column-wise (per time step) dot
// products of a panel with nb panels (b_dev: device array of panel pointers) and
// dst = scale_t * (base + sign * sum_i coef[i][t] b_i); rows = real panel rows.
int gmres_max_vectors();
int64_t gmres_dots_scratch(int64_t rows, int n_tl, int nb, int64_t *chunk, int *chunks);
// (boff: column offset applied to the b panels -- a time window of them)
cudaError_t gmres_dots(const double *a, const double *const *b_dev, int boff, int nb, int64_t rows, int64_t pitch,
                       int n_tl, double *scratch, double *out, double *hacc, bool norm, cudaStream_t st);
// row pitches (doubles) of dst, base, the b panels and dst2: the full panel pitch, or the
// window width for a compact basis (narrow Gauss-Seidel windows)
struct GmresPitch {
    int64_t dst, base, v, dst2;
};
cudaError_t gmres_combine(double *dst, const double *base, const double *const *b_dev, int boff, const double *coef,
                          int nb, double sign, const double *scale, int64_t rows, GmresPitch pitch, int n_tl,
                          cudaStream_t st, double *dst2 = nullptr);
// per step t: y = argmin || beta_t e1 - H_t y ||, H_t (k+1) x k upper Hessenberg at
// H[(i + j (k+1)) n_tl + t] (Givens rotations on the device, one thread per step)
cudaError_t gmres_lsq(const double *H, const double *beta, int k, int n_tl, double *y, cudaStream_t st);

// Chebyshev inner inverses of P~2 (cheb_kernels.cu): panels at node 0
// with the context's padding and pitch.
struct ChebArgs {
    const double *blk;      // operator blocks [i][slot][W]
    const int32_t *cols;    // ELL columns (null for BDIA)
    int64_t off[32];        // BDIA offsets
    const double *dinv;     // D_A^{-1} / D_S^{-1} per (node, comp)
    int64_t n_nodes, pitch;
    int32_t nc, n_tl;
    double *s;              // scaled residual s = D^{-1} r (in place)
    const double *d;        // d_{k-1}
    double *dn;             // d_k
    const double *y;        // y_{k-1} (null: y_1 = d_0)
    double *yn;             // y_k
    const double *x;        // x^k (last pass)
    double *xn;             // x^{k+1} (last pass)
    double *sendbuf;        // last step of x^{k+1} (multi-slab), or null
    double c1_u, c2_u, c1_p, c2_p;          // rho_k rho_{k-1}, 2 rho_k / delta per block
    double inv_theta_u, inv_theta_p;        // 1 / theta per block (the start)
    double omega;
    int32_t last;           // 1: write x^{k+1} instead of s, d, y
    int32_t rows;           // rows updated: 1 displacement, 2 pressure, 3 both (P~1 runs the blocks in turn)
    double p_sign;          // z_p = p_sign y_p: -1 for P~2 (S~p y = r_p, z_p = -y), +1 for P~1
    const double *zu;       // P~1 pressure start: the panel holding z_u
    int32_t first;          // 1: d_0 = D^{-1} r / theta computed on the fly from the Z panel in s
                            //    (no start pass); the new s goes to sn
    double *sn;
};
cudaError_t launch_cheb_init(const ChebArgs &a, cudaStream_t st);
cudaError_t launch_cheb_step(int dim, int path, int n_slots, const ChebArgs &a, cudaStream_t st);
// P~1: r~_p = B^T z_u - r_p, s_p = D_S^{-1} r~_p, d_p = s_p / theta_p (or, m = 1, the
// update), and x_u^{k+1} = x_u + omega z_u
cudaError_t launch_cheb_p1_rhs(int dim, int path, int n_slots, const ChebArgs &a, cudaStream_t st);

// scratch: finalize_scratch_doubles(groups, n_tl) doubles (two-stage reduction when
// there are many groups; both stages in a fixed order, so the result is deterministic)
int64_t finalize_scratch_doubles(int groups, int n_tl);
// slot_ctr != null: norms is the history ring [cap][n_tl][2], written at slot
// (*slot_ctr + slot_off) % cap read on the device (so a captured CUDA graph can be replayed)
// tickets (finalize_tickets(n_tl) zeroed ints): one launch instead of two (the last block
// of each column tile completes it); part0/nb0: the deferred first step's p-norm partials
cudaError_t launch_finalize(const double *partial, int groups, int n_tl, double *norms,
                            int *nonfinite, double *scratch, cudaStream_t st, const int64_t *slot_ctr = nullptr,
                            int64_t slot_off = 0, int cap = 1, int *tickets = nullptr, const double *part0 = nullptr,
                            int nb0 = 0);
int finalize_tickets(int n_tl);
// *ctr = value (add = false) or *ctr += value, on the stream
cudaError_t launch_counter(int64_t *ctr, int64_t value, bool add, cudaStream_t st);
// Gauss-Seidel wave: the window's steps t = lo..lo+len-1 carry iteration k = k0 - t;
// norms of t >= t_first go to hist[(k % cap) * n_tl + t] (the residual-history ring)
cudaError_t launch_finalize_wave(const double *partial, int groups, int len, int lo, int t_first, int64_t k0,
                                 int cap, int n_tl, double *hist, int *nonfinite, double *scratch, cudaStream_t st);

}  // namespace biot
