/*
 * biot_pit.h -- C-ABI of the B200-native parallel-in-time Biot solver
 * (arXiv 2310.10430, "A Parallel-in-time Method Based on Preconditioner for
 * Biot's Model").  Library: paper_2310_10430_b200/libbiot_pit.so (sm_100a).
 *
 * What one outer iteration computes (the hot path), for every local time
 * step n at once (Jacobi in time, BASELINE.json north star; PAPER.md L290-302
 * Algorithm 2 with the damped preconditioned update, R1-R4):
 *
 *     r_n       = A' x_{n-1}^k + s_n f - AA x_n^k
 *     x_n^{k+1} = x_n^k + omega * P^{-1} r_n               (L298; R3 damping)
 *     rho_n     = ( ||r_{n,u}||_2 , ||r_{n,p}||_2 )          (R12)
 *
 * with the stabilised P1-P1 backward-Euler operators (PAPER.md L146-231,
 * eqs. fullysystem/axb; storage S per R8, per-cell kappa per R9):
 *     AA = [[A, B], [B^T, -(S M + dt C_kappa + beta L)]]
 *     A' = [[0, 0], [B^T, -(S M + beta L)]],  f = [F; 0]
 * and the paper's block preconditioners built on the approximate Schur
 * complement S~p = S M + dt C_kappa + beta L (eqs. p1/p2),
 * whose inner inverses A^{-1}, S~p^{-1} are realised by their diagonals (R2):
 *     P~1 = [[A, 0], [B^T, -S~p]]   (block lower triangular)
 *     P~2 = [[A, 0], [0,  -S~p]]    (block diagonal)
 *
 * Conventions
 *  - Vectors exchanged through this ABI are node-interleaved fp64:
 *    x[node*(d+1) + c], c = 0..d-1 displacement, c = d pressure (R20).
 *  - Time steps are global and 1-based: n = 1..n_t; x_0 is the fixed state at
 *    t = 0.  With world > 1, rank r owns steps n in (r*n_t/world, (r+1)*n_t/world].
 *  - All host inputs are copied during biot_setup; the caller may free them on
 *    return.  Output buffers are caller-allocated host memory.
 *  - Every call returns a biot_status; nothing aborts or throws across the
 *    ABI.  On error, biot_last_error(ctx) (or biot_last_error(NULL) for
 *    errors before a context exists) holds a message.
 *  - A context is not thread-safe.  With world > 1 (NCCL), these calls are
 *    collective -- every rank makes them in the same order, or the call blocks
 *    until BIOT_NCCL_TIMEOUT_S (default 600 s) and returns BIOT_E_NCCL:
 *    biot_setup, biot_iterate, biot_iterate_gs, biot_iterate_gmres,
 *    biot_iterate_cheb, biot_iterate_gs_gmres, biot_residual_norms (it refreshes
 *    the ghost slice before its residual pass) and biot_destroy.  A failed or
 *    silent peer surfaces as BIOT_E_NCCL (ncclCommGetAsyncError is polled while
 *    waiting; the communicator is then aborted and the context unusable for
 *    further collective calls).
 *  - biot_iterate is additive: iterate(a); iterate(b) == iterate(a+b), bitwise.
 *  - Results are bitwise reproducible run to run, and the iterates x^k are
 *    bitwise independent of world (time-slab count).
 */
#ifndef BIOT_PIT_H
#define BIOT_PIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BIOT_PIT_ABI_VERSION 4

typedef struct biot_ctx biot_ctx;   /* opaque; owned by the library until biot_destroy */

typedef enum {
    BIOT_OK = 0,
    BIOT_E_INVALID = 1,     /* bad argument; no state changed                      */
    BIOT_E_NOMEM = 2,       /* host or device allocation failed                    */
    BIOT_E_CUDA = 3,        /* CUDA runtime error (no device, launch failure, ...) */
    BIOT_E_NCCL = 4,        /* NCCL missing or failed                              */
    BIOT_E_STATE = 5,       /* call not valid in the current state                 */
    BIOT_E_NONFINITE = 6    /* a residual norm became NaN/Inf                      */
} biot_status;

/* Simplicial mesh (3D per BASELINE.json configs 4-5). */
typedef struct {
    int32_t dim;             /* 2 (triangles) or 3 (tetrahedra)                          */
    int64_t n_nodes;
    const double *coords;    /* host, n_nodes*dim                                        */
    int64_t n_cells;
    const int32_t *cells;    /* host, n_cells*(dim+1), positively oriented; a degenerate
                                or inverted cell -> BIOT_E_INVALID                        */
} biot_mesh;

/* Material (R5, R8, R9). */
typedef struct {
    double lambda, mu;       /* Lame coefficients, mu > 0, lambda >= 0                   */
    double alpha;            /* Biot-Willis constant                                     */
    double storage;          /* S >= 0 (storage coefficient, R8)                         */
    const double *kappa;     /* host, per-cell permeability (n_cells), or NULL           */
    double kappa_uniform;    /* used when kappa == NULL; must be > 0                     */
    double beta;             /* stabilisation factor; < 0 => h / (4 (lambda + 2 mu))     */
    double h;                /* mesh size entering beta (R6), > 0 if beta < 0    */
} biot_material;

/* Boundary data of the column problem (R11, R16). */
typedef struct {
    const uint8_t *dirichlet;        /* host, n_nodes*(dim+1), 1 = homogeneous Dirichlet DoF */
    int64_t n_traction_facets;
    const int32_t *traction_facets;  /* host, n_facets*dim node ids of boundary facets      */
    double traction[3];              /* constant traction on those facets (first dim used)  */
    const double *load_scale;        /* host, n_t values s_n (n = 1..n_t), or NULL => 1      */
    const double *x_initial;         /* host, x_0 (n_nodes*(dim+1)), or NULL => 0            */
    /* Time-dependent body force / source and non-homogeneous Dirichlet data (PAPER.md
     * §4.1: the trigonometric test; reading R24).  The load of step n becomes
     *   f_n = s_n [F_traction; 0]
     *       + sum_q source_coef[q*n_t + n-1] [ int f_q . phi ; -dt int g_q phi ]
     *       + dirichlet_coef[n]   (-AA_{free,D} x_D)      (lifting of x_D(t_n) = c_n x_D)
     *       + dirichlet_coef[n-1] ( A'_{free,D} x_D)      (x_D(t_{n-1}) through A')
     * (free rows only).  The integrals use a fixed quadrature per cell (triangles: the
     * 7-point degree-5 rule; tetrahedra: the 4-point degree-2 rule) at points the
     * library passes to source_eval.  The iterate keeps the homogeneous form: Dirichlet
     * DoFs of x stay 0 and the caller adds dirichlet_coef[n] x_D to recover the field.
     * At most 4 of these load terms (counting the traction term) may be nonzero. */
    int32_t n_sources;               /* source fields (>= 0)                                 */
    /* Called during biot_setup only: fill vals[k*(dim+1) + c] with component c of source
     * field q (f_1..f_d, g) at point xyz[k*dim ..], k < npts.  Must not call the library. */
    void (*source_eval)(int32_t q, int64_t npts, const double *xyz, double *vals, void *user);
    void *source_user;               /* passed through to source_eval                        */
    const double *source_coef;       /* host, [n_sources][n_t], finite                       */
    const double *dirichlet_values;  /* host, n_nodes*(dim+1) x_D (read on Dirichlet DoFs),
                                        or NULL => homogeneous                              */
    const double *dirichlet_coef;    /* host, n_t+1 values c_0..c_{n_t}, or NULL => all 1    */
} biot_bc;

#define BIOT_FLAG_MANUAL_HALO 1u     /* world > 1 without NCCL: caller moves the halo with
                                        biot_last_slice / biot_set_ghost (tests, emulation) */
#define BIOT_FLAG_DEFER_STEP0 4u     /* with MANUAL_HALO, ranks > 0 run the overlapped-halo form
                                        of biot_iterate (sweep with a zero ghost, then the first
                                        local step completed from the ghost): tests / emulation  */
#define BIOT_FLAG_SWEEP_SLABS 8u     /* world > 1: partition the Gauss-Seidel SWEEPS across ranks
                                        (Alg. 4/5 pipeline) instead of time slabs:
                                        every rank holds all n_t steps; biot_iterate_gs(K) runs
                                        global sweeps rank*K/world+1 .. (rank+1)*K/world and streams
                                        each finished step's slice to rank+1 (one per wave);
                                        x^K is broadcast from rank world-1 at the end.  With
                                        MANUAL_HALO: drive biot_gs_begin/wave/end; before wave W,
                                        rank r > 0 whose step W - (r*K/world) is in range takes
                                        rank r-1's biot_last_slice through biot_set_ghost; the
                                        result stays on rank world-1.  biot_iterate: BIOT_E_STATE */
#define BIOT_FLAG_NO_GRAPH    2u     /* biot_iterate launches kernels directly; default: pairs
                                        of iterations replay one captured CUDA graph (world == 1
                                        or MANUAL_HALO; NCCL iterations always launch directly) */

typedef struct {
    int32_t precond;         /* 1 = P~1, 2 = P~2                                          */
    double omega;            /* damping, > 0 (R3; default 0.5)                            */
    int32_t device;          /* CUDA device ordinal                                       */
    int32_t rank, world;     /* time-slab partition, 0 <= rank < world; n_t % world == 0  */
    const void *nccl_id;     /* world > 1 (no MANUAL_HALO): 128-byte ncclUniqueId made by
                                biot_nccl_unique_id on rank 0 and broadcast by the caller */
    void *stream;            /* cudaStream_t to run on, or NULL => library-owned stream   */
    uint32_t flags;          /* BIOT_FLAG_*                                               */
    int32_t history;         /* iterations of residual history retained (>= 0; 0 => 1024) */
} biot_opts;

/* Read-only facts about a context. */
typedef struct {
    int32_t dim, n_comp;             /* d, d+1                                          */
    int64_t n_nodes, n_dof;          /* N, N*(d+1)                                      */
    int32_t n_t, n_t_local, first_step; /* global N_t; owned steps first_step..+n_t_local-1 */
    int64_t iterations;              /* outer iterations done since setup               */
    int32_t kernel_path;             /* 1 = BDIA offsets, 2 = ELL explicit columns,
                                        4 = 2D row-march (L1-reuse) kernel,
                                        5 = 2D TMA-pipelined tile kernel,
                                        7 = 3D TMA-pipelined tile kernel             */
    int32_t n_slots;                 /* neighbour slots per node                        */
    double beta;                     /* the beta actually used                          */
    double bytes_per_iter;           /* algorithmic bytes per outer iteration (this rank) */
    double flops_per_iter;           /* algorithmic flops per outer iteration (this rank) */
    double device_bytes;             /* device memory held by the context               */
    int32_t launches_per_iter;       /* kernels biot_iterate launches per outer iteration */
    int32_t interior_nodes;          /* nodes on the shared interior stencil (tile kernels; 0 otherwise) */
    int32_t comm_nranks;             /* ranks of the context's NCCL communicator (0: none)         */
    int32_t graph;                   /* 1: biot_iterate replays a CUDA graph per pair of iterations */
} biot_info;

/* Build the operators on the host, upload, allocate the space-time panels
 * (x^0 = 0 for all owned steps).  Collective for world > 1. */
biot_status biot_setup(const biot_mesh *mesh, const biot_material *mat, const biot_bc *bc,
                       double dt, int32_t n_t, const biot_opts *opts, biot_ctx **out);

/* Set x_n^0 for `count` consecutive owned steps starting at global step n
 * (host, [count][n_dof] node-interleaved).  Dirichlet entries are forced to 0. */
biot_status biot_set_iterate(biot_ctx *ctx, int32_t n, int32_t count, const double *x);

/* Replace the load scales s_n (host, n_t values, global steps 1..n_t). */
biot_status biot_set_load_scale(biot_ctx *ctx, const double *s);

/* K outer iterations (K >= 0; K = 0 is a no-op).  Collective for world > 1. */
biot_status biot_iterate(biot_ctx *ctx, int32_t K);

/* K Gauss-Seidel-in-time sweeps (Algorithm 2 literally: the right-hand side
 * of step n uses the CURRENT sweep's X^{n-1}), run as a pipelined wavefront of
 * n_t_local + K - 1 windows.  Same preconditioner and omega as biot_iterate; the
 * residual history records, for sweep k and step n, the residual that update used.
 * Needs a structured 2D / 3D mesh (tile kernels), else BIOT_E_STATE.  Collective for
 * world > 1: after each wave in which rank r-1 updated its last step it sends that
 * slice to rank r (NCCL), K transfers per rank pair. */
biot_status biot_iterate_gs(biot_ctx *ctx, int32_t K);

/* K outer iterations of PAPER.md Algorithm 3 with the per-step solver K = GMRES(k)
 * (the paper's experiments' solver): every step at once runs one GMRES(k) cycle on
 * AA x_n = A' x_{n-1} + f_n (Jacobi in time) from its current iterate, left-
 * preconditioned by the context's P~ with diagonal inner inverses (P~2, eq. p2, or P~1,
 * eq. p1, the paper's choice for §4.1/§4.3; reading R23).  1 <= k <= 16; needs a
 * structured 2D / 3D mesh (tile kernels; BIOT_E_STATE otherwise); allocates k+1 Krylov
 * panels on first use.  The residual history records, per iteration and step, ||b - AA x|| (u, p) at
 * the cycle's start.  Collective for world > 1 (one slice per outer iteration). */
biot_status biot_iterate_gmres(biot_ctx *ctx, int32_t K, int32_t k);

/* K outer iterations as biot_iterate with the context's P~ (P~2, eq. p2, or P~1, eq. p1;
 * P:L238-262) whose inner inverses A^{-1} and S~p^{-1} are m steps of Chebyshev
 * iteration preconditioned by the diagonal, on [lambda_max / alpha, lambda_max] of
 * D^{-1} M with lambda_max the Gershgorin bound of each block (reading R22; m = 1 is the
 * diagonal inverse divided by theta).  P~1 runs the displacement block first, then the
 * pressure block on B^T z_u - r_p.  1 <= m <= 64, alpha > 1 (30 in R22); any mesh;
 * allocates up to 4 extra space-time panels on first use.  The residual history records
 * r(x^k) as biot_iterate does.  Collective for world > 1. */
biot_status biot_iterate_cheb(biot_ctx *ctx, int32_t K, int32_t m, double alpha);

/* PAPER.md Algorithm 3 literally: Gauss-Seidel in time (b^{n,m} = A' X^{n-1,m} + f^n)
 * with one GMRES(k) cycle per step and sweep (left P~1 or P~2), run as the wavefront of
 * biot_iterate_gs.  Same conditions as biot_iterate_gmres; collective for world > 1.
 * biot_gs_begin_gmres: its wave-level form (k = 0: the Richardson update). */
biot_status biot_iterate_gs_gmres(biot_ctx *ctx, int32_t K, int32_t k);
biot_status biot_gs_begin_gmres(biot_ctx *ctx, int32_t K, int32_t k);

/* The same run one wave at a time (BIOT_FLAG_MANUAL_HALO: before wave w the caller
 * moves the predecessor rank's biot_last_slice into biot_set_ghost of every rank
 * whose first owned step n satisfies w - K + 2 <= n <= w + 1).
 * biot_gs_waves: number of waves (n_t + K - 1) of the open run. */
biot_status biot_gs_begin(biot_ctx *ctx, int32_t K);
biot_status biot_gs_waves(const biot_ctx *ctx, int32_t *out);
biot_status biot_gs_wave(biot_ctx *ctx);
biot_status biot_gs_end(biot_ctx *ctx);

/* Residual norms at the current iterate: out[n_t_local][2] = ||r_u||, ||r_p||
 * of the owned steps (a residual-only pass, no update).  Collective for world > 1:
 * the pass needs the predecessor rank's current last slice (one halo exchange). */
biot_status biot_residual_norms(biot_ctx *ctx, double *out);

/* Norms of r(x^k) computed inside iteration k (k = 0-based count since setup):
 * out[n_t_local][2].  BIOT_E_STATE if k was not run or is no longer retained. */
biot_status biot_residual_history(biot_ctx *ctx, int64_t k, double *out);

/* Current iterate of `count` consecutive owned steps from global step n
 * (n = 0 returns x_0 on rank 0): out[count][n_dof] node-interleaved. */
biot_status biot_solution(biot_ctx *ctx, int32_t n, int32_t count, double *out);

/* Manual halo (BIOT_FLAG_MANUAL_HALO): copy the current iterate of the last
 * owned step out (host, n_dof) -- for world > 1 after an iteration, the send
 * buffer the sweep wrote, i.e. exactly what the NCCL exchange would send -- and
 * set the ghost (step first_step-1) in. */
biot_status biot_last_slice(biot_ctx *ctx, double *out);
biot_status biot_set_ghost(biot_ctx *ctx, const double *x);

/* Host-only: the assembled per-step operators in node-interleaved global
 * numbering, for inspection and tests (no device needed).  COO triplets of AA
 * and A' restricted to free DoFs (explicit zeros dropped), the load f, and the
 * inverse preconditioner diagonals (0 on Dirichlet DoFs).  Pass NULL arrays
 * to query the counts first. */
biot_status biot_assemble_host(const biot_mesh *mesh, const biot_material *mat,
                               const biot_bc *bc, double dt,
                               int64_t *nnz_AA, int64_t *AA_i, int64_t *AA_j, double *AA_v,
                               int64_t *nnz_AP, int64_t *AP_i, int64_t *AP_j, double *AP_v,
                               double *f, double *dinv);

/* Host-only: the further load terms of R24 (§4.1 sources, Dirichlet lifting) as the
 * library assembles them, node-interleaved on free DoFs (no device needed).  *n_terms
 * receives their number (<= 8); F (may be NULL to query) receives [n_terms][n_dof] and
 * kinds[j] (may be NULL) the kind of term j: 0 = source field (index src[j]), 1 = lifting
 * -AA_fD x_D (coefficient c_n), 2 = lifting A'_fD x_D (coefficient c_{n-1}).  All-zero
 * terms are omitted; the traction load is biot_assemble_host's f. */
biot_status biot_assemble_loads_host(const biot_mesh *mesh, const biot_material *mat,
                                     const biot_bc *bc, double dt, int32_t *n_terms, double *F,
                                     int32_t *kinds, int32_t *src);

biot_status biot_get_info(const biot_ctx *ctx, biot_info *out);

/* Device time of the kernels of the last biot_iterate call, per iteration,
 * measured with CUDA events on the compute stream: out[0] = whole iteration,
 * out[1] = the preconditioner pass(es) alone (ms): the fused sweep kernel (P~2,
 * single-pass P~1) or both passes of the two-pass P~1; with the CUDA graph the
 * mean over the two iterations of the last replay plus any direct launches. */
biot_status biot_last_timing(const biot_ctx *ctx, double *out_ms);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 only; dlopens libnccl.so.2). */
biot_status biot_nccl_unique_id(void *out);

/* Host helpers for the paper's structured workloads (no device needed).
 *
 * biot_mesh_structured: the unit square (dim 2, n x n cells, each split by the
 * lower-left -> upper-right diagonal into (n00, n10, n11) and (n00, n11, n01)) or the unit
 * cube (dim 3, n^3 cells, 6 Kuhn tetrahedra {v, v+e_a, v+e_a+e_b, v+e_a+e_b+e_c} per cell,
 * positively oriented); node id = j(n+1)+i (2D), (k(n+1)+j)(n+1)+i (3D) at (i,j[,k])/n
 * ("uniform mesh, h = 1/2^k").  *coords (nn*dim) and
 * *cells (nc*(dim+1)) are allocated by the library; release them with biot_free.
 *
 * biot_bc_column: the Terzaghi-type column of the BASELINE configs on such a mesh
 * (PAPER.md L70-84): dirichlet[n_nodes*(dim+1)] = 1 for u_x on x in {0,1}, (3D: u_y on
 * y in {0,1}), u on the bottom, p on the top; F[n_nodes*(dim+1)] = the load of the
 * traction (0,..,-load) on the top face (exact P1 facet integral, |f|/dim per vertex;
 * pressure entries 0); facets (may be NULL) receives the top facets, dim node ids each,
 * *n_facets their number (query with facets = NULL).  Coordinates within 1e-12 of a face
 * count as on it. */
biot_status biot_mesh_structured(int32_t dim, int32_t n, double **coords, int32_t **cells, int64_t *n_nodes,
                                 int64_t *n_cells);
biot_status biot_bc_column(const biot_mesh *mesh, double load, uint8_t *dirichlet, double *F,
                           int64_t *n_facets, int32_t *facets);
void biot_free(void *p);

void biot_destroy(biot_ctx *ctx);
const char *biot_last_error(const biot_ctx *ctx);
const char *biot_status_string(biot_status s);
int32_t biot_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BIOT_PIT_H */
