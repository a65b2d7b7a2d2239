// C-ABI of the B200 Biot solver (declared in include/biot_pit.h).
//
// One context per rank.  setup: host assembly (host_assembly.cpp) -> upload ->
// two ping-pong space-time panels.  iterate(K): per outer iteration, optional
// NCCL halo (ncclSend of the last local slice to rank+1, ncclRecv of the ghost
// from rank-1; BASELINE.json north star (d), replacing the paper's MPI
// Send/Recv pipeline of Algorithm 5), then the fused sweep
// kernel (+ the P~1 second pass), then the deterministic norm finalize.
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/biot_pit.h"
#include "host_assembly.h"
#include "sweep_kernels.cuh"

namespace {

thread_local std::string g_err;

// ---------------- NCCL, loaded at run time ----------------
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;   // optional
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;                           // optional
    ncclResult_t (*CommCount)(const ncclComm_t, int *) = nullptr;              // optional
    ncclResult_t (*Bcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

NcclApi *nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names) {
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (api.h) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(api.h, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(api.h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(api.h, "ncclCommDestroy");
            api.Send = (decltype(api.Send))dlsym(api.h, "ncclSend");
            api.Recv = (decltype(api.Recv))dlsym(api.h, "ncclRecv");
            api.GroupStart = (decltype(api.GroupStart))dlsym(api.h, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(api.h, "ncclGroupEnd");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(api.h, "ncclGetErrorString");
            api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(api.h, "ncclCommGetAsyncError");
            api.CommAbort = (decltype(api.CommAbort))dlsym(api.h, "ncclCommAbort");
            api.CommCount = (decltype(api.CommCount))dlsym(api.h, "ncclCommCount");
            api.Bcast = (decltype(api.Bcast))dlsym(api.h, "ncclBroadcast");
            if (!api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.GroupStart ||
                !api.GroupEnd || !api.CommDestroy)
                api.h = nullptr;
        }
    }
    return api.h ? &api : nullptr;
}

// panel gather/scatter between [count][N*nc] host-order staging and the panel
__global__ void scatter_steps_kernel(const double *__restrict__ src, double *__restrict__ panel,
                                     const uint8_t *__restrict__ fixed, int64_t nrows, int64_t pitch,
                                     int t_first, int count) {
    const int64_t total = nrows * count;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tt = k / nrows, row = k % nrows;
        panel[row * pitch + t_first + tt] = fixed[row] ? 0.0 : src[k];
    }
}

__global__ void gather_steps_kernel(const double *__restrict__ panel, double *__restrict__ dst,
                                    int64_t nrows, int64_t pitch, int t_first, int count) {
    const int64_t total = nrows * count;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tt = k / nrows, row = k % nrows;
        dst[k] = panel[row * pitch + t_first + tt];
    }
}

// Copy the odd (parity = 1) or even (parity = 0) time columns of the first n_tl steps
// of every panel row: the Gauss-Seidel wavefront keeps step t of sweep u in panel
// (u + t) % 2 (see biot_iterate_gs).
__global__ void copy_parity_columns_kernel(const double *__restrict__ src, double *__restrict__ dst,
                                           int64_t nrows, int64_t pitch, int n_tl, int parity) {
    const int64_t half = (n_tl - parity + 1) / 2;
    const int64_t total = nrows * half;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = k / half, t = 2 * (k % half) + parity;
        dst[row * pitch + t] = src[row * pitch + t];
    }
}

}  // namespace

struct biot_ctx {
    std::string err;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int d = 0, nc = 0;
    int64_t N = 0, pad = 0, rows_alloc = 0;
    int S = 0, path = 0;
    int32_t n_t = 0, n_tl = 0, first_step = 1, rank = 0, world = 1;
    int64_t pitch = 0;
    uint32_t flags = 0;
    int precond = 2;
    double omega = 0.5;
    double beta = 0.0;
    int64_t nnz_AA = 0, nnz_AP = 0;
    std::vector<int64_t> offsets;

    double *xbase[2] = {nullptr, nullptr};
    double *x[2] = {nullptr, nullptr};        // at node 0
    double *zbase = nullptr, *z = nullptr;
    double *ghost_base = nullptr, *ghost = nullptr;
    double *blk = nullptr;
    int32_t *cols = nullptr;
    double *load = nullptr, *dinv = nullptr, *s = nullptr;
    double *loadx = nullptr;          // load terms 1..n_load-1 (R24), [(j-1)*N + i][nc]
    int n_load = 1;                   // load terms (s rows); > 1 selects the kMaxLoads kernels
    int trac_term = 0;                // s row of the traction term (biot_set_load_scale), -1: none
    int64_t s_pitch = 0;              // doubles between the rows of s
    uint8_t *fixed = nullptr;
    double *sendbuf = nullptr;        // the current last slice (what the next exchange sends)
    double *send_w = nullptr;         // where the sweep writes the new slice (= sendbuf, or the
                                      // other buffer of the overlapped exchange)
    // overlapped time-slab halo (world > 1, tile kernels): the exchange of x^k's slice runs on
    // comm_stream while the sweep runs; ranks > 0 sweep with a zero ghost (ghost_override) and
    // complete their first local step after the ghost arrived (the step-0 kernels)
    bool overlap = false, defer0 = false;
    bool x0_zero = true;              // x_0 = 0 (rank 0's ghost is identically zero)
    // Gauss-Seidel sweeps partitioned across ranks (BIOT_FLAG_SWEEP_SLABS, Alg. 4/5):
    // every rank holds all steps; sweep_in receives the predecessor rank's finished slices
    bool sweep_mode = false;
    double *sweep_in = nullptr;
    double *sendbuf2 = nullptr, *zero_ghost_base = nullptr, *zero_ghost = nullptr, *s0buf = nullptr, *part0 = nullptr;
    const double *ghost_override = nullptr;
    int step0_blocks = 0;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_comm = nullptr;
    double *partial = nullptr;
    double *fin_scratch = nullptr;    // norm reduction scratch (chunk sums)
    int *fin_tickets = nullptr;       // one-launch finalize: per 32-step column tile
    double *hist = nullptr, *norms = nullptr;
    int *nonfinite = nullptr;
    double *staging = nullptr;
    int64_t staging_steps = 0;
    int cur = 0;
    bool send_dirty = true;
    int64_t iterations = 0;
    int hist_cap = 1024;
    biot::LaunchShape shape{0, 0};
    int tw = 8, node_block = 8;
    // kernel choice: 1 generic BDIA/ELL sweep, 3 2D march, 4 2D TMA tile, 6 3D TMA tile
    int kern = 1;
    bool stencil = false;             // detect_stencil() succeeded (structured offsets)
    int mT = 2;                       // march: time steps per lane
    int64_t row_w = 0;
    int32_t n_rows = 0, rows_per_tile = 0;
    int64_t groups = 0;               // norm-partial groups of the active kernel
    // fused single-pass P~1 (tile2d MODE_P1_FUSED): its own tile shape and partial groups
    bool p1_fused = false;
    int32_t rows_per_tile_p1 = 0;
    int32_t n_rblk = 0;               // tile2d (P~2 family): balanced row blocks (Tile2dArgs::n_rblk)
    int64_t groups_p1 = 0;
    double *aux_base = nullptr;       // aux records with front padding (tile2d halo columns)
    int32_t aux_geo = 0, ux0 = 0, ux1 = -1, uy0 = 0, uy1 = -1;   // tile2d aux-uniform rectangle
    double aux_u[biot::kAuxRecU] = {0};
    // 4: TMA-pipelined 2D tile kernel
    double *aux = nullptr;
    double tmpl[7][10] = {{0}};
    CUtensorMap tmap[2];
    CUtensorMap tmapz;                // P~1 Z panel (tile kernels' second pass)
    int64_t n_interior = 0;
    int s0 = 0;                       // tile2d/tile3d zero-storage structural-zero variant
    // 6: TMA-pipelined 3D tile kernel
    double tmpl3[15][17] = {{0}};
    double *cls = nullptr;            // tile3d class stencils (device)
    // per-step GMRES (biot_iterate_gmres): Krylov panels, their tensor maps, scratch
    std::vector<double *> gm_V, gm_Vbase;
    std::vector<CUtensorMap> gm_tmap;
    double **gm_Vdev = nullptr;
    double *gm_scratch = nullptr, *gm_small = nullptr;
    // compact Krylov basis of narrow windows (Gauss-Seidel waves): k+1 vectors of
    // rows x gm_vc_w doubles, rows adjacent (gmres_cycle)
    double *gm_Vc = nullptr;
    double **gm_Vcdev = nullptr;
    int gm_vc_w = 0, gm_vc_n = 0;
    // Chebyshev inner inverses (biot_iterate_cheb): Gershgorin bounds of D^{-1} A and
    // D_S^{-1} S~p, the scaled-residual panel, d ping-pong and y panels
    double lmax_u = 0.0, lmax_p = 0.0;
    double *cb_base[4] = {nullptr, nullptr, nullptr, nullptr};
    double *cb[4] = {nullptr, nullptr, nullptr, nullptr};   // s, d0, d1, y (at node 0)
    // Gauss-Seidel wavefront state (biot_gs_begin / biot_gs_wave / biot_gs_end)
    int32_t gs_K = 0, gs_w = 0, gs_k = 0;   // gs_k > 0: each window update is a GMRES(gs_k) cycle
    int64_t gs_k0 = 0;
    int32_t n1 = 0, z_rows = 0;
    int tile_dry = 0;                 // BIOT_TILE_DRY=1: memory-pipeline measurement only
    int64_t gbase[8] = {0};
    int32_t slot[8][3] = {{0}};
    int64_t n_alloc = 0;              // nodes allocated in operator arrays (>= N, multiple of 8)
    int pass2_grid = 0;
    size_t device_bytes = 0;
    ncclComm_t comm = nullptr;
    double nccl_timeout_s = 600.0;    // BIOT_NCCL_TIMEOUT_S: a peer silent this long -> BIOT_E_NCCL
    // CUDA graph of two outer iterations per starting panel (biot_iterate, world == 1 or
    // manual halo, unless BIOT_FLAG_NO_GRAPH): the history slot comes from d_iter
    bool use_graph = false;
    int64_t *d_iter = nullptr;        // device copy of `iterations`
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    cudaEvent_t gev[4] = {nullptr, nullptr, nullptr, nullptr};   // sweep spans inside the graph
    // the captured graphs (kept: their event-record nodes re-target per replay) and those
    // nodes in gev order; gev_pool: the spans of sampled replays of the current call
    cudaGraph_t gsrc[2] = {nullptr, nullptr};
    cudaGraphNode_t gnode[2][4] = {{nullptr, nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr, nullptr}};
    std::vector<cudaEvent_t> gev_pool;
    bool gpool_set[2] = {false, false};   // the exec's nodes currently target gev_pool events
    cudaStream_t cap_stream = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr;
    std::vector<cudaEvent_t> ev_s;                 // 2 per iteration of the current call
    double last_ms_iter = 0.0, last_ms_sweep = 0.0;
};

namespace {

biot_status fail(biot_ctx *c, biot_status s, const std::string &m) {
    if (c) c->err = m;
    g_err = m;
    return s;
}

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(ctx, BIOT_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

biot_status dev_alloc(biot_ctx *ctx, void **p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 8);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, BIOT_E_NOMEM, "cudaMalloc(" + std::to_string(bytes) + " B) failed: " +
                                          cudaGetErrorString(e));
    }
    ctx->device_bytes += bytes;
    return BIOT_OK;
}

#define ALLOC(ptr, bytes)                                                  \
    do {                                                                   \
        biot_status s_ = dev_alloc(ctx, (void **)&(ptr), (size_t)(bytes)); \
        if (s_ != BIOT_OK) return s_;                                      \
    } while (0)

void free_all(biot_ctx *c) {
    cudaSetDevice(c->device);
    for (void *p : {(void *)c->xbase[0], (void *)c->xbase[1], (void *)c->zbase, (void *)c->ghost_base,
                    (void *)c->blk, (void *)c->cols, (void *)c->load, (void *)c->loadx, (void *)c->dinv, (void *)c->s,
                    (void *)c->fixed, (void *)c->sendbuf, (void *)c->sendbuf2, (void *)c->zero_ghost_base, (void *)c->s0buf, (void *)c->sweep_in,
                    (void *)c->part0, (void *)c->partial, (void *)c->hist,
                    (void *)c->norms, (void *)c->nonfinite, (void *)c->staging, (void *)c->aux_base,
                    (void *)c->cls, (void *)c->fin_scratch, (void *)c->fin_tickets, (void *)c->gm_Vdev, (void *)c->gm_scratch,
                    (void *)c->gm_small, (void *)c->gm_Vc, (void *)c->gm_Vcdev, (void *)c->d_iter})
        if (p) cudaFree(p);
    for (double *p : c->gm_Vbase) cudaFree(p);
    for (double *p : c->cb_base)
        if (p) cudaFree(p);
    for (cudaEvent_t e : {c->ev_a, c->ev_b})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_s) cudaEventDestroy(e);
    for (cudaEvent_t e : c->gev)
        if (e) cudaEventDestroy(e);
    for (cudaGraph_t g : c->gsrc)
        if (g) cudaGraphDestroy(g);
    for (cudaEvent_t e : c->gev_pool)
        if (e) cudaEventDestroy(e);
    for (cudaGraphExec_t g : c->gexec)
        if (g) cudaGraphExecDestroy(g);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    for (cudaEvent_t e : {c->ev_ready, c->ev_comm})
        if (e) cudaEventDestroy(e);
    if (c->comm && nccl()) nccl()->CommDestroy(c->comm);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
}

// Every transfer of a context goes on its own stream: the stream may be
// non-blocking, so mixing it with legacy-default-stream copies would race (a
// zero-fill enqueued earlier could land after an upload).
cudaError_t h2d(biot_ctx *c, void *dst, const void *src, size_t bytes) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(c->stream);
}

biot::SweepArgs sweep_args(biot_ctx *c, int mode, const double *xin, double *xout) {
    biot::SweepArgs a{};
    a.x = xin;
    a.xn = xout;
    a.ghost = c->ghost_override ? c->ghost_override : c->ghost;
    a.blk = c->blk;
    a.cols = c->cols;
    a.load = c->load;
    a.dinv = c->dinv;
    a.s = c->s;
    a.loadx = c->loadx;
    a.s_pitch = c->s_pitch;
    a.n_load = c->n_load;
    a.zbuf = c->z;
    a.sendbuf = (c->world > 1 && mode != biot::MODE_RESIDUAL) ? c->send_w : nullptr;
    a.partial = c->partial;
    a.n_nodes = c->N;
    a.pitch = c->pitch;
    a.n_tl = c->n_tl;
    a.tw = c->tw;
    a.node_block = c->node_block;
    a.mode = mode;
    a.omega = c->omega;
    for (int s = 0; s < 32; ++s) a.off[s] = s < (int)c->offsets.size() ? c->offsets[s] : 0;
    a.row_w = c->row_w;
    a.n_rows = c->n_rows;
    a.rows_per_tile = c->rows_per_tile;
    a.ghost_zero = (c->ghost_override && c->ghost_override == c->zero_ghost) ||
                   ((c->rank == 0 || c->sweep_mode) && c->x0_zero) ? 1 : 0;
    a.p1_out = (c->precond == 1 && (mode == biot::MODE_ZOUT || mode == biot::MODE_MATVEC)) ? 1 : 0;
    // the deferred sweep saves the ghost-independent pieces of its first step's p-update
    a.s0buf = (c->ghost_override && c->ghost_override == c->zero_ghost) ? c->s0buf : nullptr;
    return a;
}

biot_status pack_send(biot_ctx *ctx) {
    // last local step of the current iterate -> contiguous send buffer
    CU(cudaMemcpy2DAsync(ctx->sendbuf, sizeof(double), ctx->x[ctx->cur] + (ctx->n_tl - 1),
                         ctx->pitch * sizeof(double), sizeof(double), (size_t)ctx->N * ctx->nc,
                         cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->send_dirty = false;
    return BIOT_OK;
}

biot_status halo_exchange(biot_ctx *ctx) {
    if (ctx->world == 1 || (ctx->flags & BIOT_FLAG_MANUAL_HALO) || ctx->sweep_mode) return BIOT_OK;
    NcclApi *api = nccl();
    if (!api || !ctx->comm) return fail(ctx, BIOT_E_NCCL, "NCCL not initialised");
    if (ctx->send_dirty) {
        biot_status s = pack_send(ctx);
        if (s != BIOT_OK) return s;
    }
    const size_t n = (size_t)ctx->N * ctx->nc;
    ncclResult_t r = api->GroupStart();
    if (r == ncclSuccess && ctx->rank + 1 < ctx->world)
        r = api->Send(ctx->sendbuf, n, ncclFloat64, ctx->rank + 1, ctx->comm, ctx->stream);
    if (r == ncclSuccess && ctx->rank > 0)
        r = api->Recv(ctx->ghost, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->stream);
    ncclResult_t r2 = api->GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(ctx, BIOT_E_NCCL, std::string("NCCL halo exchange failed: ") +
                                          (api->GetErrorString ? api->GetErrorString(r != ncclSuccess ? r : r2) : "?"));
    return BIOT_OK;
}

// Stencil entries of two nodes of one class agree to rounding: on a uniform mesh
// whose coordinates are not dyadic, the per-node element integrals differ in the
// last bits; the tile kernels apply the class value (reading R21).
inline bool same_entry(double v, double t) {
    if (v == t) return true;
    if (v == 0.0 || t == 0.0) return false;
    return std::fabs(v - t) <= 8.0 * std::numeric_limits<double>::epsilon() * std::max(std::fabs(v), std::fabs(t));
}

// Node i may take a tile kernel's interior path (one template stencil, structural
// zeros skipped) iff none of its DoFs is fixed and every entry k <= nc*nc of every
// slot block either is the per-node AA_pp entry (carried in the aux record), or is
// a structural zero the kernel skips (then it must be 0 here), or equals the
// template, or is 0 against a fixed column DoF (x is identically 0 there, so
// template * x = 0 = entry * x).
template <class Zero>
bool template_node(const biot::HostOperator &op, int64_t i, const double *tb, Zero zero) {
    const int nc = op.nc, d = op.d, S = op.n_slots, WB = biot::block_width(nc);
    for (int c = 0; c < nc; ++c)
        if (op.fixed[(size_t)i * nc + c]) return false;
    const double *b = op.blk.data() + (size_t)i * S * WB;
    for (int s = 0; s < S; ++s) {
        const int64_t j = i + op.offsets[s];
        for (int k = 0; k <= nc * nc; ++k) {
            const double v = b[s * WB + k];
            if (zero(s, k)) {
                if (v != 0.0) return false;
                continue;
            }
            if (k == nc * nc - 1) continue;
            if (same_entry(v, tb[s * WB + k])) continue;
            const int cc = k < nc * nc ? k % nc : d;
            const bool col_fixed = j >= 0 && j < op.n_nodes && op.fixed[(size_t)j * nc + cc];
            if (v == 0.0 && col_fixed) continue;
            return false;
        }
    }
    return true;
}

// Geometric classes of the structured n1^3 Kuhn cube (x, y, z each in {0, interior,
// n1-1}: 27 classes).  On the uniform mesh every node of a class has the same blocks
// wherever its row and column DoFs are free and the neighbour exists (AA_pp aside,
// which is per node and travels in the aux record): fixed columns meet x = 0, fixed
// rows are masked in the epilogue (D^{-1} = 0), missing neighbours are zero-filled,
// so the class stencil reproduces every node's own blocks.  cls[c][s][18] holds the
// AA block column-major (cls[..][cc*4 + c] = AA[c][cc]) and A'_pp at 16.  Returns
// false if some node disagrees with its class (then tile3d is not used).
bool tile3d_classes(const biot::HostOperator &op, int64_t n1, std::vector<double> &cls) {
    constexpr int CW = biot::Tile3dArgs::kClsW;
    const int S = op.n_slots, WB = biot::block_width(op.nc);
    const int sdx[15] = {0, -1, 0, -1, 0, -1, 0, -1, 1, 0, 1, 0, 1, 0, 1};
    const int sdy[15] = {0, -1, -1, 0, 0, -1, -1, 0, 0, 1, 1, 0, 0, 1, 1};
    const int sdz[15] = {0, -1, -1, -1, -1, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1};
    auto ac = [&](int64_t v) { return v == 0 ? 0 : (v == n1 - 1 ? 2 : 1); };
    cls.assign((size_t)27 * S * CW, 0.0);
    std::vector<uint8_t> have(cls.size(), 0);
    for (int pass = 0; pass < 2; ++pass)
        for (int64_t i = 0; i < op.n_nodes; ++i) {
            const int64_t x = i % n1, y = (i / n1) % n1, z = i / (n1 * n1);
            const int cl = ac(x) + 3 * ac(y) + 9 * ac(z);
            const double *b = op.blk.data() + (size_t)i * S * WB;
            for (int q = 0; q < S; ++q) {
                const int64_t xx = x + sdx[q], yy = y + sdy[q], zz = z + sdz[q];
                if (xx < 0 || yy < 0 || zz < 0 || xx >= n1 || yy >= n1 || zz >= n1) continue;
                const int64_t j = (zz * n1 + yy) * n1 + xx;
                for (int k = 0; k <= 16; ++k) {
                    if (k == 15) continue;
                    const int rc = k < 16 ? k / 4 : 3, cc = k < 16 ? k % 4 : 3;
                    if (op.fixed[(size_t)i * 4 + rc] || op.fixed[(size_t)j * 4 + cc]) continue;
                    const size_t o = ((size_t)cl * S + q) * CW + (k < 16 ? cc * 4 + rc : 16);
                    const double v = b[q * WB + k];
                    if (pass == 0 && !have[o]) { cls[o] = v; have[o] = 1; }
                    if (pass == 1 && !same_entry(v, cls[o])) return false;
                }
            }
        }
    return true;
}

// Geometric classes of the structured 2D grid (column and row each in {0, interior,
// last}: 9 classes), as tile3d_classes: cls[c][s][10] holds the AA block
// column-major (cls[..][cc*3 + c] = AA[c][cc]) and A'_pp at 9.
bool tile2d_classes(const biot::HostOperator &op, int64_t W, int64_t nrows, std::vector<double> &cls) {
    constexpr int CW = biot::Tile2dArgs::kClsW;
    const int S = op.n_slots, WB = biot::block_width(op.nc);
    const int sdc[7] = {0, -1, 0, -1, 1, 0, 1};
    const int sdr[7] = {0, -1, -1, 0, 0, 1, 1};
    auto ac = [](int64_t v, int64_t n) { return v == 0 ? 0 : (v == n - 1 ? 2 : 1); };
    cls.assign((size_t)9 * S * CW, 0.0);
    std::vector<uint8_t> have(cls.size(), 0);
    for (int pass = 0; pass < 2; ++pass)
        for (int64_t i = 0; i < op.n_nodes; ++i) {
            const int64_t x = i % W, y = i / W;
            const int cl = ac(x, W) + 3 * ac(y, nrows);
            const double *b = op.blk.data() + (size_t)i * S * WB;
            for (int q = 0; q < S; ++q) {
                const int64_t xx = x + sdc[q], yy = y + sdr[q];
                if (xx < 0 || yy < 0 || xx >= W || yy >= nrows) continue;
                const int64_t j = yy * W + xx;
                for (int k = 0; k <= 9; ++k) {
                    if (k == 8) continue;
                    const int rc = k < 9 ? k / 3 : 2, cc = k < 9 ? k % 3 : 2;
                    if (op.fixed[(size_t)i * 3 + rc] || op.fixed[(size_t)j * 3 + cc]) continue;
                    const size_t o = ((size_t)cl * S + q) * CW + (k < 9 ? cc * 3 + rc : 9);
                    const double v = b[q * WB + k];
                    if (pass == 0 && !have[o]) { cls[o] = v; have[o] = 1; }
                    if (pass == 1 && !same_entry(v, cls[o])) return false;
                }
            }
        }
    return true;
}

// Recognise the BDIA offset sets of the structured meshes (2D right triangles,
// 3D Kuhn tetrahedra) and fill the run tables of the register-blocked kernel.
bool detect_stencil(biot_ctx *c) {
    if (c->path != biot::PATH_BDIA) return false;
    std::vector<int64_t> o(c->offsets.begin(), c->offsets.end());
    std::sort(o.begin(), o.end());
    o.erase(std::unique(o.begin(), o.end()), o.end());
    auto idx = [&](int64_t off) -> int {
        for (size_t s = 0; s < c->offsets.size(); ++s)
            if (c->offsets[s] == off) return (int)s;
        return -1;
    };
    std::vector<int64_t> bases;
    std::vector<std::pair<int, int>> ranges;
    if (c->d == 2) {
        if (o.size() != 7) return false;
        const int64_t W = o.back() - 1;
        std::vector<int64_t> want = {-W - 1, -W, -1, 0, 1, W, W + 1};
        if (W < 3 || o != want) return false;
        bases = {-W, 0, W};
        ranges = {{-1, 0}, {-1, 1}, {0, 1}};
    } else {
        if (o.size() != 15) return false;
        int64_t W = 0;
        for (int64_t v : o)
            if (v > 1) { W = v; break; }
        const int64_t V = W * W;
        std::vector<int64_t> want = {0, 1, -1, W, -W, V, -V, 1 + W, -1 - W, 1 + V, -1 - V,
                                     W + V, -W - V, 1 + W + V, -1 - W - V};
        std::sort(want.begin(), want.end());
        if (W < 3 || o != want) return false;
        bases = {-W - V, -V, -W, 0, W, V, W + V};
        ranges = {{-1, 0}, {-1, 0}, {-1, 0}, {-1, 1}, {0, 1}, {0, 1}, {0, 1}};
    }
    for (size_t g = 0; g < bases.size(); ++g) {
        c->gbase[g] = bases[g];
        for (int a = ranges[g].first; a <= ranges[g].second; ++a) {
            const int s = idx(bases[g] + a);
            if (s < 0) return false;
            c->slot[g][a - ranges[g].first] = s;
        }
    }
    return true;
}


// A time window of the panel (Gauss-Seidel waves): steps [t_off, t_off + len), the
// predecessor of step t_off read from `ghost` with stride `stride`.
struct Window {
    int t_off = 0, len = 0, t_lo = 0;   // t_lo: window steps below it are not stored (alignment)
    const double *ghost = nullptr;
    int64_t stride = 1;
    double *send = nullptr;             // send slice (only when the window ends at the slab's last step)
    bool lead = false;                  // the window starts 2 steps early (see gs_window): no ghost
};

// tmo / zb (tile kernels only): the tensor map of xin and the Z panel, when they are not
// the context's own (the GMRES Krylov panels).
cudaError_t launch_main(biot_ctx *c, int mode, const double *xin, double *xout, const Window *win = nullptr,
                        const CUtensorMap *tmo = nullptr, double *zb = nullptr) {
    if (c->kern == 6) {
        biot::Tile3dArgs a{};
        static_cast<biot::SweepArgs &>(a) = sweep_args(c, mode, xin, xout);
        std::memcpy(a.tmpl, c->tmpl3, sizeof(a.tmpl));
        a.aux = c->aux;
        a.cls = c->cls;
        a.n1 = c->n1;
        a.z_rows = c->z_rows;
        a.s0 = c->s0;
        a.dry = c->tile_dry;
        a.ghost_stride = 1;
        a.t_off = 0;
        a.t_lo = 0;
        if (win) {
            a.t_off = win->t_off;
            a.t_lo = win->t_lo;
            a.n_tl = win->len;
            a.ghost = win->ghost;
            a.ghost_stride = win->stride;
            a.sendbuf = win->send;
            if (win->ghost != c->ghost) a.ghost_zero = 0;
            if (win->lead) a.ghost_zero = 1;
        }
        if (zb) a.zbuf = zb;
        if (tmo) return biot::launch_tile3d(*tmo, a, c->shape, c->stream);
        if (mode == biot::MODE_PASS2) return biot::launch_tile3d(c->tmapz, a, c->shape, c->stream);
        return biot::launch_tile3d(c->tmap[xin == c->x[0] ? 0 : 1], a, c->shape, c->stream);
    }
    if (c->kern == 4) {
        biot::Tile2dArgs a{};
        static_cast<biot::SweepArgs &>(a) = sweep_args(c, mode, xin, xout);
        std::memcpy(a.tmpl, c->tmpl, sizeof(a.tmpl));
        a.aux = c->aux;
        a.cls = c->cls;
        a.pad_nodes = c->pad;
        a.aux_geo = c->aux_geo;
        a.ux0 = c->ux0;
        a.ux1 = c->ux1;
        a.uy0 = c->uy0;
        a.uy1 = c->uy1;
        std::memcpy(a.aux_u, c->aux_u, sizeof(a.aux_u));
        a.n_rblk = c->n_rblk;
        if (mode == biot::MODE_P1_FUSED) {
            a.rows_per_tile = c->rows_per_tile_p1;
            a.n_rblk = 0;
        }
        a.ghost_stride = 1;
        a.t_off = 0;
        a.t_lo = 0;
        if (win) {
            a.t_off = win->t_off;
            a.t_lo = win->t_lo;
            a.n_tl = win->len;
            a.ghost = win->ghost;
            a.ghost_stride = win->stride;
            a.sendbuf = win->send;
            if (win->ghost != c->ghost) a.ghost_zero = 0;
            if (win->lead) a.ghost_zero = 1;
        }
        a.s0 = c->s0;
        a.dry = c->tile_dry;
        if (zb) a.zbuf = zb;
        if (tmo) return biot::launch_tile2d(*tmo, a, c->shape, c->stream);
        if (mode == biot::MODE_PASS2) return biot::launch_tile2d(c->tmapz, a, c->shape, c->stream);
        return biot::launch_tile2d(c->tmap[xin == c->x[0] ? 0 : 1], a, c->shape, c->stream);
    }
    biot::SweepArgs a = sweep_args(c, mode, xin, xout);
    if (c->kern == 3) return biot::launch_march(c->mT, a, c->shape, c->stream);
    return biot::launch_sweep(c->d, c->path, c->S, a, c->shape, c->stream);
}

// P~1 second pass: the 2D tile mode on the Z panel, else the generic kernel.
cudaError_t launch_pass2_any(biot_ctx *ctx, const double *xin, double *xout, double *sendbuf, const Window *win) {
    if (ctx->kern == 4 || ctx->kern == 6) return launch_main(ctx, biot::MODE_PASS2, xin, xout, win);
    biot::Pass2Args p{};
    p.x = xin;
    p.xn = xout;
    p.zbuf = ctx->z;
    p.blk = ctx->blk;
    p.cols = ctx->cols;
    p.dinv = ctx->dinv;
    p.sendbuf = sendbuf;
    p.n_nodes = ctx->N;
    p.pitch = ctx->pitch;
    p.n_tl = win ? win->len : ctx->n_tl;
    p.t_off = win ? win->t_off : 0;
    p.t_lo = win ? win->t_lo : 0;
    if (win) p.sendbuf = win->send;
    p.tw = ctx->tw;
    p.node_block = ctx->node_block;
    p.omega = ctx->omega;
    for (int s = 0; s < 32; ++s) p.off[s] = s < (int)ctx->offsets.size() ? ctx->offsets[s] : 0;
    return biot::launch_pass2(ctx->d, ctx->path, ctx->S, p, ctx->pass2_grid, ctx->stream);
}

// With the overlapped exchange the persistent tile kernels leave BIOT_COMM_SMS (default 2)
// SMs free, so NCCL's send/recv kernel is scheduled while the sweep runs instead of after it.
void reserve_comm_sms(biot_ctx *c) {
    if (!c->overlap && !(c->flags & BIOT_FLAG_DEFER_STEP0)) return;
    int r = 2;
    if (const char *e = std::getenv("BIOT_COMM_SMS")) r = std::max(0, std::atoi(e));
    c->shape.grid = std::max(1, c->shape.grid - r);
}

// norm-partial groups written by a pass of `mode`
int64_t groups_of(const biot_ctx *c, int mode) { return mode == biot::MODE_P1_FUSED ? c->groups_p1 : c->groups; }

// the preconditioner pass of one outer iteration: P~2, fused P~1, or P~1's first pass
int main_mode(const biot_ctx *c) {
    return c->precond == 2 ? biot::MODE_UPDATE_P2 : c->p1_fused ? biot::MODE_P1_FUSED : biot::MODE_P1_PASS1;
}

// The kernels of one outer iteration from panel `cur` (sweep, P~1 pass 2 if two-pass,
// norm finalize).  graph_slot >= 0: the finalize writes history slot d_iter + graph_slot
// (read on the device: replayable in a CUDA graph) and the events are graph nodes.
biot_status enqueue_iteration(biot_ctx *ctx, int cur, cudaEvent_t e0, cudaEvent_t e1, int graph_slot,
                              bool finalize = true) {
    const double *xin = ctx->x[cur];
    double *xout = ctx->x[1 - cur];
    const int mode = main_mode(ctx);
    biot::SweepArgs a = sweep_args(ctx, mode, xin, xout);
    const unsigned evf = graph_slot >= 0 ? cudaEventRecordExternal : cudaEventRecordDefault;
    // timed span: every pass of the preconditioner (P~1 two-pass: both)
    if (e0) CU(cudaEventRecordWithFlags(e0, ctx->stream, evf));
    CU(launch_main(ctx, mode, xin, xout));
    if (mode == biot::MODE_P1_PASS1) CU(launch_pass2_any(ctx, xin, xout, a.sendbuf, nullptr));
    if (e1) CU(cudaEventRecordWithFlags(e1, ctx->stream, evf));
    if (!finalize) return BIOT_OK;
    if (graph_slot >= 0) {
        CU(biot::launch_finalize(ctx->partial, (int)groups_of(ctx, mode), ctx->n_tl, ctx->hist, ctx->nonfinite,
                                 ctx->fin_scratch, ctx->stream, ctx->d_iter, graph_slot, ctx->hist_cap,
                                 ctx->fin_tickets));
    } else {
        double *hslot = ctx->hist + (size_t)(ctx->iterations % ctx->hist_cap) * ctx->n_tl * 2;
        CU(biot::launch_finalize(ctx->partial, (int)groups_of(ctx, mode), ctx->n_tl, hslot, ctx->nonfinite,
                                 ctx->fin_scratch, ctx->stream, nullptr, 0, 1, ctx->fin_tickets));
    }
    return BIOT_OK;
}

// The deferred first local step of the current iterate (after the ghost is in place):
// recompute it for every node with the ghost, overwrite x^{k+1} there (and the send slice
// if the slab is one step), and replace the step's norms in history slot `hslot`.
biot_status complete_step0(biot_ctx *ctx, int mode, const double *xin, double *xout, double *hslot) {
    if (ctx->kern == 4) {
        biot::Tile2dArgs a{};
        static_cast<biot::SweepArgs &>(a) = sweep_args(ctx, mode, xin, xout);
        a.ghost = ctx->ghost;
        a.ghost_zero = 0;
        a.s0buf = ctx->s0buf;
        std::memcpy(a.tmpl, ctx->tmpl, sizeof(a.tmpl));
        a.aux = ctx->aux;
        a.cls = ctx->cls;
        a.pad_nodes = ctx->pad;
        a.ghost_stride = 1;
        a.s0 = ctx->s0;
        CU(biot::launch_tile2d_step0(a, ctx->part0, ctx->stream));
    } else {
        biot::Tile3dArgs a{};
        static_cast<biot::SweepArgs &>(a) = sweep_args(ctx, mode, xin, xout);
        a.ghost = ctx->ghost;
        a.ghost_zero = 0;
        a.s0buf = ctx->s0buf;
        std::memcpy(a.tmpl, ctx->tmpl3, sizeof(a.tmpl));
        a.aux = ctx->aux;
        a.cls = ctx->cls;
        a.n1 = ctx->n1;
        a.z_rows = ctx->z_rows;
        a.s0 = ctx->s0;
        a.ghost_stride = 1;
        CU(biot::launch_tile3d_step0(a, ctx->part0, ctx->stream));
    }
    // the norms of the iteration, with step 0's p-part from the completion's partials
    CU(biot::launch_finalize(ctx->partial, (int)groups_of(ctx, mode), ctx->n_tl, hslot, ctx->nonfinite,
                             ctx->fin_scratch, ctx->stream, nullptr, 0, 1, ctx->fin_tickets, ctx->part0,
                             ctx->step0_blocks));
    return BIOT_OK;
}

biot_status one_iteration(biot_ctx *ctx, cudaEvent_t e0, cudaEvent_t e1) {
    biot_status st = BIOT_OK;
    if (!ctx->overlap) {
        if ((st = halo_exchange(ctx)) != BIOT_OK) return st;
    } else {
        // the exchange of x^k's last slice on the comm stream, concurrent with the sweep,
        // which writes x^{k+1}'s slice into the other buffer (the compute stream first waits
        // for the previous exchange: it sent the buffer this sweep overwrites)
        NcclApi *api = nccl();
        if (!api || !ctx->comm) return fail(ctx, BIOT_E_NCCL, "NCCL not initialised");
        if (ctx->send_dirty) {
            if ((st = pack_send(ctx)) != BIOT_OK) return st;
        }
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_comm, 0));
        CU(cudaEventRecord(ctx->ev_ready, ctx->stream));
        CU(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_ready, 0));
        const size_t n = (size_t)ctx->N * ctx->nc;
        ncclResult_t r = api->GroupStart();
        if (r == ncclSuccess && ctx->rank + 1 < ctx->world)
            r = api->Send(ctx->sendbuf, n, ncclFloat64, ctx->rank + 1, ctx->comm, ctx->comm_stream);
        if (r == ncclSuccess && ctx->rank > 0)
            r = api->Recv(ctx->ghost, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->comm_stream);
        ncclResult_t r2 = api->GroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(ctx, BIOT_E_NCCL, std::string("NCCL halo exchange failed: ") +
                                              (api->GetErrorString ? api->GetErrorString(r != ncclSuccess ? r : r2) : "?"));
        CU(cudaEventRecord(ctx->ev_comm, ctx->comm_stream));
        ctx->send_w = ctx->sendbuf2;
    }
    const int mode = main_mode(ctx);
    double *hslot = ctx->hist + (size_t)(ctx->iterations % ctx->hist_cap) * ctx->n_tl * 2;
    if (ctx->defer0) ctx->ghost_override = ctx->zero_ghost;
    st = enqueue_iteration(ctx, ctx->cur, e0, e1, -1, !ctx->defer0);   // deferred: finalized after step 0
    ctx->ghost_override = nullptr;
    if (st == BIOT_OK && ctx->defer0) {
        if (ctx->overlap) CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_comm, 0));   // the ghost arrived
        st = complete_step0(ctx, mode, ctx->x[ctx->cur], ctx->x[1 - ctx->cur], hslot);
    }
    if (ctx->overlap) {
        std::swap(ctx->sendbuf, ctx->sendbuf2);        // the slice just written is the current one
        ctx->send_w = ctx->sendbuf;
    }
    if (st != BIOT_OK) return st;
    ctx->cur = 1 - ctx->cur;
    ctx->iterations++;
    if (ctx->world > 1) ctx->send_dirty = false;   // the sweep (and pass 2) wrote the slice of x^{k+1}
    return BIOT_OK;
}

// Capture two outer iterations starting from panel `cur` (ending on it again) and the
// history-counter advance into an executable graph.  Capture runs on a private stream
// (the context's stream may be the legacy default stream, which cannot capture).
biot_status build_graph(biot_ctx *ctx, int cur) {
    if (!ctx->cap_stream) CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    for (cudaEvent_t &e : ctx->gev)
        if (!e) CU(cudaEventCreate(&e));
    cudaStream_t saved = ctx->stream;
    ctx->stream = ctx->cap_stream;
    cudaError_t e = cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed);
    biot_status st = BIOT_OK;
    if (e == cudaSuccess) {
        st = enqueue_iteration(ctx, cur, ctx->gev[0], ctx->gev[1], 0);
        if (st == BIOT_OK) st = enqueue_iteration(ctx, 1 - cur, ctx->gev[2], ctx->gev[3], 1);
        if (st == BIOT_OK) {
            cudaError_t e2 = biot::launch_counter(ctx->d_iter, 2, true, ctx->cap_stream);
            if (e2 != cudaSuccess) st = fail(ctx, BIOT_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e2));
        }
    }
    cudaGraph_t g = nullptr;
    cudaError_t e3 = cudaStreamEndCapture(ctx->cap_stream, &g);
    ctx->stream = saved;
    if (e != cudaSuccess) return fail(ctx, BIOT_E_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
    if (st != BIOT_OK) {
        if (g) cudaGraphDestroy(g);
        return st;
    }
    if (e3 != cudaSuccess) return fail(ctx, BIOT_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e3));
    e = cudaGraphInstantiate(&ctx->gexec[cur], g, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(g);
        return fail(ctx, BIOT_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    }
    // the sweep-span event-record nodes, so that biot_iterate can time sampled replays
    size_t nn = 0;
    CU(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CU(cudaGraphGetNodes(g, nodes.data(), &nn));
    for (cudaGraphNode_t n : nodes) {
        cudaGraphNodeType ty;
        CU(cudaGraphNodeGetType(n, &ty));
        if (ty != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev = nullptr;
        CU(cudaGraphEventRecordNodeGetEvent(n, &ev));
        for (int h = 0; h < 4; ++h)
            if (ev == ctx->gev[h]) ctx->gnode[cur][h] = n;
    }
    ctx->gsrc[cur] = g;
    return BIOT_OK;
}

// Wait for event `ev` on the host.  With an NCCL communicator, poll its asynchronous
// error state meanwhile: a failed or silent peer (no progress for nccl_timeout_s) aborts
// the communicator and returns BIOT_E_NCCL instead of hanging.
biot_status wait_done(biot_ctx *ctx, cudaEvent_t ev) {
    NcclApi *api = ctx->comm ? nccl() : nullptr;
    if (!api || !api->CommGetAsyncError) {
        CU(cudaEventSynchronize(ev));
        return BIOT_OK;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t q = cudaEventQuery(ev);
        if (q == cudaSuccess) return BIOT_OK;
        if (q != cudaErrorNotReady) return fail(ctx, BIOT_E_CUDA, std::string("cudaEventQuery: ") + cudaGetErrorString(q));
        ncclResult_t ar = ncclSuccess;
        api->CommGetAsyncError(ctx->comm, &ar);
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if ((ar != ncclSuccess && ar != ncclInProgress) || el > ctx->nccl_timeout_s) {
            if (api->CommAbort) api->CommAbort(ctx->comm);
            ctx->comm = nullptr;
            return fail(ctx, BIOT_E_NCCL, ar != ncclSuccess && ar != ncclInProgress
                                              ? std::string("NCCL asynchronous error: ") +
                                                    (api->GetErrorString ? api->GetErrorString(ar) : "?")
                                              : "NCCL halo exchange made no progress within BIOT_NCCL_TIMEOUT_S (" +
                                                    std::to_string(ctx->nccl_timeout_s) + " s): communicator aborted");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

biot_status wait_stream(biot_ctx *ctx) {
    CU(cudaEventRecord(ctx->ev_b, ctx->stream));
    return wait_done(ctx, ctx->ev_b);
}

}  // namespace

// Per-step GMRES inside the inverted scheme (Alg. 3, with K =
// GMRES as the paper's experiments use; reading R23): each outer iteration
// runs, for every time step at once, one cycle of GMRES(k) on AA x_n = b_n from
// x_n^{m-1}, left-preconditioned by the diagonal P~2, b_n = A' x_{n-1}^{m-1} + f_n
// (Jacobi in time).  The N_t Krylov bases live in k+1 space-time panels; Arnoldi by
// classical Gram-Schmidt with one reorthogonalisation (CGS2), every dot product and
// update column-wise (one value per time step); the (k+1) x k least-squares problems
// are solved on the device by Givens rotations (one thread per step).
namespace {

biot_status gmres_alloc(biot_ctx *ctx, int k) {
    if ((int)ctx->gm_V.size() >= k + 1) return BIOT_OK;
    const size_t panel_bytes = (size_t)ctx->rows_alloc * ctx->pitch * sizeof(double);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qres;
    CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres));
    if (!fn || qres != cudaDriverEntryPointSuccess)
        return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled not available");
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    while ((int)ctx->gm_V.size() < k + 1) {
        double *base = nullptr;
        ALLOC(base, panel_bytes);
        CU(cudaMemsetAsync(base, 0, panel_bytes, ctx->stream));
        ctx->gm_Vbase.push_back(base);
        double *v0 = base + ctx->pad * ctx->nc * ctx->pitch;
        ctx->gm_V.push_back(v0);
        CUtensorMap m;
        CUresult r;
        if (ctx->kern == 4) {   // as the 2D x panels: {time, panel rows}
            uint32_t box[2];
            biot::tile2d_box(box);
            cuuint64_t dims[2] = {(cuuint64_t)ctx->pitch, (cuuint64_t)ctx->rows_alloc};
            cuuint64_t strides[1] = {(cuuint64_t)ctx->pitch * sizeof(double)};
            cuuint32_t bx[2] = {box[0], box[1]};
            cuuint32_t es[2] = {1, 1};
            r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, bx, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {                // as the 3D x panels: {time, x*4 + c, y, z} at node 0
            uint32_t box[4];
            biot::tile3d_box(box);
            const int64_t n1 = ctx->n1;
            cuuint64_t dims[4] = {(cuuint64_t)ctx->pitch, (cuuint64_t)(n1 * 4), (cuuint64_t)n1, (cuuint64_t)n1};
            const cuuint64_t rb = (cuuint64_t)ctx->pitch * sizeof(double);
            cuuint64_t strides[3] = {rb, rb * (cuuint64_t)(n1 * 4), rb * (cuuint64_t)(n1 * n1 * 4)};
            cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
            cuuint32_t es[4] = {1, 1, 1, 1};
            r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, v0, dims, strides, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled (V) failed");
        ctx->gm_tmap.push_back(m);
    }
    const int nv = (int)ctx->gm_V.size();
    if (ctx->gm_Vdev) cudaFree(ctx->gm_Vdev);
    ctx->gm_Vdev = nullptr;
    ALLOC(ctx->gm_Vdev, nv * sizeof(double *));
    CU(h2d(ctx, ctx->gm_Vdev, ctx->gm_V.data(), nv * sizeof(double *)));
    int64_t chunk;
    int chunks;
    const int64_t scr = biot::gmres_dots_scratch(ctx->N * ctx->nc, ctx->n_tl, biot::gmres_max_vectors(), &chunk, &chunks);
    if (ctx->gm_scratch) cudaFree(ctx->gm_scratch);
    if (ctx->gm_small) cudaFree(ctx->gm_small);
    ctx->gm_scratch = ctx->gm_small = nullptr;
    ALLOC(ctx->gm_scratch, scr * sizeof(double));
    // small per-step arrays: dot results, scale, beta, y, and the Hessenberg matrices
    const int mv = biot::gmres_max_vectors();
    ALLOC(ctx->gm_small, (size_t)(2 * mv + 2 + mv * (mv - 1)) * ctx->n_tl * sizeof(double));
    return BIOT_OK;
}

}  // namespace

namespace {

// Compact basis for a window of nt <= kCompactMax columns: k + 1 vectors of rows x w
// doubles, w = nt rounded up to 16 (reallocated when a wider window comes).  An allocation
// failure is not an error: the cycle then keeps the basis in the panel layout.
constexpr int kCompactMax = 64;
bool gmres_compact_alloc(biot_ctx *ctx, int k, int nt) {
    const int w = (nt + 15) / 16 * 16;
    if (ctx->gm_Vc && ctx->gm_vc_w >= w && ctx->gm_vc_n >= k + 1) return true;
    const int ww = std::max(w, ctx->gm_vc_w), nn = std::max(k + 1, ctx->gm_vc_n);
    if (ctx->gm_Vc) cudaFree(ctx->gm_Vc);
    if (ctx->gm_Vcdev) cudaFree(ctx->gm_Vcdev);
    ctx->gm_Vc = nullptr;
    ctx->gm_Vcdev = nullptr;
    ctx->gm_vc_w = ctx->gm_vc_n = 0;
    const size_t vec = (size_t)ctx->N * ctx->nc * ww;
    if (cudaMalloc((void **)&ctx->gm_Vc, vec * nn * sizeof(double)) != cudaSuccess ||
        cudaMalloc((void **)&ctx->gm_Vcdev, nn * sizeof(double *)) != cudaSuccess) {
        cudaGetLastError();
        if (ctx->gm_Vc) cudaFree(ctx->gm_Vc);
        ctx->gm_Vc = nullptr;
        return false;
    }
    std::vector<double *> ptrs(nn);
    for (int i = 0; i < nn; ++i) ptrs[i] = ctx->gm_Vc + vec * i;
    if (cudaMemcpy(ctx->gm_Vcdev, ptrs.data(), nn * sizeof(double *), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    ctx->gm_vc_w = ww;
    ctx->gm_vc_n = nn;
    return true;
}

// One GMRES(k) cycle for every step of a time window (R23): x_out = x_in + V y on
// columns [t_off + t_lo, t_off + len), the residual (with its previous-step coupling and
// norm partials) from panel xin through tensor map `tm`.  x_out may equal x_in.
biot_status gmres_cycle(biot_ctx *ctx, int k, const CUtensorMap &tm, const double *xin, double *xout,
                        const Window &win) {
    // Everything stays on the device (no host round trip): the dot kernels accumulate the
    // Hessenberg columns and produce the normalisation scales, the least-squares problems
    // are solved by one thread per step, and the combination kernels read the
    // coefficients where the dots left them.
    const int64_t rows = ctx->N * ctx->nc;
    const int c0 = win.t_off + win.t_lo, nt = win.len - win.t_lo;   // columns the cycle owns
    const int mv = biot::gmres_max_vectors();
    double *d_h = ctx->gm_small;                           // [mv][nt] dot results
    double *d_scale = d_h + (size_t)mv * ctx->n_tl;        // [nt]
    double *d_beta = d_scale + ctx->n_tl;                  // [nt]
    double *d_y = d_beta + ctx->n_tl;                      // [mv][nt]
    double *d_H = d_y + (size_t)mv * ctx->n_tl;            // [(k+1) k][nt]
    double *const *Vd = ctx->gm_Vdev;
    auto hcol = [&](int i, int j) { return d_H + (size_t)(i + j * (k + 1)) * nt; };
    const int64_t P = ctx->pitch;
    const biot::GmresPitch full{P, P, P, 0};
    auto dots = [&](const double *a, double *const *bdev, int nb, double *out, double *hacc, bool norm) {
        return biot::gmres_dots(a + c0, bdev, c0, nb, rows, P, nt, ctx->gm_scratch, out, hacc, norm, ctx->stream);
    };
    auto combine = [&](double *dst, const double *base, const double *coef, int nb, double sign,
                       const double *scale) {
        return biot::gmres_combine(dst + c0, base + c0, Vd, c0, coef, nb, sign, scale, rows, full, nt, ctx->stream);
    };
    Window w = win;          // tile passes of the cycle never write the send slice
    w.send = nullptr;
    // P~1 (eq. p1): the tile passes write the first half (z_u, r_p) of P~1^{-1} r; this pass
    // completes z_p = D_S^{-1} (B^T z_u - r_p) in place on the window's columns of panel V
    auto p1_complete = [&](double *V) -> cudaError_t {
        if (ctx->precond != 1) return cudaSuccess;
        biot::Pass2Args p{};
        p.x = V;
        p.xn = V;
        p.zbuf = V;
        p.blk = ctx->blk;
        p.cols = ctx->cols;
        p.dinv = ctx->dinv;
        p.sendbuf = nullptr;
        p.n_nodes = ctx->N;
        p.pitch = ctx->pitch;
        p.n_tl = w.len;
        p.t_off = w.t_off;
        p.t_lo = w.t_lo;
        p.tw = ctx->tw;
        p.node_block = ctx->node_block;
        p.omega = 1.0;
        p.pure = 1;
        for (int s = 0; s < 32; ++s) p.off[s] = s < (int)ctx->offsets.size() ? ctx->offsets[s] : 0;
        return biot::launch_pass2(ctx->d, ctx->path, ctx->S, p, ctx->pass2_grid, ctx->stream);
    };
    CU(cudaMemsetAsync(d_H, 0, (size_t)(k + 1) * k * nt * sizeof(double), ctx->stream));
    if (nt <= kCompactMax && !std::getenv("BIOT_GMRES_NO_COMPACT") && gmres_compact_alloc(ctx, k, nt)) {
        // Narrow window: the Krylov basis proper lives compact (row pitch nt, every dot and
        // combination streams contiguous memory); the panel-layout V_j stay the tile passes'
        // input/output only.  Per Arnoldi step: the matvec pass writes V_{j+1} (panel), one
        // gather makes it compact, CGS2 and the norm run compact, and the normalising pass
        // writes both copies.  Same arithmetic in the same order as the panel form (the dot
        // order depends on the row chunking only): results are bitwise those of that form.
        double *const *Vc = ctx->gm_Vcdev;
        std::vector<double *> vc(k + 1);
        for (int i = 0; i <= k; ++i) vc[i] = ctx->gm_Vc + (size_t)rows * ctx->gm_vc_w * i;
        const int64_t cw = nt;   // compact row pitch: the window itself
        auto cdots = [&](const double *a, double *const *bdev, int nb, double *out, double *hacc, bool norm) {
            return biot::gmres_dots(a, bdev, 0, nb, rows, cw, nt, ctx->gm_scratch, out, hacc, norm, ctx->stream);
        };
        auto gather = [&](double *dst, const double *panel) {   // compact <- panel window
            return biot::gmres_combine(dst, panel + c0, Vc, 0, nullptr, 0, 1.0, nullptr, rows,
                                       biot::GmresPitch{cw, P, cw, 0}, nt, ctx->stream);
        };
        auto cnorm = [&](double *vcj, double *panel) {   // v = scale v, compact and panel copies
            return biot::gmres_combine(vcj, vcj, Vc, 0, nullptr, 0, 1.0, d_scale, rows,
                                       biot::GmresPitch{cw, cw, cw, P}, nt, ctx->stream, panel + c0);
        };
        CU(launch_main(ctx, biot::MODE_ZOUT, xin, nullptr, &w, &tm, ctx->gm_V[0]));
        CU(p1_complete(ctx->gm_V[0]));
        CU(gather(vc[0], ctx->gm_V[0]));
        CU(cdots(vc[0], Vc, 1, d_scale, d_beta, true));
        CU(cnorm(vc[0], ctx->gm_V[0]));
        for (int j = 0; j < k; ++j) {
            CU(launch_main(ctx, biot::MODE_MATVEC, ctx->gm_V[j], ctx->gm_V[j + 1], &w, &ctx->gm_tmap[j]));
            CU(p1_complete(ctx->gm_V[j + 1]));
            CU(gather(vc[j + 1], ctx->gm_V[j + 1]));
            for (int pass = 0; pass < 2; ++pass) {
                CU(cdots(vc[j + 1], Vc, j + 1, d_h, hcol(0, j), false));
                CU(biot::gmres_combine(vc[j + 1], vc[j + 1], Vc, 0, d_h, j + 1, -1.0, nullptr, rows,
                                       biot::GmresPitch{cw, cw, cw, 0}, nt, ctx->stream));
            }
            CU(cdots(vc[j + 1], Vc + (j + 1), 1, d_scale, hcol(j + 1, j), true));
            if (j + 1 < k) {
                CU(cnorm(vc[j + 1], ctx->gm_V[j + 1]));
            } else {   // the last basis vector feeds no matvec pass: compact only
                CU(biot::gmres_combine(vc[j + 1], vc[j + 1], Vc, 0, nullptr, 0, 1.0, d_scale, rows,
                                       biot::GmresPitch{cw, cw, cw, 0}, nt, ctx->stream));
            }
        }
        CU(biot::gmres_lsq(d_H, d_beta, k, nt, d_y, ctx->stream));
        CU(biot::gmres_combine(xout + c0, xin + c0, Vc, 0, d_y, k, 1.0, nullptr, rows, biot::GmresPitch{P, P, cw, 0},
                               nt, ctx->stream));
        return BIOT_OK;
    }
    // v_0 = P~2^{-1} (b - AA x_in) with b = A' x_prev + f, and the norms of b - AA x_in
    CU(launch_main(ctx, biot::MODE_ZOUT, xin, nullptr, &w, &tm, ctx->gm_V[0]));
    CU(p1_complete(ctx->gm_V[0]));
    CU(dots(ctx->gm_V[0], Vd, 1, d_scale, d_beta, true));              // beta_t, 1 / beta_t
    CU(combine(ctx->gm_V[0], ctx->gm_V[0], nullptr, 0, 1.0, d_scale));
    for (int j = 0; j < k; ++j) {
        // w = P~2^{-1} AA v_j into v_{j+1}
        CU(launch_main(ctx, biot::MODE_MATVEC, ctx->gm_V[j], ctx->gm_V[j + 1], &w, &ctx->gm_tmap[j]));
        CU(p1_complete(ctx->gm_V[j + 1]));
        // CGS2: two passes of h = V^T w (accumulated into column j of H), w -= V h
        for (int pass = 0; pass < 2; ++pass) {
            CU(dots(ctx->gm_V[j + 1], Vd, j + 1, d_h, hcol(0, j), false));
            CU(combine(ctx->gm_V[j + 1], ctx->gm_V[j + 1], d_h, j + 1, -1.0, nullptr));
        }
        CU(dots(ctx->gm_V[j + 1], Vd + (j + 1), 1, d_scale, hcol(j + 1, j), true));   // h_{j+1,j}
        CU(combine(ctx->gm_V[j + 1], ctx->gm_V[j + 1], nullptr, 0, 1.0, d_scale));
    }
    // y_t = argmin || beta_t e1 - H_t y ||, x_out = x_in + V y
    CU(biot::gmres_lsq(d_H, d_beta, k, nt, d_y, ctx->stream));
    CU(combine(xout, xin, d_y, k, 1.0, nullptr));
    return BIOT_OK;
}

biot_status gmres_check(biot_ctx *ctx, int32_t K, int32_t k) {
    if (K < 0 || k < 1 || k > biot::gmres_max_vectors() - 1)
        return fail(ctx, BIOT_E_INVALID, "need K >= 0 and 1 <= k <= " + std::to_string(biot::gmres_max_vectors() - 1));
    if (ctx->kern != 4 && ctx->kern != 6)
        return fail(ctx, BIOT_E_STATE, "per-step GMRES needs a tile kernel (structured 2D / 3D mesh)");
    return BIOT_OK;
}

}  // namespace

extern "C" {

int32_t biot_abi_version(void) { return BIOT_PIT_ABI_VERSION; }

void biot_free(void *p) { std::free(p); }

biot_status biot_mesh_structured(int32_t dim, int32_t n, double **coords, int32_t **cells, int64_t *n_nodes,
                                 int64_t *n_cells) {
    if (!coords || !cells || !n_nodes || !n_cells) return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    if ((dim != 2 && dim != 3) || n < 1 || (dim == 3 ? (int64_t)n * n * n > 100000000LL : (int64_t)n * n > 1000000000LL))
        return fail(nullptr, BIOT_E_INVALID, "need dim in {2, 3} and a positive n of a supported size");
    const int64_t w = (int64_t)n + 1;
    const int64_t nn = dim == 2 ? w * w : w * w * w;
    const int64_t nc = dim == 2 ? 2LL * n * n : 6LL * n * n * n;
    double *X = static_cast<double *>(std::malloc((size_t)nn * dim * sizeof(double)));
    int32_t *C = static_cast<int32_t *>(std::malloc((size_t)nc * (dim + 1) * sizeof(int32_t)));
    if (!X || !C) {
        std::free(X);
        std::free(C);
        return fail(nullptr, BIOT_E_NOMEM, "host allocation failed");
    }
    if (dim == 2) {
        for (int64_t j = 0; j < w; ++j)
            for (int64_t i = 0; i < w; ++i) {
                X[(j * w + i) * 2 + 0] = (double)i / n;
                X[(j * w + i) * 2 + 1] = (double)j / n;
            }
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const int32_t n00 = (int32_t)(j * w + i), n10 = n00 + 1, n11 = (int32_t)(n00 + w + 1),
                              n01 = (int32_t)(n00 + w);
                int32_t *c = C + ((j * n + i) * 2) * 3;
                c[0] = n00; c[1] = n10; c[2] = n11;   // counter-clockwise
                c[3] = n00; c[4] = n11; c[5] = n01;
            }
    } else {
        for (int64_t k = 0; k < w; ++k)
            for (int64_t j = 0; j < w; ++j)
                for (int64_t i = 0; i < w; ++i) {
                    double *x = X + ((k * w + j) * w + i) * 3;
                    x[0] = (double)i / n;
                    x[1] = (double)j / n;
                    x[2] = (double)k / n;
                }
        const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        const int64_t stride[3] = {1, w, w * w};
        int64_t off[6][4];
        for (int p = 0; p < 6; ++p) {
            // vertices v, v+e_a, v+e_a+e_b, v+e_a+e_b+e_c; orientation from det[e_a; e_a+e_b; e_a+e_b+e_c]
            int e[3][3] = {{0}};
            e[0][perms[p][0]] = 1;
            for (int q = 0; q < 3; ++q) e[1][q] = e[0][q];
            e[1][perms[p][1]] = 1;
            for (int q = 0; q < 3; ++q) e[2][q] = 1;
            const int det = e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) -
                            e[0][1] * (e[1][0] * e[2][2] - e[1][2] * e[2][0]) +
                            e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
            off[p][0] = 0;
            for (int v = 0; v < 3; ++v) off[p][v + 1] = e[v][0] * stride[0] + e[v][1] * stride[1] + e[v][2] * stride[2];
            if (det < 0) std::swap(off[p][2], off[p][3]);
        }
        for (int64_t k = 0; k < n; ++k)
            for (int64_t j = 0; j < n; ++j)
                for (int64_t i = 0; i < n; ++i) {
                    const int64_t v = (k * w + j) * w + i, cube = (k * n + j) * n + i;
                    for (int p = 0; p < 6; ++p)
                        for (int q = 0; q < 4; ++q) C[(cube * 6 + p) * 4 + q] = (int32_t)(v + off[p][q]);
                }
    }
    *coords = X;
    *cells = C;
    *n_nodes = nn;
    *n_cells = nc;
    return BIOT_OK;
}

biot_status biot_bc_column(const biot_mesh *mesh, double load, uint8_t *dirichlet, double *F, int64_t *n_facets,
                           int32_t *facets) {
    if (!mesh || !n_facets || !mesh->coords || !mesh->cells) return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    const int d = mesh->dim, nc = d + 1;
    if (d != 2 && d != 3) return fail(nullptr, BIOT_E_INVALID, "mesh.dim must be 2 or 3");
    if (!std::isfinite(load)) return fail(nullptr, BIOT_E_INVALID, "load must be finite");
    const double eps = 1e-12;
    const int64_t N = mesh->n_nodes;
    auto on_top = [&](int64_t v) { return mesh->coords[v * d + (d - 1)] > 1.0 - eps; };
    if (dirichlet) {
        for (int64_t v = 0; v < N; ++v) {
            const double *x = mesh->coords + v * d;
            uint8_t *m = dirichlet + v * nc;
            for (int c = 0; c < nc; ++c) m[c] = 0;
            for (int ax = 0; ax < d - 1; ++ax)
                if (x[ax] < eps || x[ax] > 1.0 - eps) m[ax] = 1;   // rollers on the sides
            if (x[d - 1] < eps)
                for (int c = 0; c < d; ++c) m[c] = 1;               // fixed bottom
            if (x[d - 1] > 1.0 - eps) m[d] = 1;                     // drained top
        }
    }
    if (F)
        for (int64_t q = 0; q < N * nc; ++q) F[q] = 0.0;
    int64_t nf = 0;
    for (int64_t e = 0; e < mesh->n_cells; ++e) {
        const int32_t *cv = mesh->cells + e * nc;
        int32_t f[3];
        int cnt = 0;
        for (int a = 0; a < nc; ++a) {
            if (cv[a] < 0 || cv[a] >= N) return fail(nullptr, BIOT_E_INVALID, "cell references a node out of range");
            if (on_top(cv[a]) && cnt < 3) f[cnt++] = cv[a];
            else if (on_top(cv[a])) ++cnt;
        }
        if (cnt != d) continue;   // a facet on the top face: exactly d of the cell's vertices on it
        if (facets)
            for (int a = 0; a < d; ++a) facets[nf * d + a] = f[a];
        if (F) {
            const double *P0 = mesh->coords + (int64_t)f[0] * d, *P1 = mesh->coords + (int64_t)f[1] * d;
            double meas;
            if (d == 2) {
                meas = std::hypot(P1[0] - P0[0], P1[1] - P0[1]);
            } else {
                const double *P2 = mesh->coords + (int64_t)f[2] * d;
                const double u[3] = {P1[0] - P0[0], P1[1] - P0[1], P1[2] - P0[2]};
                const double v[3] = {P2[0] - P0[0], P2[1] - P0[1], P2[2] - P0[2]};
                const double cx = u[1] * v[2] - u[2] * v[1], cy = u[2] * v[0] - u[0] * v[2],
                             cz = u[0] * v[1] - u[1] * v[0];
                meas = 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
            }
            for (int a = 0; a < d; ++a) F[(int64_t)f[a] * nc + (d - 1)] += -load * meas / d;
        }
        ++nf;
    }
    *n_facets = nf;
    return BIOT_OK;
}

const char *biot_status_string(biot_status s) {
    switch (s) {
        case BIOT_OK: return "ok";
        case BIOT_E_INVALID: return "invalid argument";
        case BIOT_E_NOMEM: return "out of memory";
        case BIOT_E_CUDA: return "CUDA error";
        case BIOT_E_NCCL: return "NCCL error";
        case BIOT_E_STATE: return "invalid state";
        case BIOT_E_NONFINITE: return "non-finite residual";
    }
    return "unknown status";
}

const char *biot_last_error(const biot_ctx *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

biot_status biot_nccl_unique_id(void *out) {
    if (!out) return fail(nullptr, BIOT_E_INVALID, "out is NULL");
    NcclApi *api = nccl();
    if (!api) return fail(nullptr, BIOT_E_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    ncclResult_t r = api->GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, BIOT_E_NCCL, "ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof(id));
    return BIOT_OK;
}

biot_status biot_assemble_loads_host(const biot_mesh *mesh, const biot_material *mat, const biot_bc *bc,
                                     double dt, int32_t *n_terms, double *F, int32_t *kinds, int32_t *src) {
    if (!mesh || !mat || !bc || !n_terms) return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    biot::HostOperator op;
    std::string m = biot::assemble(*mesh, *mat, *bc, dt, op);
    if (!m.empty()) return fail(nullptr, BIOT_E_INVALID, m);
    *n_terms = (int32_t)op.extra.size();
    for (size_t j = 0; j < op.extra.size(); ++j) {
        if (F) std::memcpy(F + j * op.extra[j].f.size(), op.extra[j].f.data(), op.extra[j].f.size() * sizeof(double));
        if (kinds) kinds[j] = op.extra[j].kind;
        if (src) src[j] = op.extra[j].src;
    }
    return BIOT_OK;
}

biot_status biot_assemble_host(const biot_mesh *mesh, const biot_material *mat, const biot_bc *bc,
                               double dt, int64_t *nnz_AA, int64_t *AA_i, int64_t *AA_j,
                               double *AA_v, int64_t *nnz_AP, int64_t *AP_i, int64_t *AP_j,
                               double *AP_v, double *f, double *dinv) {
    if (!mesh || !mat || !bc || !nnz_AA || !nnz_AP)
        return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    biot::HostOperator op;
    std::string m = biot::assemble(*mesh, *mat, *bc, dt, op);
    if (!m.empty()) return fail(nullptr, BIOT_E_INVALID, m);
    *nnz_AA = op.nnz_AA;
    *nnz_AP = op.nnz_AP;
    const int nc = op.nc, d = op.d, S = op.n_slots, W = biot::block_width(nc);
    if (AA_i && AA_j && AA_v && AP_i && AP_j && AP_v) {
        int64_t ka = 0, kp = 0;
        for (int64_t i = 0; i < op.n_nodes; ++i)
            for (int s = 0; s < S; ++s) {
                int64_t j = op.path == biot::PATH_BDIA ? i + op.offsets[s] : op.cols[(size_t)i * S + s];
                if (j < 0 || j >= op.n_nodes) continue;
                if (op.path == biot::PATH_BDIA) {   // skip duplicate padding slots
                    bool dup = false;
                    for (int s2 = 0; s2 < s; ++s2) dup |= (op.offsets[s2] == op.offsets[s]);
                    if (dup) continue;
                } else {
                    bool dup = false;
                    for (int s2 = 0; s2 < s; ++s2) dup |= (op.cols[(size_t)i * S + s2] == j);
                    if (dup) continue;
                }
                const double *b = op.blk.data() + ((size_t)i * S + s) * W;
                for (int c = 0; c < nc; ++c)
                    for (int cc = 0; cc < nc; ++cc)
                        if (b[c * nc + cc] != 0.0) {
                            AA_i[ka] = i * nc + c;
                            AA_j[ka] = j * nc + cc;
                            AA_v[ka] = b[c * nc + cc];
                            ka++;
                        }
                for (int cc = 0; cc < d; ++cc)
                    if (b[d * nc + cc] != 0.0) {
                        AP_i[kp] = i * nc + d;
                        AP_j[kp] = j * nc + cc;
                        AP_v[kp] = b[d * nc + cc];
                        kp++;
                    }
                if (b[nc * nc] != 0.0) {
                    AP_i[kp] = i * nc + d;
                    AP_j[kp] = j * nc + d;
                    AP_v[kp] = b[nc * nc];
                    kp++;
                }
            }
    }
    if (f) std::memcpy(f, op.load.data(), op.load.size() * sizeof(double));
    if (dinv) std::memcpy(dinv, op.dinv.data(), op.dinv.size() * sizeof(double));
    return BIOT_OK;
}

biot_status biot_setup(const biot_mesh *mesh, const biot_material *mat, const biot_bc *bc, double dt,
                       int32_t n_t, const biot_opts *opts, biot_ctx **out) {
    if (!out) return fail(nullptr, BIOT_E_INVALID, "out is NULL");
    *out = nullptr;
    if (!mesh || !mat || !bc || !opts) return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    if (n_t < 1) return fail(nullptr, BIOT_E_INVALID, "n_t must be >= 1");
    if (opts->precond != 1 && opts->precond != 2)
        return fail(nullptr, BIOT_E_INVALID, "precond must be 1 (P~1) or 2 (P~2)");
    if (!(opts->omega > 0.0) || !std::isfinite(opts->omega))
        return fail(nullptr, BIOT_E_INVALID, "omega must be > 0");
    if (opts->world < 1 || opts->rank < 0 || opts->rank >= opts->world)
        return fail(nullptr, BIOT_E_INVALID, "need 0 <= rank < world");
    const bool sweep_slabs = opts->world > 1 && (opts->flags & BIOT_FLAG_SWEEP_SLABS);
    if (n_t % opts->world != 0 && !sweep_slabs)
        return fail(nullptr, BIOT_E_INVALID, "n_t must be divisible by world (time slabs)");
    if (opts->world > 1 && !(opts->flags & BIOT_FLAG_MANUAL_HALO) && !opts->nccl_id)
        return fail(nullptr, BIOT_E_INVALID, "world > 1 needs nccl_id (or BIOT_FLAG_MANUAL_HALO)");
    if (opts->history < 0) return fail(nullptr, BIOT_E_INVALID, "history must be >= 0");
    if (bc->load_scale)
        for (int32_t n = 0; n < n_t; ++n)
            if (!std::isfinite(bc->load_scale[n]))
                return fail(nullptr, BIOT_E_INVALID, "load_scale must be finite");

    if (bc->n_sources > 0)
        for (int64_t k = 0; k < (int64_t)bc->n_sources * n_t; ++k)
            if (!std::isfinite(bc->source_coef[k])) return fail(nullptr, BIOT_E_INVALID, "source_coef must be finite");
    if (bc->dirichlet_coef)
        for (int32_t n = 0; n <= n_t; ++n)
            if (!std::isfinite(bc->dirichlet_coef[n]))
                return fail(nullptr, BIOT_E_INVALID, "dirichlet_coef must be finite");

    auto op = std::make_unique<biot::HostOperator>();
    std::string m = biot::assemble(*mesh, *mat, *bc, dt, *op);
    if (!m.empty()) return fail(nullptr, BIOT_E_INVALID, m);

    // load terms f_n = sum_j coef_j(n) F_j (R16, R24): the traction term (unless it is zero
    // and others exist), then the sources and the Dirichlet lifting; term 0 travels in the
    // per-node records, the rest in loadx
    std::vector<std::vector<double>> lterm_f, lterm_c;   // [term][N*nc], [term][n_t]
    int trac_term = -1;
    {
        bool trac_nz = false;
        for (double v : op->load) trac_nz |= (v != 0.0);
        if (trac_nz || op->extra.empty()) {
            trac_term = 0;
            lterm_f.push_back(op->load);
            std::vector<double> c(n_t);
            for (int32_t n = 0; n < n_t; ++n) c[n] = bc->load_scale ? bc->load_scale[n] : 1.0;
            lterm_c.push_back(std::move(c));
        }
        for (auto &t : op->extra) {
            std::vector<double> c(n_t);
            for (int32_t n = 1; n <= n_t; ++n) {
                if (t.kind == 0) c[n - 1] = bc->source_coef[(size_t)t.src * n_t + (n - 1)];
                else if (t.kind == 1) c[n - 1] = bc->dirichlet_coef ? bc->dirichlet_coef[n] : 1.0;
                else c[n - 1] = bc->dirichlet_coef ? bc->dirichlet_coef[n - 1] : 1.0;
            }
            lterm_f.push_back(t.f);
            lterm_c.push_back(std::move(c));
        }
        if ((int)lterm_f.size() > biot::kMaxLoads)
            return fail(nullptr, BIOT_E_INVALID, "at most " + std::to_string(biot::kMaxLoads) +
                                                     " nonzero load terms (traction, sources, Dirichlet lifting)");
        op->load = lterm_f[0];
    }

    std::unique_ptr<biot_ctx> holder(new biot_ctx());
    biot_ctx *ctx = holder.get();
    // any early return below releases what was acquired so far
    struct Guard {
        std::unique_ptr<biot_ctx> &h;
        bool armed = true;
        ~Guard() { if (armed && h) free_all(h.get()); }
    } guard{holder};
    ctx->device = opts->device;
    CU(cudaSetDevice(ctx->device));
    int cc_major = 0;
    CU(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, ctx->device));
    if (cc_major != 10)
        return fail(ctx, BIOT_E_CUDA, "this build targets sm_100a (B200); device has CC major " +
                                          std::to_string(cc_major));
    ctx->d = op->d;
    ctx->nc = op->nc;
    ctx->N = op->n_nodes;
    ctx->S = op->n_slots;
    ctx->path = op->path;
    ctx->offsets = op->offsets;
    ctx->pad = op->path == biot::PATH_BDIA ? op->max_abs_offset : 0;
    ctx->n_t = n_t;
    ctx->rank = opts->rank;
    ctx->world = opts->world;
    ctx->sweep_mode = sweep_slabs;
    ctx->n_tl = sweep_slabs ? n_t : n_t / opts->world;            // sweep partition: every rank holds all steps
    ctx->first_step = sweep_slabs ? 1 : ctx->rank * ctx->n_tl + 1;
    ctx->flags = opts->flags;
    ctx->precond = opts->precond;
    ctx->omega = opts->omega;
    ctx->n_load = (int)lterm_f.size();
    ctx->trac_term = trac_term;
    ctx->beta = op->beta;
    ctx->nnz_AA = op->nnz_AA;
    ctx->nnz_AP = op->nnz_AP;
    {
        // Gershgorin bounds of the diagonally scaled inner blocks (R22): max over free rows of
        // sum_j |M_ij| / M_ii, M = A (displacement rows) or S~p = -AA_pp (pressure rows)
        const int ncc = op->nc, dd = op->d, WB = biot::block_width(ncc);
        double lu = 0.0, lp = 0.0;
        for (int64_t i = 0; i < op->n_nodes; ++i)
            for (int c = 0; c < ncc; ++c) {
                const double dv = op->dinv[(size_t)i * ncc + c];
                if (dv == 0.0) continue;
                double sum = 0.0;
                for (int sl = 0; sl < op->n_slots; ++sl) {
                    const double *b = op->blk.data() + ((size_t)i * op->n_slots + sl) * WB;
                    if (c < dd)
                        for (int cc = 0; cc < dd; ++cc) sum += std::fabs(b[c * ncc + cc]);
                    else
                        sum += std::fabs(b[dd * ncc + dd]);
                }
                if (c < dd) lu = std::max(lu, sum * std::fabs(dv));
                else lp = std::max(lp, sum * std::fabs(dv));
            }
        ctx->lmax_u = lu;
        ctx->lmax_p = lp;
    }
    ctx->hist_cap = opts->history > 0 ? opts->history : 1024;
    ctx->pitch = ((int64_t)ctx->n_tl + biot::kChunk - 1) / biot::kChunk * biot::kChunk;
    ctx->node_block = 8;
    std::vector<double> cls3, cls2;   // tile3d / tile2d class stencils (host)
    {
        const char *kenv = std::getenv("BIOT_KERNEL");
        const bool force_generic = kenv && std::string(kenv) == "generic";
        ctx->stencil = detect_stencil(ctx);
        if (const char *e = std::getenv("BIOT_MARCH_T")) ctx->mT = std::atoi(e);
        std::string want = kenv ? std::string(kenv) : std::string();
        if (force_generic || !ctx->stencil) {
            ctx->kern = 1;
        } else if (ctx->d == 2) {
            ctx->row_w = -ctx->gbase[0];              // W
            ctx->n_rows = (int32_t)(ctx->N / ctx->row_w);
            const std::vector<int64_t> order = {0, -ctx->row_w - 1, -ctx->row_w, -1, 1, ctx->row_w, ctx->row_w + 1};
            const bool grid_ok = ctx->row_w * ctx->n_rows == ctx->N;
            if (!grid_ok) ctx->kern = 1;
            else if (want == "march") ctx->kern = (ctx->mT == 2 || ctx->mT == 4) ? 3 : 1;
            else ctx->kern = (ctx->offsets == order && tile2d_classes(*op, ctx->row_w, ctx->n_rows, cls2)) ? 4 : 3;
        } else {
            // 3D: structured n1^3 Kuhn cube in the slot order tile3d_kernels.cu walks
            const int64_t W = ctx->gbase[4], V = W * W;
            const std::vector<int64_t> order = {0, -V - W - 1, -V - W, -V - 1, -V, -W - 1, -W, -1,
                                                1, W, W + 1, V, V + 1, V + W, V + W + 1};
            if (W * V == ctx->N && ctx->offsets == order && want != "march" && W >= biot::tile3d_min_n1() &&
                tile3d_classes(*op, W, cls3)) {
                ctx->kern = 6;
                ctx->n1 = (int32_t)W;
            } else {
                ctx->kern = 1;
            }
        }
    }
    if (ctx->n_load > 1 && ctx->kern != 1 && ctx->kern != 4) ctx->kern = 1;   // kMaxLoads kernels: generic, tile2d
    if (ctx->kern == 4) {
        // the fused P~1 tile reads x two grid rows above its first row (panel padding), and
        // P~1 runs in one pass unless BIOT_P1_TWOPASS=1 (the two-pass form, kept for comparison)
        ctx->pad = std::max<int64_t>(ctx->pad, 2 * ctx->row_w + 2);
        const char *tp = std::getenv("BIOT_P1_TWOPASS");
        ctx->p1_fused = ctx->precond == 1 && !(tp && std::atoi(tp) == 1);
    }
    {
        // overlapped halo for the tile kernels' Jacobi sweep: NCCL exchange on a comm stream;
        // ranks > 0 defer their first local step (also forced with MANUAL_HALO for tests).
        // The step-0 kernels exist for P~2 and the fused 2D / two-pass 3D P~1.
        const bool tile = ctx->kern == 4 || ctx->kern == 6;
        const bool s0ok = ctx->precond == 2 || (ctx->kern == 4 ? ctx->p1_fused : true);
        const char *no = std::getenv("BIOT_NO_OVERLAP");
        const bool allow = tile && s0ok && !(no && std::atoi(no) == 1) && opts->world > 1 && !sweep_slabs;
        ctx->overlap = allow && !(opts->flags & BIOT_FLAG_MANUAL_HALO);
        ctx->defer0 = allow && opts->rank > 0 &&
                      (ctx->overlap || (opts->flags & BIOT_FLAG_DEFER_STEP0));
    }
    const int64_t chunk = ctx->kern == 3 ? 32 * ctx->mT
                        : ctx->kern == 4 ? biot::tile2d_chunk()
                        : ctx->kern == 6 ? biot::tile3d_chunk()
                                         : biot::kChunk;
    const int64_t nchunks = (ctx->n_tl + chunk - 1) / chunk;
    ctx->tw = 1;
    while (ctx->tw < 8 && ctx->tw < nchunks) ctx->tw *= 2;
    ctx->n_alloc = (ctx->N + 7) / 8 * 8;

    if (opts->stream) {
        ctx->stream = (cudaStream_t)opts->stream;
    } else {
        CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    CU(cudaEventCreate(&ctx->ev_a));
    CU(cudaEventCreate(&ctx->ev_b));
    ALLOC(ctx->d_iter, sizeof(int64_t));
    ctx->use_graph = !(opts->flags & BIOT_FLAG_NO_GRAPH) && (opts->world == 1 || (opts->flags & BIOT_FLAG_MANUAL_HALO)) &&
                     !(opts->flags & BIOT_FLAG_DEFER_STEP0);
    if (const char *e = std::getenv("BIOT_NCCL_TIMEOUT_S")) ctx->nccl_timeout_s = std::max(1.0, std::atof(e));

    const int nc = ctx->nc;
    const int W = biot::block_width(nc);
    // nodes: [pad | N | pad + 8]; the blocked kernel may touch up to 7 dummy rows past N
    ctx->rows_alloc = (ctx->N + 2 * ctx->pad + 8) * nc;
    const size_t panel_bytes = (size_t)ctx->rows_alloc * ctx->pitch * sizeof(double);
    for (int k = 0; k < 2; ++k) {
        ALLOC(ctx->xbase[k], panel_bytes);
        CU(cudaMemsetAsync(ctx->xbase[k], 0, panel_bytes, ctx->stream));
        ctx->x[k] = ctx->xbase[k] + ctx->pad * nc * ctx->pitch;
    }
    if (ctx->precond == 1 && !ctx->p1_fused) {   // the Z panel of the two-pass P~1
        ALLOC(ctx->zbase, panel_bytes);
        CU(cudaMemsetAsync(ctx->zbase, 0, panel_bytes, ctx->stream));
        ctx->z = ctx->zbase + ctx->pad * nc * ctx->pitch;
    }
    const size_t vec_bytes = (size_t)ctx->N * nc * sizeof(double);
    ALLOC(ctx->ghost_base, (size_t)ctx->rows_alloc * sizeof(double));
    CU(cudaMemsetAsync(ctx->ghost_base, 0, (size_t)ctx->rows_alloc * sizeof(double), ctx->stream));
    ctx->ghost = ctx->ghost_base + ctx->pad * nc;
    if (bc->x_initial && (ctx->rank == 0 || ctx->sweep_mode)) {
        std::vector<double> x0(bc->x_initial, bc->x_initial + (size_t)ctx->N * nc);
        for (size_t q = 0; q < x0.size(); ++q)
            if (op->fixed[q]) x0[q] = 0.0;
        for (double v : x0) ctx->x0_zero = ctx->x0_zero && v == 0.0;
        CU(h2d(ctx, ctx->ghost, x0.data(), vec_bytes));
    }
    // operator arrays padded to n_alloc nodes with zeros (dummy rows of the blocked kernel)
    const size_t blk_bytes = (size_t)ctx->n_alloc * ctx->S * W * sizeof(double);
    ALLOC(ctx->blk, blk_bytes);
    CU(cudaMemsetAsync(ctx->blk, 0, blk_bytes, ctx->stream));
    CU(h2d(ctx, ctx->blk, op->blk.data(), op->blk.size() * sizeof(double)));
    if (ctx->path == biot::PATH_ELL) {
        ALLOC(ctx->cols, op->cols.size() * sizeof(int32_t));
        CU(h2d(ctx, ctx->cols, op->cols.data(), op->cols.size() * sizeof(int32_t)));
    }
    const size_t vec_alloc = (size_t)ctx->n_alloc * nc * sizeof(double);
    ALLOC(ctx->load, vec_alloc);
    CU(cudaMemsetAsync(ctx->load, 0, vec_alloc, ctx->stream));
    CU(h2d(ctx, ctx->load, op->load.data(), vec_bytes));
    ALLOC(ctx->dinv, vec_alloc);
    CU(cudaMemsetAsync(ctx->dinv, 0, vec_alloc, ctx->stream));
    CU(h2d(ctx, ctx->dinv, op->dinv.data(), vec_bytes));
    ALLOC(ctx->fixed, (size_t)ctx->N * nc);
    CU(h2d(ctx, ctx->fixed, op->fixed.data(), (size_t)ctx->N * nc));
    {
        // one row per load term (the kMaxLoads kernels read them all: unused rows are zero),
        // zero past n_tl (window reads may overrun)
        ctx->s_pitch = ctx->pitch + 128;
        const int rows = ctx->n_load > 1 ? biot::kMaxLoads : 1;
        std::vector<double> sl((size_t)rows * ctx->s_pitch, 0.0);
        for (int j = 0; j < ctx->n_load; ++j)
            for (int32_t t = 0; t < ctx->n_tl; ++t)
                sl[(size_t)j * ctx->s_pitch + t] = lterm_c[j][ctx->first_step - 1 + t];
        ALLOC(ctx->s, sl.size() * sizeof(double));
        CU(h2d(ctx, ctx->s, sl.data(), sl.size() * sizeof(double)));
        if (ctx->n_load > 1) {
            // load vectors of terms 1..kMaxLoads-1; unused terms are zero vectors
            std::vector<double> lx((size_t)(biot::kMaxLoads - 1) * ctx->N * nc, 0.0);
            for (int j = 1; j < ctx->n_load; ++j)
                std::copy(lterm_f[j].begin(), lterm_f[j].end(), lx.begin() + (size_t)(j - 1) * ctx->N * nc);
            ALLOC(ctx->loadx, lx.size() * sizeof(double));
            CU(h2d(ctx, ctx->loadx, lx.data(), lx.size() * sizeof(double)));
        }
    }
    ALLOC(ctx->sendbuf, vec_bytes);
    CU(cudaMemsetAsync(ctx->sendbuf, 0, vec_bytes, ctx->stream));
    ctx->send_w = ctx->sendbuf;
    if (ctx->sweep_mode) {
        ALLOC(ctx->sweep_in, vec_bytes);
        CU(cudaMemsetAsync(ctx->sweep_in, 0, vec_bytes, ctx->stream));
    }
    if (ctx->overlap) {
        ALLOC(ctx->sendbuf2, vec_bytes);
        CU(cudaMemsetAsync(ctx->sendbuf2, 0, vec_bytes, ctx->stream));
        CU(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&ctx->ev_comm, cudaEventDisableTiming));
        CU(cudaEventRecord(ctx->ev_comm, ctx->stream));
    }
    if (ctx->defer0) {
        ALLOC(ctx->zero_ghost_base, (size_t)ctx->rows_alloc * sizeof(double));
        CU(cudaMemsetAsync(ctx->zero_ghost_base, 0, (size_t)ctx->rows_alloc * sizeof(double), ctx->stream));
        ctx->zero_ghost = ctx->zero_ghost_base + ctx->pad * nc;
        ALLOC(ctx->s0buf, (size_t)ctx->N * 8 * sizeof(double));
        CU(cudaMemsetAsync(ctx->s0buf, 0, (size_t)ctx->N * 8 * sizeof(double), ctx->stream));
        ctx->step0_blocks = ctx->kern == 4 ? biot::tile2d_step0_blocks(ctx->N) : biot::tile3d_step0_blocks(ctx->N);
        ALLOC(ctx->part0, (size_t)ctx->step0_blocks * sizeof(double));   // step-0 p-norm partials
    }

    const int nwp = 8 / ctx->tw;
    ctx->shape.smem = (size_t)nwp * (nchunks * chunk) * 2 * sizeof(double);
    if (ctx->kern == 3) {
        CU(biot::march_shape(ctx->mT, ctx->device, &ctx->shape));
        // rows per tile: enough tiles for ~8 waves, at least 16 rows per tile
        const int64_t n_seg = (ctx->row_w + 7) / 8;
        int64_t rpt = ctx->n_rows;
        while (rpt > 16 && n_seg * ((ctx->n_rows + rpt - 1) / rpt) * nchunks < 8 * (int64_t)ctx->shape.grid)
            rpt = (rpt + 1) / 2;
        if (const char *e = std::getenv("BIOT_MARCH_ROWS")) rpt = std::max(1, std::atoi(e));
        ctx->rows_per_tile = (int32_t)rpt;
        biot::SweepArgs tmp = sweep_args(ctx, biot::MODE_RESIDUAL, nullptr, nullptr);
        ctx->groups = biot::march_groups(tmp);
    } else if (ctx->kern == 4) {
        CU(biot::tile2d_shape(ctx->device, &ctx->shape));
        reserve_comm_sms(ctx);
        // row blocks: n_rblk balanced blocks (sizes floor / ceil of n_rows / n_rblk, at most
        // the kernel's row capacity), chosen to minimise the rows streamed per CTA -- every
        // block reads its two halo rows again (mostly from HBM: measured) -- plus
        // half the excess of the busiest CTA (the last round of tiles)
        const int64_t n_seg = (ctx->row_w + biot::tile2d_seg() - 1) / biot::tile2d_seg();
        const int64_t cap = biot::tile2d_max_rows(), G = ctx->shape.grid;
        int64_t nrb = (ctx->n_rows + cap - 1) / cap;
        double best = 1e300;
        for (int64_t nb = (ctx->n_rows + cap - 1) / cap; nb <= ctx->n_rows; ++nb) {
            const int64_t tiles = n_seg * nb, rounds = (tiles + G - 1) / G;
            const double avg = (double)n_seg * (double)(ctx->n_rows + 2 * nb) / (double)G;
            const double crit = (double)rounds * (double)((ctx->n_rows + nb - 1) / nb + 2);
            const double cost = avg + 0.5 * std::max(0.0, crit - avg);
            if (cost < best - 1e-9) { best = cost; nrb = nb; }
            if (rounds > 64) break;
        }
        int64_t rpt = (ctx->n_rows + nrb - 1) / nrb;
        ctx->n_rblk = (int32_t)nrb;
        if (const char *e = std::getenv("BIOT_MARCH_ROWS")) {   // uniform blocks of this many rows
            rpt = std::max(1, std::atoi(e));
            ctx->n_rblk = 0;
        }
        if (const char *e = std::getenv("BIOT_ROW_BLOCKS")) {   // this many balanced blocks
            ctx->n_rblk = std::max(1, std::atoi(e));
            rpt = (ctx->n_rows + ctx->n_rblk - 1) / ctx->n_rblk;
        }
        if (rpt > biot::tile2d_max_rows())
            return fail(ctx, BIOT_E_INVALID, "row blocks exceed the tile kernel's row capacity");
        ctx->rows_per_tile = (int32_t)rpt;
        biot::Tile2dArgs tmp{};
        tmp.row_w = ctx->row_w;
        tmp.n_rows = ctx->n_rows;
        tmp.rows_per_tile = ctx->rows_per_tile;
        tmp.n_rblk = ctx->n_rblk;
        ctx->groups = biot::tile2d_groups(tmp, ctx->shape.grid);
        {
            // fused P~1: 10 owned columns per tile, 2 extra z_u rows and 4 extra x rows per tile
            const int64_t n_seg1 = (ctx->row_w + biot::tile2d_seg_p1() - 1) / biot::tile2d_seg_p1();
            int64_t r1 = 1;
            double best1 = 1e300;
            for (int64_t rr = 1; rr <= biot::tile2d_max_rows(); ++rr) {
                const int64_t waves = (n_seg1 * ((ctx->n_rows + rr - 1) / rr) + ctx->shape.grid - 1) / ctx->shape.grid;
                const double cost = (double)waves * ((double)std::min<int64_t>(rr, ctx->n_rows) + 2.5);
                if (cost < best1 - 1e-9) { best1 = cost; r1 = rr; }
            }
            if (const char *e = std::getenv("BIOT_P1_ROWS")) r1 = std::max(1, std::min(biot::tile2d_max_rows(), std::atoi(e)));
            ctx->rows_per_tile_p1 = (int32_t)r1;
            tmp.rows_per_tile = ctx->rows_per_tile_p1;
            tmp.mode = biot::MODE_P1_FUSED;
            ctx->groups_p1 = biot::tile2d_groups(tmp, ctx->shape.grid);
        }
        // interior template + per-node aux records
        const int S = 7, WB = 10, KA = ctx->n_load > 1 ? biot::Tile2dArgs::kAuxML : biot::Tile2dArgs::kAux;
        const int64_t tnode = (int64_t)(ctx->n_rows / 2) * ctx->row_w + ctx->row_w / 2;
        const double *tb = op->blk.data() + (size_t)tnode * S * WB;
        for (int q = 0; q < S; ++q)
            for (int k = 0; k < WB; ++k) ctx->tmpl[q][k] = tb[q * WB + k];
        // structural zeros the kernel skips (must match tmpl_zero in tile2d_kernels.cu)
        auto tz = [](int q, int e, bool z0) {
            return (q == 0) ? (e == 2 || e == 5 || e == 6 || e == 7)
                            : (q == 1 || q == 6) ? (e == 0 || e == 4 || (z0 && (e == 8 || e == 9))) : false;
        };
        bool base_ok = true;
        for (int q = 0; q < S; ++q)
            for (int k = 0; k < WB; ++k)
                if (k != 8 && tz(q, k, false) && ctx->tmpl[q][k] != 0.0) base_ok = false;
        const bool z0 = base_ok && ctx->tmpl[1][9] == 0.0 && ctx->tmpl[6][9] == 0.0 &&
                        ctx->tmpl[1][8] == 0.0 && ctx->tmpl[6][8] == 0.0;
        ctx->s0 = z0 ? 1 : 0;
        if (const char *e = std::getenv("BIOT_TILE_DRY")) ctx->tile_dry = std::atoi(e);
        ALLOC(ctx->cls, cls2.size() * sizeof(double));
        CU(h2d(ctx, ctx->cls, cls2.data(), cls2.size() * sizeof(double)));
        // records for every node a tile's bulk copy can touch: the last row's segment may
        // extend up to one segment past node N-1
        const int64_t aux_nodes = ctx->N + 2 * biot::tile2d_seg() + 8, aux_front = 16;   // front: halo column -1
        std::vector<double> aux((size_t)(aux_front + aux_nodes) * KA, 0.0);
        int64_t n_int = 0;
        for (int64_t i = 0; i < ctx->N; ++i) {
            const double *b = op->blk.data() + (size_t)i * S * WB;
            const bool same = base_ok && template_node(*op, i, tb, [&](int q, int k) { return tz(q, k, z0); });
            double *r = aux.data() + (size_t)(aux_front + i) * KA;
            for (int q = 0; q < S; ++q) r[q] = b[q * WB + 8];
            for (int c = 0; c < 3; ++c) {
                r[7 + c] = op->load[(size_t)i * 3 + c];
                r[10 + c] = op->dinv[(size_t)i * 3 + c];
            }
            r[13] = same ? 1.0 : 2.0;   // path flag: 1 interior template, 2 geometric-class stencil
            for (int j = 1; j < ctx->n_load; ++j)   // further load vectors (kMaxLoads kernels)
                for (int c = 0; c < 3; ++c) r[14 + 3 * (j - 1) + c] = lterm_f[j][(size_t)i * 3 + c];
            n_int += same;
        }
        ctx->n_interior = n_int;
        {
            // aux-uniform rectangle (single-load problems): the largest [m, W-1-m] x [m, n_rows-1-m]
            // (m = 1, 2) whose nodes all carry the template node's record, up to pp entries that
            // are 0 against a fixed pressure column (they multiply x = 0 there)
            const double *R = aux.data() + (size_t)(aux_front + tnode) * KA;
            auto uniform = [&](int64_t i) {
                const double *r = aux.data() + (size_t)(aux_front + i) * KA;
                if (r[13] != 1.0) return false;
                for (int k = 0; k < 14; ++k) {
                    if (r[k] == R[k]) continue;
                    if (k < 7 && r[k] == 0.0) {
                        const int64_t j = i + ctx->offsets[k];
                        if (j >= 0 && j < ctx->N && op->fixed[(size_t)j * 3 + 2]) continue;
                    }
                    return false;
                }
                return true;
            };
            for (int m = 1; m <= 2 && ctx->n_load == 1 && !std::getenv("BIOT_NO_AUX_SKIP"); ++m) {
                const int64_t x0 = m, x1 = ctx->row_w - 1 - m, y0 = m, y1 = ctx->n_rows - 1 - m;
                if (x1 - x0 < 2 * biot::tile2d_seg() || y1 < y0) break;
                bool ok = true;
                for (int64_t y = y0; y <= y1 && ok; ++y)
                    for (int64_t x = x0; x <= x1 && ok; ++x) ok = uniform(y * ctx->row_w + x);
                if (ok) {
                    ctx->aux_geo = 1;
                    ctx->ux0 = (int32_t)x0;
                    ctx->ux1 = (int32_t)x1;
                    ctx->uy0 = (int32_t)y0;
                    ctx->uy1 = (int32_t)y1;
                    for (int k = 0; k < biot::kAuxRecU; ++k) ctx->aux_u[k] = R[k];
                    break;
                }
            }
        }
        if (std::getenv("BIOT_DEBUG"))
            std::fprintf(stderr, "[biot] tile2d: W=%lld rows/tile=%d groups=%lld interior=%lld/%lld s0=%d\n",
                         (long long)ctx->row_w, ctx->rows_per_tile, (long long)ctx->groups, (long long)n_int,
                         (long long)ctx->N, ctx->s0);
        ALLOC(ctx->aux_base, aux.size() * sizeof(double));
        CU(h2d(ctx, ctx->aux_base, aux.data(), aux.size() * sizeof(double)));
        ctx->aux = ctx->aux_base + aux_front * KA;
        // TMA tensor maps of the two panels: {time (pitch), panel rows}
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qres;
        CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres));
        if (!fn || qres != cudaDriverEntryPointSuccess)
            return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled not available");
        auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        uint32_t box[2];
        biot::tile2d_box(box);
        for (int k = 0; k < 2; ++k) {
            cuuint64_t dims[2] = {(cuuint64_t)ctx->pitch, (cuuint64_t)ctx->rows_alloc};
            cuuint64_t strides[1] = {(cuuint64_t)ctx->pitch * sizeof(double)};
            cuuint32_t bx[2] = {box[0], box[1]};
            cuuint32_t es[2] = {1, 1};
            CUresult r = encode(&ctx->tmap[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ctx->xbase[k], dims, strides,
                                bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
            if (k == 0 && ctx->zbase) {
                r = encode(&ctx->tmapz, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ctx->zbase, dims, strides, bx, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS)
                    return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled (Z) failed: " + std::to_string((int)r));
            }
        }
    } else if (ctx->kern == 6) {
        CU(biot::tile3d_shape(ctx->device, &ctx->shape));
        reserve_comm_sms(ctx);
        // planes per tile: minimise (waves of tiles) x (planes + halo cost)
        const int64_t n1 = ctx->n1, npp = biot::tile3d_patches(n1);
        int64_t best_zr = n1;
        double best = 1e300;
        for (int64_t nzr = std::max<int64_t>(2, (n1 + biot::tile3d_max_zrows() - 1) / biot::tile3d_max_zrows());
             nzr <= 8; ++nzr) {
            const int64_t zr = (n1 + nzr - 1) / nzr;
            const int64_t waves = (npp * ((n1 + zr - 1) / zr) + ctx->shape.grid - 1) / ctx->shape.grid;
            const double cost = (double)waves * ((double)zr + 0.25);
            if (cost < best - 1e-9) { best = cost; best_zr = zr; }
        }
        if (const char *e = std::getenv("BIOT_ZROWS")) best_zr = std::max(1, std::atoi(e));
        if (best_zr > biot::tile3d_max_zrows() || best_zr >= n1)
            return fail(ctx, BIOT_E_INVALID, "BIOT_ZROWS must be < n1 and <= the tile kernel's plane capacity");
        ctx->z_rows = (int32_t)best_zr;
        biot::Tile3dArgs tmp{};
        tmp.n1 = ctx->n1;
        tmp.z_rows = ctx->z_rows;
        ctx->groups = biot::tile3d_groups(tmp);
        // interior template (centre node) + per-node aux records
        const int S = 15, WB = biot::block_width(4), KA = biot::Tile3dArgs::kAux;
        const int64_t c1 = n1 / 2, tnode = (c1 * n1 + c1) * n1 + c1;
        const double *tb = op->blk.data() + (size_t)tnode * S * WB;
        for (int q = 0; q < S; ++q)
            for (int k = 0; k < 17; ++k) ctx->tmpl3[q][k] = tb[q * WB + k];
        // structural zeros the kernel skips (must match tmpl3_zero in tile3d_kernels.cu)
        auto diag = [](int q) { return q == 1 || q == 2 || q == 3 || q == 5 || q == 10 || q == 12 || q == 13 || q == 14; };
        auto tz = [&](int q, int e, bool z0) {
            return (q == 0) ? (e == 3 || e == 7 || e == 11 || e == 12 || e == 13 || e == 14)
                            : diag(q) ? (e == 0 || e == 5 || e == 10 || (z0 && (e == 15 || e == 16))) : false;
        };
        bool base_ok = true;
        for (int q = 0; q < S; ++q)
            for (int k = 0; k < 17; ++k)
                if (k != 15 && tz(q, k, false) && ctx->tmpl3[q][k] != 0.0) base_ok = false;
        bool z0 = base_ok;
        for (int q = 0; q < S; ++q)
            if (diag(q) && (ctx->tmpl3[q][15] != 0.0 || ctx->tmpl3[q][16] != 0.0)) z0 = false;
        // the zero-storage variant needs AA_pp = 0 on the diagonal slots of every interior node
        if (z0)
            for (int64_t i = 0; i < ctx->N && z0; ++i)
                for (int q = 0; q < S; ++q)
                    if (diag(q) && op->blk[((size_t)i * S + q) * WB + 15] != 0.0 &&
                        template_node(*op, i, tb, [&](int qq, int k) { return tz(qq, k, false); })) {
                        z0 = false;
                        break;
                    }
        ctx->s0 = z0 ? 1 : 0;
        if (const char *e = std::getenv("BIOT_TILE_DRY")) ctx->tile_dry = std::atoi(e);
        std::vector<double> aux((size_t)(ctx->N + 8) * KA, 0.0);
        int64_t n_int = 0;
        for (int64_t i = 0; i < ctx->N; ++i) {
            const int64_t x = i % n1, y = (i / n1) % n1, z = i / (n1 * n1);
            const bool inner = x > 0 && y > 0 && z > 0 && x < n1 - 1 && y < n1 - 1 && z < n1 - 1;
            const bool same = base_ok && inner && template_node(*op, i, tb, [&](int q, int k) { return tz(q, k, z0); });
            const double *b = op->blk.data() + (size_t)i * S * WB;
            double *r = aux.data() + (size_t)i * KA;
            for (int q = 0; q < S; ++q) r[q] = b[q * WB + 15];
            for (int c = 0; c < 4; ++c) {
                r[15 + c] = op->load[(size_t)i * 4 + c];
                r[19 + c] = op->dinv[(size_t)i * 4 + c];
            }
            // path flag: 1 interior template, 2 geometric-class stencil
            r[23] = same ? 1.0 : 2.0;
            n_int += same;
        }
        ctx->n_interior = n_int;
        ALLOC(ctx->cls, cls3.size() * sizeof(double));
        CU(h2d(ctx, ctx->cls, cls3.data(), cls3.size() * sizeof(double)));
        if (std::getenv("BIOT_DEBUG"))
            std::fprintf(stderr, "[biot] tile3d: n1=%d z_rows=%d tiles=%lld interior=%lld/%lld s0=%d grid=%d\n",
                         ctx->n1, ctx->z_rows, (long long)ctx->groups, (long long)n_int, (long long)ctx->N, ctx->s0,
                         ctx->shape.grid);
        ALLOC(ctx->aux_base, aux.size() * sizeof(double));
        CU(h2d(ctx, ctx->aux_base, aux.data(), aux.size() * sizeof(double)));
        ctx->aux = ctx->aux_base;
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qres;
        CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres));
        if (!fn || qres != cudaDriverEntryPointSuccess)
            return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled not available");
        auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        uint32_t box[4];
        biot::tile3d_box(box);
        for (int k = 0; k < 2; ++k) {
            // {time, x*4 + c, y, z} over the panel at node 0; out-of-mesh boxes are zero-filled
            cuuint64_t dims[4] = {(cuuint64_t)ctx->pitch, (cuuint64_t)(n1 * 4), (cuuint64_t)n1, (cuuint64_t)n1};
            const cuuint64_t rb = (cuuint64_t)ctx->pitch * sizeof(double);
            cuuint64_t strides[3] = {rb, rb * (cuuint64_t)(n1 * 4), rb * (cuuint64_t)(n1 * n1 * 4)};
            cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
            cuuint32_t es[4] = {1, 1, 1, 1};
            CUresult r = encode(&ctx->tmap[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, ctx->x[k], dims, strides, bx, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled (4D) failed: " + std::to_string((int)r));
            if (k == 0 && ctx->z) {
                // the P~1 second pass stages z_u only: {time, component, x, y, z}, box of 3
                // components (r_p is read per node)
                uint32_t bz[5];
                biot::tile3d_box_z(bz);
                cuuint64_t dz[5] = {(cuuint64_t)ctx->pitch, 4, (cuuint64_t)n1, (cuuint64_t)n1, (cuuint64_t)n1};
                cuuint64_t sz[4] = {rb, rb * 4, rb * (cuuint64_t)(n1 * 4), rb * (cuuint64_t)(n1 * n1 * 4)};
                cuuint32_t bxz[5] = {bz[0], bz[1], bz[2], bz[3], bz[4]};
                cuuint32_t esz[5] = {1, 1, 1, 1, 1};
                r = encode(&ctx->tmapz, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, ctx->z, dz, sz, bxz, esz,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS)
                    return fail(ctx, BIOT_E_CUDA, "cuTensorMapEncodeTiled (5D, Z) failed: " + std::to_string((int)r));
            }
        }
    } else {
        CU(biot::sweep_shape(ctx->d, ctx->path, ctx->S, ctx->n_load > 1, ctx->device, &ctx->shape));
        ctx->groups = ctx->shape.grid;
    }
    // P~1 pass 2 uses the generic shape
    {
        biot::LaunchShape p2{0, 0};
        CU(biot::sweep_shape(ctx->d, ctx->path, ctx->S, false, ctx->device, &p2));
        ctx->pass2_grid = p2.grid;
    }
    const int64_t gmax = std::max(ctx->groups, ctx->groups_p1);
    ALLOC(ctx->partial, (size_t)gmax * ctx->n_tl * 2 * sizeof(double));
    ALLOC(ctx->fin_scratch, (size_t)std::max<int64_t>(1, biot::finalize_scratch_doubles((int)gmax, ctx->n_tl)) *
                                sizeof(double));
    ALLOC(ctx->fin_tickets, (size_t)biot::finalize_tickets(ctx->n_tl) * sizeof(int));
    CU(cudaMemsetAsync(ctx->fin_tickets, 0, (size_t)biot::finalize_tickets(ctx->n_tl) * sizeof(int), ctx->stream));
    ALLOC(ctx->hist, (size_t)ctx->hist_cap * ctx->n_tl * 2 * sizeof(double));
    ALLOC(ctx->norms, (size_t)ctx->n_tl * 2 * sizeof(double));
    ALLOC(ctx->nonfinite, sizeof(int));
    CU(cudaMemsetAsync(ctx->nonfinite, 0, sizeof(int), ctx->stream));
    ctx->staging_steps = std::max<int64_t>(1, std::min<int64_t>(ctx->n_tl, (256ll << 20) / (int64_t)vec_bytes));
    ALLOC(ctx->staging, (size_t)ctx->staging_steps * vec_bytes);

    if (ctx->world > 1 && !(ctx->flags & BIOT_FLAG_MANUAL_HALO)) {
        NcclApi *api = nccl();
        if (!api) return fail(ctx, BIOT_E_NCCL, "libnccl.so.2 could not be loaded");
        ncclUniqueId id;
        std::memcpy(&id, opts->nccl_id, sizeof(id));
        ncclResult_t r = api->CommInitRank(&ctx->comm, ctx->world, id, ctx->rank);
        if (r != ncclSuccess)
            return fail(ctx, BIOT_E_NCCL, std::string("ncclCommInitRank: ") +
                                              (api->GetErrorString ? api->GetErrorString(r) : "?"));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    guard.armed = false;
    *out = holder.release();
    return BIOT_OK;
}

biot_status biot_set_iterate(biot_ctx *ctx, int32_t n, int32_t count, const double *x) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!x || count < 0) return fail(ctx, BIOT_E_INVALID, "x is NULL or count < 0");
    if (n < ctx->first_step || n + count > ctx->first_step + ctx->n_tl)
        return fail(ctx, BIOT_E_INVALID, "steps outside the owned slab");
    CU(cudaSetDevice(ctx->device));
    const int64_t rows = ctx->N * ctx->nc;
    const size_t vb = (size_t)rows * sizeof(double);
    for (int32_t done = 0; done < count;) {
        const int32_t m = (int32_t)std::min<int64_t>(ctx->staging_steps, count - done);
        CU(cudaMemcpyAsync(ctx->staging, x + (size_t)done * rows, (size_t)m * vb, cudaMemcpyHostToDevice,
                           ctx->stream));
        const int t_first = n - ctx->first_step + done;
        scatter_steps_kernel<<<1184, 256, 0, ctx->stream>>>(ctx->staging, ctx->x[ctx->cur], ctx->fixed,
                                                            rows, ctx->pitch, t_first, m);
        CU(cudaGetLastError());
        done += m;
    }
    ctx->send_dirty = true;
    CU(cudaStreamSynchronize(ctx->stream));
    return BIOT_OK;
}

biot_status biot_set_load_scale(biot_ctx *ctx, const double *s) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!s) return fail(ctx, BIOT_E_INVALID, "s is NULL");
    if (ctx->trac_term < 0) return fail(ctx, BIOT_E_STATE, "the problem has no traction load term");
    CU(cudaSetDevice(ctx->device));
    CU(cudaMemcpyAsync(ctx->s + (size_t)ctx->trac_term * ctx->s_pitch, s + (ctx->first_step - 1),
                       (size_t)ctx->n_tl * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return BIOT_OK;
}

biot_status biot_iterate(biot_ctx *ctx, int32_t K) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (K < 0) return fail(ctx, BIOT_E_INVALID, "K must be >= 0");
    if (ctx->sweep_mode && K > 0)
        return fail(ctx, BIOT_E_STATE, "sweep partition (BIOT_FLAG_SWEEP_SLABS): use the Gauss-Seidel calls");
    if (K == 0) return BIOT_OK;
    CU(cudaSetDevice(ctx->device));
    // pairs of iterations replay the context's CUDA graph (no NCCL inside: world == 1 or
    // manual halo); an odd remainder, and every NCCL iteration, launches directly
    const int32_t pairs = ctx->use_graph ? K / 2 : 0;
    const int32_t eager = K - 2 * pairs;
    if (pairs > 0 && !ctx->gexec[ctx->cur]) {
        biot_status s = build_graph(ctx, ctx->cur);
        if (s != BIOT_OK) return s;
    }
    while ((int32_t)ctx->ev_s.size() < 2 * eager) {
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        ctx->ev_s.push_back(e);
    }
    CU(cudaEventRecord(ctx->ev_a, ctx->stream));
    // the sweep spans of up to 8 replays spread over the call are kept (each sampled replay
    // records into its own events; the others into gev, re-targeted only when the target
    // changes: a few host calls per call), so last_timing's sweep time is an average over
    // the whole call, not the final replay alone
    const int cg = ctx->cur;
    const bool sample = pairs > 0 && ctx->gnode[cg][0] && ctx->gnode[cg][1] && ctx->gnode[cg][2] && ctx->gnode[cg][3];
    const int32_t stride = std::max<int32_t>(1, (pairs + 7) / 8);
    int32_t nsamp = 0;
    if (sample) {
        const size_t need = 4 * (size_t)((pairs + stride - 1) / stride);
        while (ctx->gev_pool.size() < need) {
            cudaEvent_t e;
            CU(cudaEventCreate(&e));
            ctx->gev_pool.push_back(e);
        }
    }
    if (pairs > 0) {
        CU(biot::launch_counter(ctx->d_iter, ctx->iterations, false, ctx->stream));
        bool on_pool = ctx->gpool_set[cg];
        for (int32_t k = 0; k < pairs; ++k) {
            const bool take = sample && (pairs - 1 - k) % stride == 0;   // the last replay is always sampled
            if (take || on_pool) {
                for (int h = 0; h < 4; ++h)
                    CU(cudaGraphExecEventRecordNodeSetEvent(ctx->gexec[cg], ctx->gnode[cg][h],
                                                            take ? ctx->gev_pool[4 * nsamp + h] : ctx->gev[h]));
                on_pool = take;
            }
            CU(cudaGraphLaunch(ctx->gexec[cg], ctx->stream));
            if (take) ++nsamp;
        }
        ctx->gpool_set[cg] = on_pool;
        ctx->iterations += 2 * pairs;
    }
    for (int32_t k = 0; k < eager; ++k) {
        biot_status s = one_iteration(ctx, ctx->ev_s[2 * k], ctx->ev_s[2 * k + 1]);
        if (s != BIOT_OK) return s;
    }
    // the last overlapped exchange completes inside the call (later collectives of the
    // communicator, and the caller's reads of the ghost, are ordered after it)
    if (ctx->overlap) CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_comm, 0));
    CU(cudaEventRecord(ctx->ev_b, ctx->stream));
    {
        biot_status s = wait_done(ctx, ctx->ev_b);
        if (s != BIOT_OK) return s;
    }
    float tot = 0.f;
    CU(cudaEventElapsedTime(&tot, ctx->ev_a, ctx->ev_b));
    // preconditioner-pass time per iteration: every direct launch, and (graph) the two
    // iterations of the last replay
    double sweep_ms = 0.0;
    int spans = 0;
    for (int32_t k = 0; k < eager; ++k) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev_s[2 * k], ctx->ev_s[2 * k + 1]));
        sweep_ms += ms;
        ++spans;
    }
    for (int32_t k = 0; k < nsamp; ++k)
        for (int h = 0; h < 2; ++h) {
            float ms = 0.f;
            CU(cudaEventElapsedTime(&ms, ctx->gev_pool[4 * k + 2 * h], ctx->gev_pool[4 * k + 2 * h + 1]));
            sweep_ms += ms;
            ++spans;
        }
    if (pairs > 0 && nsamp == 0)
        for (int h = 0; h < 2; ++h) {
            float ms = 0.f;
            CU(cudaEventElapsedTime(&ms, ctx->gev[2 * h], ctx->gev[2 * h + 1]));
            sweep_ms += ms;
            ++spans;
        }
    ctx->last_ms_iter = tot / K;
    ctx->last_ms_sweep = sweep_ms / spans;
    int nf = 0;
    CU(cudaMemcpyAsync(&nf, ctx->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (nf) return fail(ctx, BIOT_E_NONFINITE, "a residual norm became non-finite");
    return BIOT_OK;
}

// Gauss-Seidel in time (Alg. 2 read literally: b^{n,m} =
// A' X^{n-1,m} + f^n), pipelined as a wavefront over the global steps: sweep u of
// step t runs in wave w = t + u - 1 and needs only wave w-1 (X^{t,u-1} and X^{t-1,u}),
// so wave w updates the window of steps max(0, w-K+1)..min(N_t-1, w) at once; each
// rank runs its part of the window.  Wave w reads panel (cur + w) % 2 and writes the
// other, so global step t's iterate of sweep u lives in panel (cur + t + u) % 2: the
// columns of odd global step are moved before and after (checkerboard).  Across
// time slabs, rank r-1 sends the slice of its last step after each wave in which it
// updated it, and rank r receives it as the ghost of the next wave (K transfers).
namespace {

bool gs_recv(const biot_ctx *c, int w) {   // this rank needs its predecessor's slice at wave w
    const int g0 = c->first_step - 1;
    return c->rank > 0 && w - g0 >= 0 && w - g0 <= c->gs_K - 1;
}
bool gs_send(const biot_ctx *c, int w) {   // rank r+1 needs this rank's last slice at wave w
    const int g1 = c->first_step - 1 + c->n_tl;
    return c->rank + 1 < c->world && w - g1 >= 0 && w - g1 <= c->gs_K - 1;
}

biot_status gs_parity_copy(biot_ctx *ctx, const double *src, double *dst, int parity) {
    copy_parity_columns_kernel<<<1184, 256, 0, ctx->stream>>>(src, dst, ctx->N * ctx->nc, ctx->pitch, ctx->n_tl,
                                                              parity);
    CU(cudaGetLastError());
    return BIOT_OK;
}

// Sweep partition (BIOT_FLAG_SWEEP_SLABS): this rank runs global sweeps u0..u1 of the K; at
// global wave W it receives step W - u0 + 1 at its sweep u0 - 1 (from rank - 1's last sweep,
// finished at wave W - 1) and finishes step W - u1 + 1 at its last sweep (sent at W + 1).
int sw_u0(const biot_ctx *c) { return (int)((int64_t)c->rank * c->gs_K / c->world) + 1; }
int sw_u1(const biot_ctx *c) { return (int)((int64_t)(c->rank + 1) * c->gs_K / c->world); }
bool sw_in(const biot_ctx *c, int W, int *t) {
    *t = W - sw_u0(c) + 1;
    return c->rank > 0 && *t >= 0 && *t < c->n_t;
}
bool sw_out(const biot_ctx *c, int W, int *t) {
    *t = W - sw_u1(c) + 1;
    return c->rank + 1 < c->world && *t >= 0 && *t < c->n_t;
}

biot_status gs_window(biot_ctx *ctx, int w, int K, int64_t kbase);

biot_status gs_run_wave(biot_ctx *ctx) {
    const int W = ctx->gs_w++;
    if (!ctx->sweep_mode) return gs_window(ctx, W, ctx->gs_K, ctx->gs_k0);
    const int u0 = sw_u0(ctx), Kg = sw_u1(ctx) - u0 + 1;
    const size_t rows = (size_t)ctx->N * ctx->nc;
    int t;
    if (sw_in(ctx, W, &t))   // X^{t, u0-1} (the predecessor's last sweep) into panel (cur + t) % 2
        CU(cudaMemcpy2DAsync(ctx->x[(ctx->cur + t) % 2] + t, ctx->pitch * sizeof(double), ctx->sweep_in, sizeof(double),
                             sizeof(double), rows, cudaMemcpyDeviceToDevice, ctx->stream));
    const int wl = W - (u0 - 1);
    if (wl >= 0 && wl < ctx->n_t + Kg - 1) {
        biot_status st = gs_window(ctx, wl, Kg, ctx->gs_k0 + (u0 - 1));
        if (st != BIOT_OK) return st;
    }
    if (sw_out(ctx, W, &t)) {   // X^{t, u1} (this rank's last sweep) for rank + 1
        CU(cudaMemcpy2DAsync(ctx->sendbuf, sizeof(double), ctx->x[(ctx->cur + t + Kg) % 2] + t,
                             ctx->pitch * sizeof(double), sizeof(double), rows, cudaMemcpyDeviceToDevice, ctx->stream));
        ctx->send_dirty = false;
    }
    return BIOT_OK;
}

// One wave of the wavefront: window of steps whose sweeps 1..K (local numbering) update at
// wave w; history slots kbase + sweep - 1.
biot_status gs_window(biot_ctx *ctx, int w, int K, int64_t kbase) {
    const int L = ctx->n_tl, g0 = ctx->first_step - 1;
    const int lo = std::max(0, w - K + 1 - g0), hi = std::min(L - 1, w - g0);
    if (lo > hi) return BIOT_OK;   // the wavefront is not in this slab
    const int r = (ctx->cur + w) % 2;
    Window win;
    win.t_off = lo & ~1;                 // 16-B aligned columns; step lo-1 (if any) is not stored
    win.t_lo = lo - win.t_off;
    win.len = hi - win.t_off + 1;
    if (win.t_off == 0) {
        win.ghost = ctx->ghost;          // x_0, or the predecessor slab's slice of this wave
        win.stride = 1;
    } else {
        win.ghost = ctx->x[r] + (win.t_off - 1);
        win.stride = ctx->pitch;
    }
    // tile kernels (2D P~2 / fused P~1, 3D): start the window two steps early (steps below lo
    // computed, not stored or counted). q(lo-1) then comes out of the march itself -- lane
    // 0's second step, in the march's FMA order, which is ghost_q's order: bitwise the same --
    // instead of lane 0 gathering the ghost column through L2 at every node of the pass
    if ((ctx->kern == 4 || ctx->kern == 6) && ctx->gs_k == 0 && win.t_off >= 2 && !std::getenv("BIOT_GS_NO_LEAD")) {
        win.t_off -= 2;
        win.t_lo = lo - win.t_off;
        win.len = hi - win.t_off + 1;
        win.ghost = ctx->x[r] + (win.t_off - 1 >= 0 ? win.t_off - 1 : 0);   // not read: ghost_zero
        win.stride = ctx->pitch;
        win.lead = true;
    }
    win.send = (ctx->world > 1 && hi == L - 1 && !ctx->sweep_mode) ? ctx->sendbuf : nullptr;
    int64_t wave_groups = ctx->groups;
    if (ctx->gs_k > 0) {   // Alg. 3 literal: a GMRES(k) cycle per step of the window
        biot_status st = gmres_cycle(ctx, ctx->gs_k, ctx->tmap[r], ctx->x[r], ctx->x[1 - r], win);
        if (st != BIOT_OK) return st;
        if (win.send)      // the slice of the slab's last step for the next slab
            CU(cudaMemcpy2DAsync(win.send, sizeof(double), ctx->x[1 - r] + (L - 1), ctx->pitch * sizeof(double),
                                 sizeof(double), (size_t)ctx->N * ctx->nc, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        const int mode = main_mode(ctx);
        CU(launch_main(ctx, mode, ctx->x[r], ctx->x[1 - r], &win));
        if (mode == biot::MODE_P1_PASS1) CU(launch_pass2_any(ctx, ctx->x[r], ctx->x[1 - r], win.send, &win));
        wave_groups = groups_of(ctx, mode);
    }
    CU(biot::launch_finalize_wave(ctx->partial, (int)wave_groups, win.len, win.t_off, lo, kbase + w - g0,
                                  ctx->hist_cap, L, ctx->hist, ctx->nonfinite, ctx->fin_scratch, ctx->stream));
    if (win.send) ctx->send_dirty = false;
    return BIOT_OK;
}

}  // namespace

biot_status biot_gs_begin_gmres(biot_ctx *ctx, int32_t K, int32_t k) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (k > 0) {
        biot_status st = gmres_check(ctx, K, k);
        if (st != BIOT_OK) return st;
        CU(cudaSetDevice(ctx->device));
        if ((st = gmres_alloc(ctx, k)) != BIOT_OK) return st;
    }
    if (K < 1) return fail(ctx, BIOT_E_INVALID, "K must be >= 1");
    if (ctx->kern != 4 && ctx->kern != 6)
        return fail(ctx, BIOT_E_STATE, "Gauss-Seidel in time needs a tile kernel (structured 2D / 3D mesh)");
    if (ctx->gs_K) return fail(ctx, BIOT_E_STATE, "a Gauss-Seidel run is already open");
    if (ctx->sweep_mode && K < ctx->world)
        return fail(ctx, BIOT_E_INVALID, "sweep partition: K must be >= world (at least one sweep per rank)");
    CU(cudaSetDevice(ctx->device));
    ctx->gs_K = K;
    ctx->gs_k = k;
    ctx->gs_w = 0;
    ctx->gs_k0 = ctx->iterations;
    ctx->send_dirty = true;
    CU(cudaEventRecord(ctx->ev_a, ctx->stream));
    // global step g0 + t starts in panel (cur + g0 + t) % 2
    return gs_parity_copy(ctx, ctx->x[ctx->cur], ctx->x[1 - ctx->cur], (ctx->first_step - 1) % 2 == 0 ? 1 : 0);
}

biot_status biot_gs_begin(biot_ctx *ctx, int32_t K) { return biot_gs_begin_gmres(ctx, K, 0); }

biot_status biot_gs_waves(const biot_ctx *ctx, int32_t *out) {
    if (!ctx || !out) return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    *out = ctx->n_t + ctx->gs_K - 1;
    return BIOT_OK;
}

biot_status biot_gs_wave(biot_ctx *ctx) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!ctx->gs_K) return fail(ctx, BIOT_E_STATE, "no Gauss-Seidel run open (biot_gs_begin)");
    if (ctx->gs_w >= ctx->n_t + ctx->gs_K - 1) return fail(ctx, BIOT_E_STATE, "all waves of the run are done");
    CU(cudaSetDevice(ctx->device));
    return gs_run_wave(ctx);
}

biot_status biot_gs_end(biot_ctx *ctx) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!ctx->gs_K) return fail(ctx, BIOT_E_STATE, "no Gauss-Seidel run open (biot_gs_begin)");
    if (ctx->gs_w != ctx->n_t + ctx->gs_K - 1) return fail(ctx, BIOT_E_STATE, "waves of the run still pending");
    CU(cudaSetDevice(ctx->device));
    const int K = ctx->gs_K;
    // global step g0 + t ends in panel (cur + g0 + t + K) % 2 (sweep partition: this rank's
    // K_g sweeps): gather it into cur'
    const int Kl = ctx->sweep_mode ? sw_u1(ctx) - sw_u0(ctx) + 1 : K;
    ctx->cur = (ctx->cur + Kl + ctx->first_step - 1) % 2;
    biot_status st = gs_parity_copy(ctx, ctx->x[1 - ctx->cur], ctx->x[ctx->cur], 1);
    if (st != BIOT_OK) return st;
    CU(cudaEventRecord(ctx->ev_b, ctx->stream));
    {
        biot_status ws = wait_done(ctx, ctx->ev_b);
        if (ws != BIOT_OK) return ws;
    }
    float tot = 0.f;
    CU(cudaEventElapsedTime(&tot, ctx->ev_a, ctx->ev_b));
    ctx->last_ms_iter = tot / K;
    ctx->last_ms_sweep = tot / K;
    ctx->iterations += K;
    ctx->gs_K = 0;
    ctx->gs_k = 0;
    ctx->send_dirty = true;
    int nf = 0;
    CU(cudaMemcpyAsync(&nf, ctx->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (nf) return fail(ctx, BIOT_E_NONFINITE, "a residual norm became non-finite");
    return BIOT_OK;
}

static biot_status iterate_gs_sweeps(biot_ctx *ctx, int32_t K, int32_t k);

biot_status biot_iterate_gs_gmres(biot_ctx *ctx, int32_t K, int32_t k) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (K < 0) return fail(ctx, BIOT_E_INVALID, "K must be >= 0");
    if (K == 0) return BIOT_OK;
    if (ctx->world > 1 && (ctx->flags & BIOT_FLAG_MANUAL_HALO))
        return fail(ctx, BIOT_E_STATE, "manual halo: drive the waves with biot_gs_begin/wave/end");
    if (ctx->sweep_mode) return iterate_gs_sweeps(ctx, K, k);
    NcclApi *api = ctx->world > 1 ? nccl() : nullptr;
    if (ctx->world > 1 && (!api || !ctx->comm)) return fail(ctx, BIOT_E_NCCL, "NCCL not initialised");
    biot_status st = biot_gs_begin_gmres(ctx, K, k);
    if (st != BIOT_OK) return st;
    const size_t n = (size_t)ctx->N * ctx->nc;
    for (int w = 0; w < ctx->n_t + K - 1; ++w) {
        if (api && (gs_recv(ctx, w) || gs_send(ctx, w))) {   // one slice per wave between neighbours
            ncclResult_t r = api->GroupStart();
            if (r == ncclSuccess && gs_send(ctx, w))
                r = api->Send(ctx->sendbuf, n, ncclFloat64, ctx->rank + 1, ctx->comm, ctx->stream);
            if (r == ncclSuccess && gs_recv(ctx, w))
                r = api->Recv(ctx->ghost, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->stream);
            ncclResult_t r2 = api->GroupEnd();
            if (r != ncclSuccess || r2 != ncclSuccess) return fail(ctx, BIOT_E_NCCL, "NCCL wave exchange failed");
        }
        st = gs_run_wave(ctx);
        if (st != BIOT_OK) return st;
    }
    return biot_gs_end(ctx);
}

// Sweep partition over NCCL: lockstep global waves; at the start of wave W every rank sends
// the slice it finished at wave W - 1 and receives the one it starts from at W; at the end
// the last rank's x^K is broadcast so that every rank continues from it.
static biot_status iterate_gs_sweeps(biot_ctx *ctx, int32_t K, int32_t k) {
    NcclApi *api = nccl();
    if (!api || !ctx->comm || !api->Bcast) return fail(ctx, BIOT_E_NCCL, "NCCL not initialised");
    biot_status st = biot_gs_begin_gmres(ctx, K, k);
    if (st != BIOT_OK) return st;
    const size_t n = (size_t)ctx->N * ctx->nc;
    for (int W = 0; W < ctx->n_t + K - 1; ++W) {
        int ti, to;
        const bool rin = sw_in(ctx, W, &ti), sout = W > 0 && sw_out(ctx, W - 1, &to);
        if (rin || sout) {
            ncclResult_t r = api->GroupStart();
            if (r == ncclSuccess && sout) r = api->Send(ctx->sendbuf, n, ncclFloat64, ctx->rank + 1, ctx->comm, ctx->stream);
            if (r == ncclSuccess && rin) r = api->Recv(ctx->sweep_in, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->stream);
            ncclResult_t r2 = api->GroupEnd();
            if (r != ncclSuccess || r2 != ncclSuccess) return fail(ctx, BIOT_E_NCCL, "NCCL sweep-pipeline exchange failed");
        }
        if ((st = gs_run_wave(ctx)) != BIOT_OK) return st;
    }
    if ((st = biot_gs_end(ctx)) != BIOT_OK) return st;
    const size_t panel = (size_t)ctx->rows_alloc * ctx->pitch;
    ncclResult_t r = api->Bcast(ctx->xbase[ctx->cur], ctx->xbase[ctx->cur], panel, ncclFloat64, ctx->world - 1,
                                ctx->comm, ctx->stream);
    if (r != ncclSuccess) return fail(ctx, BIOT_E_NCCL, "NCCL broadcast of x^K failed");
    return wait_stream(ctx);
}

biot_status biot_iterate_gs(biot_ctx *ctx, int32_t K) { return biot_iterate_gs_gmres(ctx, K, 0); }

biot_status biot_iterate_gmres(biot_ctx *ctx, int32_t K, int32_t k) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    biot_status st = gmres_check(ctx, K, k);
    if (st != BIOT_OK || K == 0) return st;
    CU(cudaSetDevice(ctx->device));
    if ((st = gmres_alloc(ctx, k)) != BIOT_OK) return st;
    CU(cudaEventRecord(ctx->ev_a, ctx->stream));
    for (int32_t it = 0; it < K; ++it) {
        if ((st = halo_exchange(ctx)) != BIOT_OK) return st;
        Window win;
        win.len = ctx->n_tl;
        win.ghost = ctx->ghost;
        double *x = ctx->x[ctx->cur];
        if ((st = gmres_cycle(ctx, k, ctx->tmap[ctx->cur], x, x, win)) != BIOT_OK) return st;
        double *hslot = ctx->hist + (size_t)(ctx->iterations % ctx->hist_cap) * ctx->n_tl * 2;
        CU(biot::launch_finalize(ctx->partial, (int)ctx->groups, ctx->n_tl, hslot, ctx->nonfinite, ctx->fin_scratch,
                                 ctx->stream, nullptr, 0, 1, ctx->fin_tickets));
        ctx->send_dirty = true;
        ctx->iterations++;
    }
    CU(cudaEventRecord(ctx->ev_b, ctx->stream));
    {
        biot_status ws = wait_done(ctx, ctx->ev_b);
        if (ws != BIOT_OK) return ws;
    }
    float tot = 0.f;
    CU(cudaEventElapsedTime(&tot, ctx->ev_a, ctx->ev_b));
    ctx->last_ms_iter = tot / K;
    ctx->last_ms_sweep = tot / K;
    int nf = 0;
    CU(cudaMemcpyAsync(&nf, ctx->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (nf) return fail(ctx, BIOT_E_NONFINITE, "a residual norm became non-finite");
    return BIOT_OK;
}

// Chebyshev inner inverses inside P~2: per outer iteration the
// residual with its norms (main kernel, P~1 first-pass mode: Z = (D_A^{-1} r_u, r_p)),
// then m Chebyshev steps for A and S~p on all steps at once (cheb_kernels.cu), and the
// damped update.  Jacobi in time; any mesh (generic kernels for the inner steps).
biot_status biot_iterate_cheb(biot_ctx *ctx, int32_t K, int32_t m, double alpha) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (K < 0 || m < 1 || m > 64 || !(alpha > 1.0) || !std::isfinite(alpha))
        return fail(ctx, BIOT_E_INVALID, "need K >= 0, 1 <= m <= 64 and alpha > 1");
    if (K == 0) return BIOT_OK;
    const bool p1 = ctx->precond == 1;
    CU(cudaSetDevice(ctx->device));
    const size_t panel_bytes = (size_t)ctx->rows_alloc * ctx->pitch * sizeof(double);
    const int need = m == 1 ? 2 : 4;   // s (Z), d0 [, d1, y]
    for (int q = 0; q < need; ++q)
        if (!ctx->cb_base[q]) {
            ALLOC(ctx->cb_base[q], panel_bytes);
            CU(cudaMemsetAsync(ctx->cb_base[q], 0, panel_bytes, ctx->stream));
            ctx->cb[q] = ctx->cb_base[q] + ctx->pad * ctx->nc * ctx->pitch;
        }
    auto bounds = [&](double lmax, double &theta, double &delta) {
        theta = 0.5 * (lmax + lmax / alpha);
        delta = 0.5 * (lmax - lmax / alpha);
    };
    double th_u, de_u, th_p, de_p;
    bounds(ctx->lmax_u, th_u, de_u);
    bounds(ctx->lmax_p, th_p, de_p);
    biot::ChebArgs c{};
    c.blk = ctx->blk;
    c.cols = ctx->cols;
    for (int q = 0; q < 32; ++q) c.off[q] = q < (int)ctx->offsets.size() ? ctx->offsets[q] : 0;
    c.dinv = ctx->dinv;
    c.n_nodes = ctx->N;
    c.pitch = ctx->pitch;
    c.nc = ctx->nc;
    c.n_tl = ctx->n_tl;
    c.omega = ctx->omega;
    c.inv_theta_u = th_u > 0.0 ? 1.0 / th_u : 0.0;
    c.inv_theta_p = th_p > 0.0 ? 1.0 / th_p : 0.0;
    c.rows = p1 ? 1 : 3;
    c.p_sign = p1 ? 1.0 : -1.0;
    CU(cudaEventRecord(ctx->ev_a, ctx->stream));
    double *const zsave = ctx->z;
    for (int32_t it = 0; it < K; ++it) {
        biot_status st = halo_exchange(ctx);
        if (st != BIOT_OK) { ctx->z = zsave; return st; }
        const double *xin = ctx->x[ctx->cur];
        double *xout = ctx->x[1 - ctx->cur];
        // r and its norms; Z = (D_A^{-1} r_u, r_p) into the s panel (x_u into xout is
        // overwritten by the last Chebyshev pass)
        ctx->z = ctx->cb[0];
        cudaError_t e = launch_main(ctx, biot::MODE_P1_PASS1, xin, xout);
        ctx->z = zsave;
        CU(e);
        double *hslot = ctx->hist + (size_t)(ctx->iterations % ctx->hist_cap) * ctx->n_tl * 2;
        CU(biot::launch_finalize(ctx->partial, (int)ctx->groups, ctx->n_tl, hslot, ctx->nonfinite,
                                 ctx->fin_scratch, ctx->stream, nullptr, 0, 1, ctx->fin_tickets));
        c.s = ctx->cb[0];
        c.x = xin;
        c.xn = xout;
        c.sendbuf = ctx->world > 1 ? ctx->sendbuf : nullptr;
        // P~2: both blocks at once.  P~1 (eq. p1): the displacement block first (it cannot
        // write x yet), then r~_p = B^T z_u - r_p and the pressure block on it.
        auto run_block = [&](int rows, bool final_block) -> cudaError_t {
            c.rows = rows;
            c.last = final_block && m == 1;
            c.dn = ctx->cb[1];
            c.first = 0;
            c.sn = nullptr;
            cudaError_t e2 = cudaSuccess;
            if (rows != 2 && m >= 2) {
                // P~2 (and the P~1 displacement block): the start is fused into the first step,
                // which reads the Z panel (cb[0])
                // and writes s to cb[1]; d alternates cb[2] (odd k) / cb[0] (even k)
                double rho_u = de_u / th_u, rho_p = de_p / th_p;
                for (int k = 1; k < m; ++k) {
                    const double ru = 1.0 / (2.0 * th_u / de_u - rho_u), rp = 1.0 / (2.0 * th_p / de_p - rho_p);
                    c.c1_u = ru * rho_u;
                    c.c2_u = 2.0 * ru / de_u;
                    c.c1_p = rp * rho_p;
                    c.c2_p = 2.0 * rp / de_p;
                    rho_u = ru;
                    rho_p = rp;
                    c.first = k == 1;
                    c.s = k == 1 ? ctx->cb[0] : ctx->cb[1];
                    c.sn = k == 1 ? ctx->cb[1] : nullptr;
                    c.d = k == 1 ? nullptr : (k % 2 == 0 ? ctx->cb[2] : ctx->cb[0]);
                    c.dn = k % 2 == 1 ? ctx->cb[2] : ctx->cb[0];
                    c.y = k == 1 ? nullptr : ctx->cb[3];
                    c.yn = ctx->cb[3];
                    c.last = final_block && k == m - 1;
                    e2 = biot::launch_cheb_step(ctx->d, ctx->path, ctx->S, c, ctx->stream);
                    if (e2 != cudaSuccess) return e2;
                }
                c.first = 0;
                c.sn = nullptr;
                c.s = ctx->cb[0];
                return cudaSuccess;
            }
            if (rows != 2) e2 = biot::launch_cheb_init(c, ctx->stream);
            if (e2 != cudaSuccess) return e2;
            if (rows == 2) {        // P~1 pressure start from z_u
                c.zu = m == 1 ? ctx->cb[1] : ctx->cb[3];
                c.last = m == 1;
                e2 = biot::launch_cheb_p1_rhs(ctx->d, ctx->path, ctx->S, c, ctx->stream);
                if (e2 != cudaSuccess) return e2;
            }
            double rho_u = de_u / th_u, rho_p = de_p / th_p;   // rho_0 = 1 / sigma
            for (int k = 1; k < m; ++k) {
                const double ru = 1.0 / (2.0 * th_u / de_u - rho_u), rp = 1.0 / (2.0 * th_p / de_p - rho_p);
                c.c1_u = ru * rho_u;
                c.c2_u = 2.0 * ru / de_u;
                c.c1_p = rp * rho_p;
                c.c2_p = 2.0 * rp / de_p;
                rho_u = ru;
                rho_p = rp;
                c.d = ctx->cb[1 + (k - 1) % 2];
                c.dn = ctx->cb[1 + k % 2];
                c.y = k == 1 ? nullptr : ctx->cb[3];
                c.yn = ctx->cb[3];
                c.last = final_block && k == m - 1;
                e2 = biot::launch_cheb_step(ctx->d, ctx->path, ctx->S, c, ctx->stream);
                if (e2 != cudaSuccess) return e2;
            }
            return cudaSuccess;
        };
        if (p1) {
            CU(run_block(1, false));
            CU(run_block(2, true));
        } else {
            CU(run_block(3, true));
        }
        ctx->cur = 1 - ctx->cur;
        ctx->iterations++;
        if (ctx->world > 1) ctx->send_dirty = false;
    }
    CU(cudaEventRecord(ctx->ev_b, ctx->stream));
    {
        biot_status ws = wait_done(ctx, ctx->ev_b);
        if (ws != BIOT_OK) return ws;
    }
    float tot = 0.f;
    CU(cudaEventElapsedTime(&tot, ctx->ev_a, ctx->ev_b));
    ctx->last_ms_iter = tot / K;
    ctx->last_ms_sweep = tot / K;
    int nf = 0;
    CU(cudaMemcpyAsync(&nf, ctx->nonfinite, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (nf) return fail(ctx, BIOT_E_NONFINITE, "a residual norm became non-finite");
    return BIOT_OK;
}

biot_status biot_residual_norms(biot_ctx *ctx, double *out) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!out) return fail(ctx, BIOT_E_INVALID, "out is NULL");
    CU(cudaSetDevice(ctx->device));
    biot_status st = halo_exchange(ctx);
    if (st != BIOT_OK) return st;
    CU(launch_main(ctx, biot::MODE_RESIDUAL, ctx->x[ctx->cur], nullptr));
    CU(biot::launch_finalize(ctx->partial, (int)ctx->groups, ctx->n_tl, ctx->norms, ctx->nonfinite,
                             ctx->fin_scratch, ctx->stream, nullptr, 0, 1, ctx->fin_tickets));
    CU(cudaMemcpyAsync(out, ctx->norms, (size_t)ctx->n_tl * 2 * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    return wait_stream(ctx);
    return BIOT_OK;
}

biot_status biot_residual_history(biot_ctx *ctx, int64_t k, double *out) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!out) return fail(ctx, BIOT_E_INVALID, "out is NULL");
    if (k < 0 || k >= ctx->iterations || k < ctx->iterations - ctx->hist_cap)
        return fail(ctx, BIOT_E_STATE, "iteration " + std::to_string(k) + " not retained");
    CU(cudaSetDevice(ctx->device));
    CU(cudaMemcpyAsync(out, ctx->hist + (size_t)(k % ctx->hist_cap) * ctx->n_tl * 2,
                       (size_t)ctx->n_tl * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return BIOT_OK;
}

biot_status biot_solution(biot_ctx *ctx, int32_t n, int32_t count, double *out) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!out || count < 0) return fail(ctx, BIOT_E_INVALID, "out is NULL or count < 0");
    CU(cudaSetDevice(ctx->device));
    const int64_t rows = ctx->N * ctx->nc;
    const size_t vb = (size_t)rows * sizeof(double);
    if (n == ctx->first_step - 1 && count == 1) {   // the ghost / x_0
        CU(cudaMemcpyAsync(out, ctx->ghost, vb, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        return BIOT_OK;
    }
    if (n < ctx->first_step || n + count > ctx->first_step + ctx->n_tl)
        return fail(ctx, BIOT_E_INVALID, "steps outside the owned slab");
    for (int32_t done = 0; done < count;) {
        const int32_t m = (int32_t)std::min<int64_t>(ctx->staging_steps, count - done);
        const int t_first = n - ctx->first_step + done;
        gather_steps_kernel<<<1184, 256, 0, ctx->stream>>>(ctx->x[ctx->cur], ctx->staging, rows,
                                                           ctx->pitch, t_first, m);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(out + (size_t)done * rows, ctx->staging, (size_t)m * vb, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        done += m;
    }
    return BIOT_OK;
}

biot_status biot_last_slice(biot_ctx *ctx, double *out) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (ctx->world > 1 && !ctx->send_dirty) {
        // the slice NCCL would send: the send buffer the sweep kernels wrote (so the
        // manual-halo tests check exactly the data path of the NCCL exchange)
        if (!out) return fail(ctx, BIOT_E_INVALID, "out is NULL");
        CU(cudaSetDevice(ctx->device));
        CU(cudaMemcpyAsync(out, ctx->sendbuf, (size_t)ctx->N * ctx->nc * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        return BIOT_OK;
    }
    return biot_solution(ctx, ctx->first_step + ctx->n_tl - 1, 1, out);
}

biot_status biot_set_ghost(biot_ctx *ctx, const double *x) {
    if (!ctx) return fail(nullptr, BIOT_E_INVALID, "ctx is NULL");
    if (!x) return fail(ctx, BIOT_E_INVALID, "x is NULL");
    if (ctx->rank == 0 && ctx->world > 1)
        return fail(ctx, BIOT_E_STATE, "rank 0's ghost is x_0 (fixed)");
    CU(cudaSetDevice(ctx->device));
    if (ctx->sweep_mode) {   // the predecessor's finished slice for the next wave
        CU(cudaMemcpyAsync(ctx->sweep_in, x, (size_t)ctx->N * ctx->nc * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        return BIOT_OK;
    }
    if (ctx->rank == 0) ctx->x0_zero = false;   // a replaced x_0 is no longer known to be zero
    CU(cudaMemcpyAsync(ctx->ghost, x, (size_t)ctx->N * ctx->nc * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return BIOT_OK;
}

biot_status biot_get_info(const biot_ctx *ctx, biot_info *o) {
    if (!ctx || !o) return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    o->dim = ctx->d;
    o->n_comp = ctx->nc;
    o->n_nodes = ctx->N;
    o->n_dof = ctx->N * ctx->nc;
    o->n_t = ctx->n_t;
    o->n_t_local = ctx->n_tl;
    o->first_step = ctx->first_step;
    o->iterations = ctx->iterations;
    o->kernel_path = ctx->kern == 1 ? ctx->path : ctx->kern + 1;   // 4 march, 5 tile2d, 7 tile3d
    o->n_slots = ctx->S;
    o->beta = ctx->beta;
    const double st = (double)ctx->N * ctx->nc * ctx->n_tl;
    o->bytes_per_iter = 16.0 * st + 8.0 * (double)(ctx->nnz_AA + ctx->nnz_AP);
    o->flops_per_iter = 2.0 * (double)(ctx->nnz_AA + ctx->nnz_AP) * ctx->n_tl;
    o->device_bytes = (double)ctx->device_bytes;
    const int mm = main_mode(ctx);
    o->launches_per_iter = 1 + (mm == biot::MODE_P1_PASS1 ? 1 : 0) + 1 + (ctx->defer0 ? 1 : 0);   // sweep (+ pass 2), finalize (+ step 0)
    o->interior_nodes = (int32_t)ctx->n_interior;
    o->comm_nranks = 0;
    if (ctx->comm && nccl() && nccl()->CommCount) nccl()->CommCount(ctx->comm, &o->comm_nranks);
    o->graph = ctx->use_graph ? 1 : 0;
    return BIOT_OK;
}

biot_status biot_last_timing(const biot_ctx *ctx, double *out_ms) {
    if (!ctx || !out_ms) return fail(nullptr, BIOT_E_INVALID, "NULL argument");
    out_ms[0] = ctx->last_ms_iter;
    out_ms[1] = ctx->last_ms_sweep;
    return BIOT_OK;
}

void biot_destroy(biot_ctx *ctx) {
    if (!ctx) return;
    free_all(ctx);
    delete ctx;
}

}  // extern "C"
