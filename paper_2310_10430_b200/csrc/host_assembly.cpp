// Host-side assembly of the stabilised P1-P1 Biot operators (setup, not hot path).
//
// PAPER.md L87-105 (bilinear forms a, b, c), L120-132 (stabilisation beta),
// L134-231 (backward Euler, matrix form AA X^m = A' X^{m-1} + f^m), with the
// readings of DESIGN.md: R7 (lambda div-div term in a), R8 (storage S M), R9
// (per-cell kappa; (beta/K) c -> beta L), R11 (homogeneous Dirichlet by
// elimination), R16 (constant top traction, load switched on for n >= 1).
//
// Layout: node-interleaved (d+1)x(d+1) blocks per (row node, neighbour slot),
// so that the sweep kernel does d+1 FMAs per gathered x value.  Two neighbour
// encodings: BDIA (column = row + offsets[slot], offsets shared by all nodes --
// true for structured meshes in their natural numbering) and ELL (explicit
// column per slot) for anything else.
#include "host_assembly.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <cstring>
#include <unordered_map>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace biot {

int block_width(int nc) { return (nc * nc + 2) / 2 * 2; }   // (d+1)^2 + 1, padded to 16 B

namespace {

// Barycentric gradients of a simplex by Gauss-Jordan inversion of the
// (d+1)x(d+1) Vandermonde-type matrix V[a] = [1, x_a]: phi_a(x) = sum_k
// Vinv[k][a] [1, x]_k, hence grad phi_a = (Vinv[1..d][a]).  det V = det of the
// edge matrix, so det V > 0 <=> positive orientation; |T| = det V / d!.
// Returns signed measure (<= 0 -> degenerate / inverted).
double simplex_gradients(int d, const double *const *X, double g[4][3]) {
    const int n = d + 1;
    double V[4][8];
    for (int a = 0; a < n; ++a) {
        V[a][0] = 1.0;
        for (int k = 0; k < d; ++k) V[a][1 + k] = X[a][k];
        for (int k = 0; k < n; ++k) V[a][n + k] = (a == k) ? 1.0 : 0.0;
    }
    double det = 1.0;
    for (int col = 0; col < n; ++col) {
        int piv = col;
        for (int r = col + 1; r < n; ++r)
            if (std::fabs(V[r][col]) > std::fabs(V[piv][col])) piv = r;
        if (V[piv][col] == 0.0) return 0.0;
        if (piv != col) {
            for (int k = 0; k < 2 * n; ++k) std::swap(V[piv][k], V[col][k]);
            det = -det;
        }
        const double p = V[col][col];
        det *= p;
        for (int k = 0; k < 2 * n; ++k) V[col][k] /= p;
        for (int r = 0; r < n; ++r) {
            if (r == col) continue;
            const double m = V[r][col];
            if (m == 0.0) continue;
            for (int k = 0; k < 2 * n; ++k) V[r][k] -= m * V[col][k];
        }
    }
    // V[:, n:] now holds Vinv; grad phi_a[k] = Vinv[1+k][a]
    double gmax = 0.0;
    for (int a = 0; a < n; ++a)
        for (int k = 0; k < d; ++k) {
            g[a][k] = V[1 + k][n + a];
            gmax = std::max(gmax, std::fabs(g[a][k]));
        }
    // components that vanish exactly (axis-aligned edges/faces) come out of the
    // elimination as rounding residue; store them as the 0 they are (reading R21)
    for (int a = 0; a < n; ++a)
        for (int k = 0; k < d; ++k)
            if (std::fabs(g[a][k]) <= 16.0 * std::numeric_limits<double>::epsilon() * gmax) g[a][k] = 0.0;
    return det / (d == 2 ? 2.0 : 6.0);
}

}  // namespace

std::string assemble(const biot_mesh &mesh, const biot_material &mat, const biot_bc &bc,
                     double dt, HostOperator &op) {
    // ---------------- validation ----------------
    if (mesh.dim != 2 && mesh.dim != 3) return "mesh.dim must be 2 or 3";
    if (mesh.n_nodes <= 0 || mesh.n_cells <= 0 || !mesh.coords || !mesh.cells)
        return "mesh must have nodes, cells, coords and connectivity";
    if (mesh.n_nodes > (int64_t)2000000000) return "mesh too large (n_nodes > 2e9)";
    if (!(dt > 0.0) || !std::isfinite(dt)) return "dt must be positive and finite";
    if (!(mat.mu > 0.0) || !(mat.lambda >= 0.0) || !std::isfinite(mat.alpha) ||
        !(mat.storage >= 0.0))
        return "material: need mu > 0, lambda >= 0, finite alpha, storage >= 0";
    if (!mat.kappa && !(mat.kappa_uniform > 0.0)) return "material: kappa_uniform must be > 0";
    if (mat.beta < 0.0 && !(mat.h > 0.0)) return "material: h must be > 0 when beta < 0";
    if (!bc.dirichlet) return "bc.dirichlet mask is required";
    if (bc.n_traction_facets < 0 || (bc.n_traction_facets > 0 && !bc.traction_facets))
        return "bc: traction facets missing";
    if (bc.n_sources < 0 || (bc.n_sources > 0 && (!bc.source_eval || !bc.source_coef)))
        return "bc: n_sources > 0 needs source_eval and source_coef";

    const int d = mesh.dim, nc = d + 1, nv = d + 1;
    const int64_t N = mesh.n_nodes, NC = mesh.n_cells;
    op.d = d;
    op.nc = nc;
    op.n_nodes = N;
    for (int64_t e = 0; e < NC; ++e)
        for (int a = 0; a < nv; ++a) {
            int32_t v = mesh.cells[e * nv + a];
            if (v < 0 || v >= N) return "cell references a node out of range";
        }
    if (mat.kappa)
        for (int64_t e = 0; e < NC; ++e)
            if (!(mat.kappa[e] > 0.0) || !std::isfinite(mat.kappa[e]))
                return "kappa must be positive and finite";

    // beta = h / (4 (lambda + 2 mu))
    op.beta = mat.beta >= 0.0 ? mat.beta : mat.h / (4.0 * (mat.lambda + 2.0 * mat.mu));

    // ---------------- neighbour structure ----------------
    // distinct column-row offsets over all cell-local node pairs
    std::vector<int64_t> offs;
    {
        std::unordered_map<int64_t, int> seen;
        bool too_many = false;
        for (int64_t e = 0; e < NC && !too_many; ++e) {
            const int32_t *cn = mesh.cells + e * nv;
            for (int a = 0; a < nv; ++a)
                for (int b = 0; b < nv; ++b) {
                    int64_t o = (int64_t)cn[b] - cn[a];
                    if (seen.emplace(o, 1).second) {
                        offs.push_back(o);
                        if ((int)offs.size() > kMaxSlots) { too_many = true; break; }
                    }
                }
        }
        if (too_many) offs.clear();
    }
    const int bdia_cap = (d == 2) ? 7 : 15;   // kernel instantiations
    std::vector<std::vector<int32_t>> adj;     // ELL only
    if (!offs.empty() && (int)offs.size() <= bdia_cap) {
        op.path = PATH_BDIA;
        std::sort(offs.begin(), offs.end(), [](int64_t a, int64_t b) {
            if ((a == 0) != (b == 0)) return a == 0;
            return a < b;
        });
        while ((int)offs.size() < bdia_cap) offs.push_back(0);   // padding slots: zero blocks
        op.offsets = offs;
        op.n_slots = bdia_cap;
        op.max_abs_offset = 0;
        for (auto o : offs) op.max_abs_offset = std::max<int64_t>(op.max_abs_offset, std::llabs(o));
    } else {
        op.path = PATH_ELL;
        adj.assign(N, {});
        for (int64_t e = 0; e < NC; ++e) {
            const int32_t *cn = mesh.cells + e * nv;
            for (int a = 0; a < nv; ++a)
                for (int b = 0; b < nv; ++b) adj[cn[a]].push_back(cn[b]);
        }
        int maxdeg = 0;
        for (int64_t i = 0; i < N; ++i) {
            auto &v = adj[i];
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            // self first
            auto it = std::find(v.begin(), v.end(), (int32_t)i);
            std::rotate(v.begin(), it, it + 1);
            maxdeg = std::max<int>(maxdeg, (int)v.size());
        }
        int S = maxdeg <= 8 ? 8 : maxdeg <= 16 ? 16 : maxdeg <= 32 ? 32 : -1;
        if (S < 0) return "mesh node degree exceeds 31 neighbours (unsupported)";
        op.n_slots = S;
        op.cols.assign((size_t)N * S, 0);
        for (int64_t i = 0; i < N; ++i)
            for (int s = 0; s < S; ++s)
                op.cols[(size_t)i * S + s] = s < (int)adj[i].size() ? adj[i][s] : (int32_t)i;
    }
    const int S = op.n_slots;
    const int W = block_width(nc);

    // node -> incident cells (counting sort), so nodes can be assembled in parallel
    std::vector<int64_t> inc_ptr(N + 1, 0);
    for (int64_t e = 0; e < NC; ++e)
        for (int a = 0; a < nv; ++a) inc_ptr[mesh.cells[e * nv + a] + 1]++;
    for (int64_t i = 0; i < N; ++i) inc_ptr[i + 1] += inc_ptr[i];
    std::vector<int64_t> inc(inc_ptr[N]);
    {
        std::vector<int64_t> fill(inc_ptr.begin(), inc_ptr.end() - 1);
        for (int64_t e = 0; e < NC; ++e)
            for (int a = 0; a < nv; ++a) inc[fill[mesh.cells[e * nv + a]]++] = e;
    }

    op.blk.assign((size_t)N * S * W, 0.0);
    const double lam = mat.lambda, mu = mat.mu, alpha = mat.alpha, Sst = mat.storage;
    const double beta = op.beta, tau = dt;
    const double mass_den = (double)(nv * (nv + 1));
    int bad_cell = -1;
    std::unordered_map<int64_t, int> off2slot;
    if (op.path == PATH_BDIA)
        for (int s = S - 1; s >= 0; --s) off2slot[op.offsets[s]] = s;   // first occurrence wins

#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < N; ++i) {
        double *bi = op.blk.data() + (size_t)i * S * W;
        // |contributions| per entry: sums that vanish in exact arithmetic (e.g. the
        // u_x-u_x coupling of diagonal Kuhn neighbours, the self-block B entries of an
        // interior node) leave a rounding residue; it is stored as the exact 0 it is
        // (reading R21), so every kernel sees the structural zeros
        double absb[kMaxSlots * 18];
        for (int k = 0; k < S * W; ++k) absb[k] = 0.0;
        auto add = [&](int slot, int k, double v, double mag) {
            bi[(size_t)slot * W + k] += v;
            absb[slot * W + k] += mag;
        };
        for (int64_t q = inc_ptr[i]; q < inc_ptr[i + 1]; ++q) {
            const int64_t e = inc[q];
            const int32_t *cn = mesh.cells + e * nv;
            const double *X[4];
            for (int a = 0; a < nv; ++a) X[a] = mesh.coords + (size_t)cn[a] * d;
            double g[4][3];
            const double vol = simplex_gradients(d, X, g);
            if (!(vol > 0.0)) {
#pragma omp critical
                bad_cell = (int)std::min<int64_t>(e, 2147483647);
                continue;
            }
            const double kap = mat.kappa ? mat.kappa[e] : mat.kappa_uniform;
            int a = 0;
            while (cn[a] != i) ++a;   // local index of the row node
            for (int b = 0; b < nv; ++b) {
                const int64_t j = cn[b];
                int slot;
                if (op.path == PATH_BDIA) {
                    slot = off2slot.at(j - i);
                } else {
                    const int32_t *ci = op.cols.data() + (size_t)i * S;
                    slot = 0;
                    while (ci[slot] != j) ++slot;
                }
                double gab = 0.0, gabs = 0.0;
                for (int k = 0; k < d; ++k) {
                    gab += g[a][k] * g[b][k];
                    gabs += std::fabs(g[a][k] * g[b][k]);
                }
                const double lab = vol * gab;                                  // L_ab
                const double mab = vol * (a == b ? 2.0 : 1.0) / mass_den;      // M_ab
                // displacement rows: a(u, v) incl. lambda div div  (P:L96 + R7)
                for (int c = 0; c < d; ++c)
                    for (int ee = 0; ee < d; ++ee)
                        add(slot, c * nc + ee,
                            vol * (mu * gab * (c == ee ? 1.0 : 0.0) + mu * g[a][ee] * g[b][c] +
                                   lam * g[a][c] * g[b][ee]),
                            vol * (mu * gabs * (c == ee ? 1.0 : 0.0) + std::fabs(mu * g[a][ee] * g[b][c]) +
                                   std::fabs(lam * g[a][c] * g[b][ee])));
                // B = -b(v, p): -alpha int q_b div v_(a,c)
                for (int c = 0; c < d; ++c) {
                    const double v = -alpha * vol * g[a][c] / nv;
                    add(slot, c * nc + d, v, std::fabs(v));
                }
                // B^T: pressure row a, displacement column (b, e)
                for (int ee = 0; ee < d; ++ee) {
                    const double v = -alpha * vol * g[b][ee] / nv;
                    add(slot, d * nc + ee, v, std::fabs(v));
                }
                // -(S M + tau C_kappa + beta L)  (P:L159 with R8, R9)
                add(slot, d * nc + d, -(Sst * mab + (tau * kap + beta) * lab),
                    Sst * mab + (tau * kap + beta) * vol * gabs);
                // A' pressure-pressure: -(S M + beta L)
                add(slot, nc * nc, -(Sst * mab + beta * lab), Sst * mab + beta * vol * gabs);
            }
        }
        const double tol = 32.0 * std::numeric_limits<double>::epsilon();
        for (int k = 0; k < S * W; ++k)
            if (std::fabs(bi[k]) <= tol * absb[k]) bi[k] = 0.0;
    }
    if (bad_cell >= 0) return "degenerate or inverted cell " + std::to_string(bad_cell);

    // ---------------- Dirichlet elimination, diagonals, load ----------------
    op.fixed.assign(bc.dirichlet, bc.dirichlet + (size_t)N * nc);
    for (auto &m : op.fixed) m = m ? 1 : 0;

    // further load terms (R24), from the blocks before the Dirichlet columns are dropped
    {
        auto column_of = [&](int64_t i, int s) -> int64_t {
            if (op.path == PATH_BDIA) {
                const int64_t j = i + op.offsets[s];
                return (j < 0 || j >= N) ? -1 : j;
            }
            return op.cols[(size_t)i * S + s];
        };
        auto nonzero = [](const std::vector<double> &v) {
            for (double x : v)
                if (x != 0.0) return true;
            return false;
        };
        // sources: [ int f . phi_a ; -dt int g phi_a ] on free rows, by a fixed quadrature
        // per cell (R24): triangles the 7-point degree-5 rule, tetrahedra the 4-point
        // degree-2 rule; barycentric points, weights relative to |T|
        if (bc.n_sources > 0) {
            std::vector<std::array<double, 4>> qp;
            std::vector<double> qw;
            if (d == 2) {
                const double a1 = 0.059715871789770, b1 = 0.470142064105115;
                const double a2 = 0.797426985353087, b2 = 0.101286507323456;
                const double w1 = 0.132394152788506, w2 = 0.125939180544827;
                qp = {{1.0 / 3, 1.0 / 3, 1.0 / 3, 0}, {a1, b1, b1, 0}, {b1, a1, b1, 0}, {b1, b1, a1, 0},
                      {a2, b2, b2, 0}, {b2, a2, b2, 0}, {b2, b2, a2, 0}};
                qw = {0.225, w1, w1, w1, w2, w2, w2};
            } else {
                const double a = 0.5854101966249685, b = 0.1381966011250105;
                qp = {{a, b, b, b}, {b, a, b, b}, {b, b, a, b}, {b, b, b, a}};
                qw = {0.25, 0.25, 0.25, 0.25};
            }
            const int nq = (int)qw.size();
            std::vector<double> xyz((size_t)NC * nq * d), vol(NC);
#pragma omp parallel for schedule(static)
            for (int64_t e = 0; e < NC; ++e) {
                const int32_t *cn = mesh.cells + e * nv;
                const double *X[4];
                for (int a = 0; a < nv; ++a) X[a] = mesh.coords + (size_t)cn[a] * d;
                double g[4][3];
                vol[e] = simplex_gradients(d, X, g);
                for (int k = 0; k < nq; ++k)
                    for (int c = 0; c < d; ++c) {
                        double v = 0.0;
                        for (int a = 0; a < nv; ++a) v += qp[k][a] * X[a][c];
                        xyz[((size_t)e * nq + k) * d + c] = v;
                    }
            }
            std::vector<double> vals((size_t)NC * nq * nc);
            for (int q = 0; q < bc.n_sources; ++q) {
                std::fill(vals.begin(), vals.end(), std::numeric_limits<double>::quiet_NaN());
                bc.source_eval(q, NC * nq, xyz.data(), vals.data(), bc.source_user);
                for (double v : vals)
                    if (!std::isfinite(v)) return "bc: source_eval returned a non-finite value";
                HostOperator::LoadTerm t;
                t.kind = 0;
                t.src = q;
                t.f.assign((size_t)N * nc, 0.0);
#pragma omp parallel for schedule(dynamic, 1024)
                for (int64_t i = 0; i < N; ++i)
                    for (int64_t r = inc_ptr[i]; r < inc_ptr[i + 1]; ++r) {
                        const int64_t e = inc[r];
                        const int32_t *cn = mesh.cells + e * nv;
                        int a = 0;
                        while (cn[a] != i) ++a;
                        for (int k = 0; k < nq; ++k) {
                            const double wk = vol[e] * qw[k] * qp[k][a];
                            const double *fv = vals.data() + ((size_t)e * nq + k) * nc;
                            for (int c = 0; c < d; ++c) t.f[(size_t)i * nc + c] += wk * fv[c];
                            t.f[(size_t)i * nc + d] += -tau * wk * fv[d];
                        }
                    }
                for (size_t k = 0; k < t.f.size(); ++k)
                    if (op.fixed[k]) t.f[k] = 0.0;
                if (nonzero(t.f)) op.extra.push_back(std::move(t));
            }
        }
        // Dirichlet lifting: the columns of fixed DoFs times x_D
        if (bc.dirichlet_values) {
            const double *xd = bc.dirichlet_values;
            for (size_t k = 0; k < (size_t)N * nc; ++k)
                if (op.fixed[k] && !std::isfinite(xd[k])) return "bc: dirichlet_values must be finite";
            HostOperator::LoadTerm now, prev;
            now.kind = 1;
            prev.kind = 2;
            now.f.assign((size_t)N * nc, 0.0);
            prev.f.assign((size_t)N * nc, 0.0);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < N; ++i)
                for (int s = 0; s < S; ++s) {
                    const int64_t j = column_of(i, s);
                    if (j < 0) continue;
                    const double *b = op.blk.data() + ((size_t)i * S + s) * W;
                    for (int cc = 0; cc < nc; ++cc) {
                        if (!op.fixed[(size_t)j * nc + cc]) continue;
                        const double v = xd[(size_t)j * nc + cc];
                        for (int c = 0; c < nc; ++c) now.f[(size_t)i * nc + c] -= b[c * nc + cc] * v;
                        // A' row p: B^T columns (= AA's), H column for the pressure
                        prev.f[(size_t)i * nc + d] += (cc < d ? b[d * nc + cc] : b[nc * nc]) * v;
                    }
                }
            for (size_t k = 0; k < (size_t)N * nc; ++k)
                if (op.fixed[k]) now.f[k] = prev.f[k] = 0.0;
            if (nonzero(now.f)) op.extra.push_back(std::move(now));
            if (nonzero(prev.f)) op.extra.push_back(std::move(prev));
        }
    }
    op.dinv.assign((size_t)N * nc, 0.0);
    // diagonals before masking (only read on free DoFs)
    for (int64_t i = 0; i < N; ++i) {
        const double *b0 = op.blk.data() + (size_t)i * S * W;   // slot 0 is self
        for (int c = 0; c < nc; ++c) {
            if (op.fixed[(size_t)i * nc + c]) continue;
            const double diag = (c < d) ? b0[c * nc + c] : -b0[d * nc + d];
            if (!(diag > 0.0)) return "non-positive preconditioner diagonal at node " +
                                      std::to_string(i);
            op.dinv[(size_t)i * nc + c] = 1.0 / diag;
        }
    }
    int64_t nnzA = 0, nnzP = 0;
#pragma omp parallel for reduction(+ : nnzA, nnzP)
    for (int64_t i = 0; i < N; ++i) {
        for (int s = 0; s < S; ++s) {
            int64_t j;
            if (op.path == PATH_BDIA) {
                j = i + op.offsets[s];
                if (j < 0 || j >= N) j = -1;
            } else {
                j = op.cols[(size_t)i * S + s];
            }
            double *blk = op.blk.data() + ((size_t)i * S + s) * W;
            for (int c = 0; c < nc; ++c)
                for (int cc = 0; cc < nc; ++cc) {
                    double &v = blk[c * nc + cc];
                    if (j < 0 || op.fixed[(size_t)i * nc + c] || op.fixed[(size_t)j * nc + cc]) v = 0.0;
                    if (v != 0.0) nnzA++;
                }
            double &hp = blk[nc * nc];
            if (j < 0 || op.fixed[(size_t)i * nc + d] || op.fixed[(size_t)j * nc + d]) hp = 0.0;
            if (hp != 0.0) nnzP++;
            for (int cc = 0; cc < d; ++cc)
                if (blk[d * nc + cc] != 0.0) nnzP++;
        }
    }
    op.nnz_AA = nnzA;
    op.nnz_AP = nnzP;

    // f = [F; 0]: constant traction on boundary facets, int_f phi_a = |f|/d
    op.load.assign((size_t)N * nc, 0.0);
    for (int64_t k = 0; k < bc.n_traction_facets; ++k) {
        const int32_t *fv = bc.traction_facets + k * d;
        for (int a = 0; a < d; ++a)
            if (fv[a] < 0 || fv[a] >= N) return "traction facet references a node out of range";
        double meas;
        const double *P0 = mesh.coords + (size_t)fv[0] * d;
        const double *P1 = mesh.coords + (size_t)fv[1] * d;
        if (d == 2) {
            meas = std::hypot(P1[0] - P0[0], P1[1] - P0[1]);
        } else {
            const double *P2 = mesh.coords + (size_t)fv[2] * d;
            const double u[3] = {P1[0] - P0[0], P1[1] - P0[1], P1[2] - P0[2]};
            const double v[3] = {P2[0] - P0[0], P2[1] - P0[1], P2[2] - P0[2]};
            const double cx = u[1] * v[2] - u[2] * v[1], cy = u[2] * v[0] - u[0] * v[2],
                         cz = u[0] * v[1] - u[1] * v[0];
            meas = 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
        }
        for (int a = 0; a < d; ++a)
            for (int c = 0; c < d; ++c) op.load[(size_t)fv[a] * nc + c] += meas / d * bc.traction[c];
    }
    for (size_t q = 0; q < op.load.size(); ++q)
        if (op.fixed[q]) op.load[q] = 0.0;
    return "";
}

}  // namespace biot
