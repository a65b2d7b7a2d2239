/*
 * biot_oracle.c -- TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * Plain, slow, obviously-correct CPU oracle for one outer iteration of the
 * inverted (parallel-in-time) time-stepping scheme of arXiv 2310.10430,
 * in the Jacobi-in-time form named by BASELINE.json's north star.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with paper_2310_10430_b200/ (the CUDA product).
 *
 * Citations: "P:Lnnn" = line of PAPER.md (section / equation / algorithm);
 * "R#" = a reading listed in DESIGN.md.
 *
 * Unknown ordering (eq. fullysystem): X = [U; P], U node-major
 * (U[node*d + c]), P[node].  Everything is IEEE fp64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Lame coefficients from E, nu: P:L66-69 (§2.1). */
void oracle_lame(double E, double nu, double *lam, double *mu)
{
    *lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    *mu = E / (2.0 * (1.0 + nu));
}

/* Stabilization factor beta = h / (4 (lambda + 2 mu)): P:L128-132 (§2.2), R5/R6. */
double oracle_beta(double h, double lam, double mu)
{
    return h / (4.0 * (lam + 2.0 * mu));
}

/*
 * Gradients of the P1 barycentric basis on one simplex and its measure |T|.
 * X: (d+1) x d vertex coordinates.  grad: (d+1) x d.  Returns |T| (> 0 for a
 * positively oriented cell), or 0 for a degenerate one.
 * Standard P1 facts: with J = [X_1-X_0 ... X_d-X_0] (columns), the gradients
 * of phi_1..phi_d are the rows of J^{-1}, grad phi_0 = -sum of the others,
 * |T| = |det J| / d!.
 */
static double p1_gradients(int d, const double *X, double *grad)
{
    double J[3][3] = {{0}};
    for (int r = 0; r < d; r++)
        for (int c = 0; c < d; c++)
            J[r][c] = X[(c + 1) * d + r] - X[0 * d + r];   /* column c = X_{c+1} - X_0 */
    double det, inv[3][3];
    if (d == 2) {
        det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        if (det == 0.0) return 0.0;
        inv[0][0] = J[1][1] / det;  inv[0][1] = -J[0][1] / det;
        inv[1][0] = -J[1][0] / det; inv[1][1] = J[0][0] / det;
    } else {
        double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
        if (det == 0.0) return 0.0;
        inv[0][0] = c00 / det;
        inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
        inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
        inv[1][0] = c01 / det;
        inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
        inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
        inv[2][0] = c02 / det;
        inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
        inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    }
    /* grad phi_{a} for a = 1..d is row (a-1) of J^{-1} */
    for (int a = 1; a <= d; a++)
        for (int c = 0; c < d; c++)
            grad[a * d + c] = inv[a - 1][c];
    for (int c = 0; c < d; c++) {
        double s = 0.0;
        for (int a = 1; a <= d; a++) s += grad[a * d + c];
        grad[0 * d + c] = -s;
    }
    double vol = fabs(det) / (d == 2 ? 2.0 : 6.0);
    return det > 0 ? vol : -vol;
}

/*
 * Element matrices of one simplex (P:L87-105 bilinear forms, §2.1; P:L146-154
 * matrix map; readings R7 (lambda term), R9 (kappa per cell), R8 (mass)).
 *   Ae[(a,c),(b,e)] = |T| ( mu (grad phi_a . grad phi_b) delta_ce
 *                          + mu d_e phi_a d_c phi_b + lambda d_c phi_a d_e phi_b )
 *                     -> a(u,v) = int 2 mu eps(u):eps(v) + lambda div u div v
 *   Be[(a,c), b]     = -alpha |T| d_c phi_a / (d+1)   -> "-b(v,p) -> B"
 *   Le[a,b]          = |T| grad phi_a . grad phi_b    -> c(p,q)/K
 *   Me[a,b]          = |T| (1 + delta_ab) / ((d+1)(d+2))   (exact P1 mass)
 * Sizes: Ae (d(d+1))^2 row-major over (a,c); Be d(d+1) x (d+1); Le, Me (d+1)^2.
 * Returns the signed measure (<= 0 signals a degenerate / inverted cell).
 */
double oracle_element(int d, const double *X, double lam, double mu, double alpha,
                      double *Ae, double *Be, double *Le, double *Me)
{
    double g[4 * 3];
    double vol = p1_gradients(d, X, g);
    if (vol <= 0.0) return vol;
    int nv = d + 1, nu = d * nv;
    for (int a = 0; a < nv; a++)
        for (int c = 0; c < d; c++)
            for (int b = 0; b < nv; b++)
                for (int e = 0; e < d; e++) {
                    double gg = 0.0;
                    for (int k = 0; k < d; k++) gg += g[a * d + k] * g[b * d + k];
                    double v = mu * gg * (c == e ? 1.0 : 0.0)
                             + mu * g[a * d + e] * g[b * d + c]
                             + lam * g[a * d + c] * g[b * d + e];
                    Ae[(a * d + c) * nu + (b * d + e)] = vol * v;
                }
    for (int a = 0; a < nv; a++)
        for (int c = 0; c < d; c++)
            for (int b = 0; b < nv; b++)
                Be[(a * d + c) * nv + b] = -alpha * vol * g[a * d + c] / (double)nv;
    for (int a = 0; a < nv; a++)
        for (int b = 0; b < nv; b++) {
            double gg = 0.0;
            for (int k = 0; k < d; k++) gg += g[a * d + k] * g[b * d + k];
            Le[a * nv + b] = vol * gg;
            Me[a * nv + b] = vol * (a == b ? 2.0 : 1.0) / (double)(nv * (nv + 1));
        }
    return vol;
}

/*
 * Global assembly into COO triplets (duplicates are summed by the caller).
 * Global indices: u dof = node*d + c, p dof = node.  Per element it emits
 * (d(d+1))^2 entries of A, d(d+1)^2 of B (row u, col p), and (d+1)^2 each of
 * L, C (= kappa_e L_e, R9) and M.  Returns 0, or 1 + index of the first
 * degenerate cell.
 */
int64_t oracle_assemble(int d, int64_t n_nodes, const double *coords, int64_t n_cells,
                        const int32_t *cells, double lam, double mu, double alpha,
                        const double *kappa,
                        int64_t *Ai, int64_t *Aj, double *Av,
                        int64_t *Bi, int64_t *Bj, double *Bv,
                        int64_t *Pi, int64_t *Pj, double *Lv, double *Cv, double *Mv)
{
    (void)n_nodes;
    int nv = d + 1, nu = d * nv;
    int64_t na = (int64_t)nu * nu, nb = (int64_t)nu * nv, np = (int64_t)nv * nv;
    for (int64_t e = 0; e < n_cells; e++) {
        double X[4 * 3], Ae[144], Be[48], Le[16], Me[16];
        const int32_t *cn = cells + e * nv;
        for (int a = 0; a < nv; a++)
            for (int k = 0; k < d; k++) X[a * d + k] = coords[(int64_t)cn[a] * d + k];
        double vol = oracle_element(d, X, lam, mu, alpha, Ae, Be, Le, Me);
        if (vol <= 0.0) return e + 1;
        for (int r = 0; r < nu; r++)
            for (int s = 0; s < nu; s++) {
                int64_t k = e * na + r * nu + s;
                Ai[k] = (int64_t)cn[r / d] * d + r % d;
                Aj[k] = (int64_t)cn[s / d] * d + s % d;
                Av[k] = Ae[r * nu + s];
            }
        for (int r = 0; r < nu; r++)
            for (int b = 0; b < nv; b++) {
                int64_t k = e * nb + r * nv + b;
                Bi[k] = (int64_t)cn[r / d] * d + r % d;
                Bj[k] = cn[b];
                Bv[k] = Be[r * nv + b];
            }
        for (int a = 0; a < nv; a++)
            for (int b = 0; b < nv; b++) {
                int64_t k = e * np + a * nv + b;
                Pi[k] = cn[a];
                Pj[k] = cn[b];
                Lv[k] = Le[a * nv + b];
                Cv[k] = kappa[e] * Le[a * nv + b];
                Mv[k] = Me[a * nv + b];
            }
    }
    return 0;
}

/* y = M x for CSR M (plain row loop). */
static void csr_mv(int64_t nrows, const int64_t *rp, const int32_t *ci, const double *v,
                   const double *x, double *y)
{
    for (int64_t i = 0; i < nrows; i++) {
        double s = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; k++) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

/*
 * Residual of step n (Alg. 2 lines 1-2, Jacobi form R4):
 *   r = A' x_prev + f^n - AA x_cur,   f^n = sum_{j<J} s[j][n-1] F[j]
 * with AA = [[A, B], [B^T, -(S M + tau C + beta L)]] and
 * A' = [[0, 0], [B^T, -(S M + beta L)]] (eqs. fullysystem/axb, P:L156-231,
 * R8/R9), both already restricted to free DoFs by the caller (R11).  The load
 * f^n ("f^m") is a sum of J fixed vectors with per-step coefficients:
 * J = 1 is the traction load s_n F (R16); §4.1's sources and Dirichlet lifting
 * add terms (R24).  F is [J][ndof], s is [J][nt].
 */
static void step_residual(int64_t ndof, int32_t J, int32_t nt, int32_t n,
                          const int64_t *Arp, const int32_t *Aci, const double *Av,
                          const int64_t *Prp, const int32_t *Pci, const double *Pv,
                          const double *F, const double *s, const double *x_prev,
                          const double *x_cur, double *r, double *tmp)
{
    csr_mv(ndof, Prp, Pci, Pv, x_prev, r);        /* A' x_{n-1} */
    csr_mv(ndof, Arp, Aci, Av, x_cur, tmp);       /* AA x_n     */
    for (int64_t i = 0; i < ndof; i++) {
        double f = 0.0;
        for (int32_t j = 0; j < J; j++) f += s[(size_t)j * nt + (n - 1)] * F[(size_t)j * ndof + i];
        r[i] = r[i] + f - tmp[i];
    }
}

/*
 * Preconditioner application z = P^{-1} r (eqs. p1/p2 with the
 * approximate Schur complement; readings R2: A^{-1} and S~p^{-1} realised by
 * their diagonals, DAinv / DSinv = 1/diag on free DoFs and 0 on fixed ones).
 *   P~2 = [[A,0],[0,-S~p]]:    z_u = A^{-1} r_u,  z_p = -S~p^{-1} r_p
 *   P~1 = [[A,0],[B^T,-S~p]]:  z_u = A^{-1} r_u,  z_p =  S~p^{-1} (B^T z_u - r_p)
 * BT is the (np x nu) block B^T of AA (free DoFs only).
 */
static void apply_precond(int precond, int64_t nu, int64_t np, const double *DAinv,
                          const double *DSinv, const int64_t *Brp, const int32_t *Bci,
                          const double *Bv, const double *r, double *z, double *tmp)
{
    for (int64_t i = 0; i < nu; i++) z[i] = DAinv[i] * r[i];
    if (precond == 2) {
        for (int64_t q = 0; q < np; q++) z[nu + q] = -DSinv[q] * r[nu + q];
    } else {
        csr_mv(np, Brp, Bci, Bv, z, tmp);          /* B^T z_u (z_u = first nu entries) */
        for (int64_t q = 0; q < np; q++) z[nu + q] = DSinv[q] * (tmp[q] - r[nu + q]);
    }
}

/*
 * K outer iterations of the inverted time-stepping method over all steps at
 * once, Jacobi in time (Alg. 2; BJ north star; R1, R3, R4):
 *   for k: for n = 1..nt (independent, may run in parallel):
 *       r_n = A' x_{n-1}^k + f^n - AA x_n^k       (f^n as in step_residual)
 *       x_n^{k+1} = x_n^k + omega P^{-1} r_n
 * X holds rows 0..nt of length ndof; row 0 (x_0, or a window's ghost step)
 * is never updated.  hist (optional) receives ||r_{n,u}||_2, ||r_{n,p}||_2 of
 * the residual at x^k, laid out [k][n-1][2] (R12).  Returns 0 or -1 (OOM).
 */
int oracle_iterate(int64_t nu, int64_t np, int32_t nt, int32_t K,
                   const int64_t *Arp, const int32_t *Aci, const double *Av,
                   const int64_t *Prp, const int32_t *Pci, const double *Pv,
                   const int64_t *Brp, const int32_t *Bci, const double *Bv,
                   int32_t J, const double *F, const double *s, const double *DAinv, const double *DSinv,
                   int32_t precond, double omega, double *X, double *hist, int32_t nthreads)
{
    int64_t ndof = nu + np;
    double *Y = (double *)malloc(sizeof(double) * (size_t)(nt + 1) * (size_t)ndof);
    if (!Y) return -1;
    memcpy(Y, X, sizeof(double) * (size_t)ndof);      /* row 0 is fixed */
    double *cur = X, *nxt = Y;
    int fail = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (int32_t k = 0; k < K; k++) {
#pragma omp parallel
        {
            double *r = (double *)malloc(sizeof(double) * (size_t)ndof);
            double *z = (double *)malloc(sizeof(double) * (size_t)ndof);
            double *t = (double *)malloc(sizeof(double) * (size_t)ndof);
            if (!r || !z || !t) {
#pragma omp atomic write
                fail = 1;
            } else {
#pragma omp for schedule(static)
                for (int32_t n = 1; n <= nt; n++) {
                    const double *xp = cur + (size_t)(n - 1) * ndof;
                    const double *xc = cur + (size_t)n * ndof;
                    double *xn = nxt + (size_t)n * ndof;
                    step_residual(ndof, J, nt, n, Arp, Aci, Av, Prp, Pci, Pv, F, s, xp, xc, r, t);
                    apply_precond(precond, nu, np, DAinv, DSinv, Brp, Bci, Bv, r, z, t);
                    for (int64_t i = 0; i < ndof; i++) xn[i] = xc[i] + omega * z[i];
                    if (hist) {
                        double su = 0.0, sp = 0.0;
                        for (int64_t i = 0; i < nu; i++) su += r[i] * r[i];
                        for (int64_t i = nu; i < ndof; i++) sp += r[i] * r[i];
                        hist[((size_t)k * nt + (n - 1)) * 2 + 0] = sqrt(su);
                        hist[((size_t)k * nt + (n - 1)) * 2 + 1] = sqrt(sp);
                    }
                }
            }
            free(r); free(z); free(t);
        }
        if (fail) break;
        double *sw = cur; cur = nxt; nxt = sw;
    }
    if (cur != X) memcpy(X + ndof, cur + ndof, sizeof(double) * (size_t)nt * (size_t)ndof);
    free(Y);
    return fail ? -1 : 0;
}

/*
 * Residual norms at the current iterate without updating it (R12):
 * out[n-1][0..1] = ||r_{n,u}||_2, ||r_{n,p}||_2, r as in step_residual.
 */
int oracle_residual_norms(int64_t nu, int64_t np, int32_t nt,
                          const int64_t *Arp, const int32_t *Aci, const double *Av,
                          const int64_t *Prp, const int32_t *Pci, const double *Pv,
                          int32_t J, const double *F, const double *s, const double *X, double *out,
                          double *r_out, int32_t nthreads)
{
    int64_t ndof = nu + np;
    int fail = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        double *r = (double *)malloc(sizeof(double) * (size_t)ndof);
        double *t = (double *)malloc(sizeof(double) * (size_t)ndof);
        if (!r || !t) {
#pragma omp atomic write
            fail = 1;
        } else {
#pragma omp for schedule(static)
            for (int32_t n = 1; n <= nt; n++) {
                step_residual(ndof, J, nt, n, Arp, Aci, Av, Prp, Pci, Pv, F, s,
                              X + (size_t)(n - 1) * ndof, X + (size_t)n * ndof, r, t);
                double su = 0.0, sp = 0.0;
                for (int64_t i = 0; i < nu; i++) su += r[i] * r[i];
                for (int64_t i = nu; i < ndof; i++) sp += r[i] * r[i];
                out[(size_t)(n - 1) * 2 + 0] = sqrt(su);
                out[(size_t)(n - 1) * 2 + 1] = sqrt(sp);
                if (r_out) memcpy(r_out + (size_t)(n - 1) * ndof, r, sizeof(double) * (size_t)ndof);
            }
        }
        free(r); free(t);
    }
    return fail ? -1 : 0;
}
