/*
 * ldu_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded fp64 CPU reference
 * for the hot path of arXiv 1505.07630 (AlOnazi, Keyes, Lastovetsky, Rychkov, ParCFD 2014).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no code, header, table or helper with the CUDA library in
 * paper_1505_07630_b200/ and never calls it; the product path never calls this.
 *
 * Built with:  gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC  (no OpenMP, no FMA
 * contraction), so every operation is an IEEE fp64 round-to-nearest op in source order.
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n; "SURVEY §8(c) cK" = the step-by-step
 * algorithm transcribed in SURVEY.md §8(c); readings Z1..Z23 are listed in DESIGN.md.
 *
 * What each function follows:
 *   oracle_amul      SpMV y = A x, OpenFOAM lduMatrix::Amul face loop ("sparse matrix vector
 *                    multiply kernel"; P:206 lduMatrix).  Pinned by tests against
 *                    a dense numpy mat-vec, worked examples S:42-43, closed-form eigenpairs.
 *   oracle_iface     processor-interface update y[fc[i]] -= coeff[i]*x_nbr[i] (P:79, P:81 halo
 *                    layer; reading Z10).  Pinned by slab-reconstruction tests.
 *   oracle_pcg       Jacobi-preconditioned CG (Eq 4).  Pinned by
 *                    dense Cholesky, n-step termination, closed-form eigen RHS,
 *                    manufactured solutions, A-norm monotonicity, Table 2 128^3/64^3 ratio.
 *   oracle_pipecg    Ghysels-Vanroose pipelined CG, literal
 *                    form (mode 0, u, q, m stored) and Jacobi-specialised form (mode 1, u = rD*r,
 *                    q = rD*s, m = rD*w never stored).  Pinned by iterate-wise equality with
 *                    oracle_pcg and the same solution pins.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_NOT_CONVERGED = 1, OR_BREAKDOWN = 2, OR_ERR_ARG = -1 };
enum { OR_NORM_L2 = 0, OR_NORM_OPENFOAM = 1 };

/* ---- SpMV ------------------------------------------------------------------------------- */

/* y = A x.  A[c][c] = diag[c]; A[l[f]][u[f]] = upper[f]; A[u[f]][l[f]] = lower[f] (lower == NULL
 * means symmetric, lower := upper; reading Z10).  Face loop in face order. */
void oracle_amul(int n, int nf, const int *l, const int *u, const double *diag,
                 const double *lower, const double *upper, const double *x, double *y)
{
    const double *lo = lower ? lower : upper;
    for (int c = 0; c < n; ++c) y[c] = diag[c] * x[c];
    for (int f = 0; f < nf; ++f) {
        y[u[f]] += lo[f] * x[l[f]];
        y[l[f]] += upper[f] * x[u[f]];
    }
}

/* Interface update: y[fc[i]] -= coeff[i] * xnbr[i], faces in order (readings Z10, Z23). */
void oracle_iface(int nfc, const int *fc, const double *coeff, const double *xnbr, double *y)
{
    for (int i = 0; i < nfc; ++i) y[fc[i]] -= coeff[i] * xnbr[i];
}

/* ---- helpers (plain loops, sequential summation order) ----------------------------------- */

static double dot(int n, const double *a, const double *b)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static double sum_abs(int n, const double *a)
{
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += fabs(a[i]);
    return s;
}

typedef struct {
    int n, nf;
    const int *l, *u;
    const double *diag, *lower, *upper;
} ldu_t;

static void amul(const ldu_t *A, const double *x, double *y)
{
    oracle_amul(A->n, A->nf, A->l, A->u, A->diag, A->lower, A->upper, x, y);
}

/* Convergence criterion (reading Z1).
 * OR_NORM_L2:       res = ||r||_2 / ||b||_2.
 * OR_NORM_OPENFOAM: res = sum|r| / normFactor, normFactor = sum|A x0 - xbar sumA| +
 *                   sum|b - xbar sumA| + 1e-20, xbar = mean(x0), sumA = A * 1. */
typedef struct { int norm; double scale; } crit_t;

static int crit_init(const ldu_t *A, int norm, const double *b, const double *x0,
                     const double *Ax0, crit_t *cr)
{
    int n = A->n;
    cr->norm = norm;
    if (norm == OR_NORM_L2) {
        cr->scale = sqrt(dot(n, b, b));
        return 0;
    }
    if (norm != OR_NORM_OPENFOAM) return -1;
    double *one = malloc(sizeof(double) * (size_t)n), *sumA = malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) one[i] = 1.0;
    amul(A, one, sumA);
    double xbar = 0.0;
    for (int i = 0; i < n; ++i) xbar += x0[i];
    xbar /= (double)n;
    double nf = 0.0;
    for (int i = 0; i < n; ++i) nf += fabs(Ax0[i] - xbar * sumA[i]) + fabs(b[i] - xbar * sumA[i]);
    cr->scale = nf + 1e-20;
    free(one);
    free(sumA);
    return 0;
}

static double crit_eval(const crit_t *cr, int n, const double *r)
{
    if (cr->norm == OR_NORM_L2) return sqrt(dot(n, r, r)) / cr->scale;
    return sum_abs(n, r) / cr->scale;
}

/* Stopping test (readings Z2, Z2', Z26): after `it` x-updates the solve stops when it >= minIter
 * and (res < tol, or r is exactly zero, or relTol > 0 and res < relTol * res0) -- OpenFOAM's
 * checkConvergence with its relTol and minIter controls. */
typedef struct { double tol, relTol, res0; int minIter; } stop_t;
static int converged(const stop_t *sp, double res, int it)
{
    if (it < sp->minIter) return 0;
    return res < sp->tol || res == 0.0 || (sp->relTol > 0.0 && res < sp->relTol * sp->res0);
}

/* ---- classical Jacobi-PCG (OpenFOAM PCG order) -------------------------- */

int oracle_pcg(int n, int nf, const int *l, const int *u, const double *diag,
               const double *lower, const double *upper, const double *b, double *x,
               double tol, int maxIter, int norm, int *nIter, double *finalRes, double *hist,
               double relTol, int minIter)
{
    if (n <= 0 || nf < 0 || maxIter < 0 || !b || !x || !diag || relTol < 0 || minIter < 0)
        return OR_ERR_ARG;
    stop_t sp = {tol, relTol, 0.0, minIter};
    ldu_t A = {n, nf, l, u, diag, lower, upper};
    size_t bytes = sizeof(double) * (size_t)n;
    double *r = malloc(bytes), *z = malloc(bytes), *p = malloc(bytes), *q = malloc(bytes);
    double *rD = malloc(bytes);
    int status = OR_NOT_CONVERGED;
    for (int c = 0; c < n; ++c) rD[c] = 1.0 / diag[c]; /* DiagonalPreconditioner */

    amul(&A, x, q);                                     /* r = b - A x */
    for (int c = 0; c < n; ++c) r[c] = b[c] - q[c];
    crit_t cr;
    if (crit_init(&A, norm, b, x, q, &cr)) { status = OR_ERR_ARG; goto out; }
    if (norm == OR_NORM_L2 && cr.scale == 0.0) {        /* b = 0: x = 0 (reading Z1) */
        for (int c = 0; c < n; ++c) x[c] = 0.0;
        *nIter = 0; *finalRes = 0.0;
        if (hist) hist[0] = 0.0;
        status = OR_OK;
        goto out;
    }
    double res = crit_eval(&cr, n, r);
    sp.res0 = res;
    if (hist) hist[0] = res;
    *nIter = 0; *finalRes = res;
    if (converged(&sp, res, 0)) { status = OR_OK; goto out; }

    double rho_old = 0.0;
    for (int k = 0; k < maxIter; ++k) {
        for (int c = 0; c < n; ++c) z[c] = rD[c] * r[c];     /* z = M^-1 r */
        double rho = dot(n, z, r);                            /* rho = (z, r) */
        if (k == 0) {
            for (int c = 0; c < n; ++c) p[c] = z[c];
        } else {
            double beta = rho / rho_old;
            for (int c = 0; c < n; ++c) p[c] = z[c] + beta * p[c];
        }
        amul(&A, p, q);                                       /* q = A p */
        double pq = dot(n, p, q);
        if (!(pq > 0.0) || !isfinite(pq)) {                   /* reading Z19 */
            *nIter = k; status = OR_BREAKDOWN; goto out;
        }
        double alpha = rho / pq;
        for (int c = 0; c < n; ++c) x[c] += alpha * p[c];
        for (int c = 0; c < n; ++c) r[c] -= alpha * q[c];
        res = crit_eval(&cr, n, r);
        *nIter = k + 1; *finalRes = res;
        if (hist) hist[k + 1] = res;
        if (converged(&sp, res, k + 1)) { status = OR_OK; goto out; }
        rho_old = rho;
    }
    status = OR_NOT_CONVERGED;
out:
    free(r); free(z); free(p); free(q); free(rD);
    return status;
}

/* ---- pipelined CG, Ghysels & Vanroose Alg. 4 with M = diag ------------- */

int oracle_pipecg(int n, int nf, const int *l, const int *u, const double *diag,
                  const double *lower, const double *upper, const double *b, double *x,
                  double tol, int maxIter, int norm, int mode, int *nIter, double *finalRes,
                  double *hist, double relTol, int minIter)
{
    if (n <= 0 || nf < 0 || maxIter < 0 || !b || !x || !diag || (mode != 0 && mode != 1) ||
        relTol < 0 || minIter < 0)
        return OR_ERR_ARG;
    stop_t sp = {tol, relTol, 0.0, minIter};
    ldu_t A = {n, nf, l, u, diag, lower, upper};
    size_t bytes = sizeof(double) * (size_t)n;
    double *r = malloc(bytes), *uu = malloc(bytes), *w = malloc(bytes), *m = malloc(bytes);
    double *nn = malloc(bytes), *z = malloc(bytes), *q = malloc(bytes), *s = malloc(bytes);
    double *p = malloc(bytes), *rD = malloc(bytes);
    int status = OR_NOT_CONVERGED;
    for (int c = 0; c < n; ++c) rD[c] = 1.0 / diag[c];

    amul(&A, x, w);                                           /* r = b - A x */
    for (int c = 0; c < n; ++c) r[c] = b[c] - w[c];
    crit_t cr;
    if (crit_init(&A, norm, b, x, w, &cr)) { status = OR_ERR_ARG; goto out; }
    if (norm == OR_NORM_L2 && cr.scale == 0.0) {
        for (int c = 0; c < n; ++c) x[c] = 0.0;
        *nIter = 0; *finalRes = 0.0;
        if (hist) hist[0] = 0.0;
        status = OR_OK;
        goto out;
    }
    for (int c = 0; c < n; ++c) uu[c] = rD[c] * r[c];        /* u = M^-1 r */
    amul(&A, uu, w);                                          /* w = A u */

    double gamma_old = 0.0, alpha_old = 0.0;
    for (int i = 0; i <= maxIter; ++i) {
        /* the single fused reduction: gamma = (r,u), delta = (w,u), res = crit(r) */
        if (mode == 1)
            for (int c = 0; c < n; ++c) uu[c] = rD[c] * r[c];
        double gamma = dot(n, r, uu);
        double delta = dot(n, w, uu);
        double res = crit_eval(&cr, n, r);
        if (i == 0) sp.res0 = res;
        if (hist) hist[i] = res;
        *nIter = i; *finalRes = res;
        if (converged(&sp, res, i)) { status = OR_OK; goto out; }
        if (i == maxIter) { status = OR_NOT_CONVERGED; goto out; }

        for (int c = 0; c < n; ++c) m[c] = rD[c] * w[c];      /* m = M^-1 w */
        amul(&A, m, nn);                                      /* n = A m */
        double alpha, beta;
        if (i == 0) {
            beta = 0.0;
            if (!(delta > 0.0) || !isfinite(delta)) { status = OR_BREAKDOWN; goto out; }
            alpha = gamma / delta;
        } else {
            beta = gamma / gamma_old;
            double den = delta - beta * gamma / alpha_old;
            if (!(den > 0.0) || !isfinite(den)) { status = OR_BREAKDOWN; goto out; }
            alpha = gamma / den;
        }
        if (i == 0) {
            for (int c = 0; c < n; ++c) {
                z[c] = nn[c]; q[c] = m[c]; s[c] = w[c]; p[c] = uu[c];
            }
        } else {
            for (int c = 0; c < n; ++c) {
                z[c] = nn[c] + beta * z[c];
                q[c] = m[c] + beta * q[c];
                s[c] = w[c] + beta * s[c];
                p[c] = uu[c] + beta * p[c];
            }
        }
        for (int c = 0; c < n; ++c) {
            x[c] += alpha * p[c];
            r[c] -= alpha * s[c];
            if (mode == 0) uu[c] -= alpha * q[c];
            w[c] -= alpha * z[c];
        }
        gamma_old = gamma;
        alpha_old = alpha;
    }
out:
    free(r); free(uu); free(w); free(m); free(nn); free(z); free(q); free(s); free(p); free(rD);
    return status;
}
