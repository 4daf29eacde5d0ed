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
 *   oracle_dic,      OpenFOAM DIC preconditioner and DIC-(Pipe)CG (readings
 *   oracle_dic_pcg   Z35-Z36).  Pinned by tests/test_oracle_dic.py: diag(M) = diag(A), IC(0) on
 *                    hex meshes, exact Cholesky on a chain, dense M w = r, dense solves.
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

/* Optional preconditioner z = M^-1 r (NULL => Jacobi, z = r / diag).  Used by the AMG
 * V-cycle below (NEXT-2). */
typedef struct { void (*apply)(const void *ctx, const double *r, double *z); const void *ctx; } prec_t;

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

static int pcg_core(int n, int nf, const int *l, const int *u, const double *diag,
                    const double *lower, const double *upper, const double *b, double *x,
                    double tol, int maxIter, int norm, int *nIter, double *finalRes, double *hist,
                    double relTol, int minIter, const prec_t *M)
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
        if (M) M->apply(M->ctx, r, z);                        /* z = M^-1 r */
        else for (int c = 0; c < n; ++c) z[c] = rD[c] * r[c];
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

int oracle_pcg(int n, int nf, const int *l, const int *u, const double *diag,
               const double *lower, const double *upper, const double *b, double *x,
               double tol, int maxIter, int norm, int *nIter, double *finalRes, double *hist,
               double relTol, int minIter)
{
    return pcg_core(n, nf, l, u, diag, lower, upper, b, x, tol, maxIter, norm, nIter, finalRes,
                    hist, relTol, minIter, NULL);
}

/* ---- pipelined CG, Ghysels & Vanroose Alg. 4 with M = diag ------------- */

/* replaceEvery > 0 (NEXT-4, residual replacement; Ghysels & Vanroose 2014, Sec. 4 [ext]): after
 * the updates of every iteration i with (i + 1) % replaceEvery == 0 the recurrence vectors are
 * recomputed from their definitions -- r = b - A x, u = M r, w = A u, s = A p, q = M s,
 * z = A q -- before the next fused reduction.  Equal iterates in exact arithmetic. */
static int pipecg_core(int n, int nf, const int *l, const int *u, const double *diag,
                       const double *lower, const double *upper, const double *b, double *x,
                       double tol, int maxIter, int norm, int mode, int *nIter, double *finalRes,
                       double *hist, double relTol, int minIter, const prec_t *M,
                       int replaceEvery)
{
    if (n <= 0 || nf < 0 || maxIter < 0 || !b || !x || !diag || (mode != 0 && mode != 1) ||
        relTol < 0 || minIter < 0 || (M && mode != 0))
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
    if (M) M->apply(M->ctx, r, uu);                           /* u = M^-1 r */
    else for (int c = 0; c < n; ++c) uu[c] = rD[c] * r[c];
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

        if (M) M->apply(M->ctx, w, m);                        /* m = M^-1 w */
        else for (int c = 0; c < n; ++c) m[c] = rD[c] * w[c];
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
        if (replaceEvery > 0 && (i + 1) % replaceEvery == 0) {   /* residual replacement */
            amul(&A, x, nn);
            for (int c = 0; c < n; ++c) r[c] = b[c] - nn[c];        /* r = b - A x          */
            if (M) M->apply(M->ctx, r, uu);                          /* u = M r              */
            else for (int c = 0; c < n; ++c) uu[c] = rD[c] * r[c];
            amul(&A, uu, w);                                         /* w = A u              */
            amul(&A, p, s);                                          /* s = A p              */
            if (M) M->apply(M->ctx, s, q);                           /* q = M s              */
            else for (int c = 0; c < n; ++c) q[c] = rD[c] * s[c];
            amul(&A, q, z);                                          /* z = A q              */
        }
    }
out:
    free(r); free(uu); free(w); free(m); free(nn); free(z); free(q); free(s); free(p); free(rD);
    return status;
}

int oracle_pipecg(int n, int nf, const int *l, const int *u, const double *diag,
                  const double *lower, const double *upper, const double *b, double *x,
                  double tol, int maxIter, int norm, int mode, int *nIter, double *finalRes,
                  double *hist, double relTol, int minIter)
{
    return pipecg_core(n, nf, l, u, diag, lower, upper, b, x, tol, maxIter, norm, mode, nIter,
                       finalRes, hist, relTol, minIter, NULL, 0);
}

/* pipelined CG with residual replacement every replaceEvery iterations (NEXT-4) */
int oracle_pipecg_rr(int n, int nf, const int *l, const int *u, const double *diag,
                     const double *lower, const double *upper, const double *b, double *x,
                     double tol, int maxIter, int norm, int mode, int *nIter, double *finalRes,
                     double *hist, double relTol, int minIter, int replaceEvery)
{
    if (replaceEvery < 0) return OR_ERR_ARG;
    return pipecg_core(n, nf, l, u, diag, lower, upper, b, x, tol, maxIter, norm, mode, nIter,
                       finalRes, hist, relTol, minIter, NULL, replaceEvery);
}

/* ==== Aggregation AMG preconditioner (NEXT-2; Table 2) =====================
 *
 * The paper preconditions its CG and pipelined CG with CUSP's aggregation AMG: "a V-cycle of an
 * aggregation-based AMG with weighted Jacobi iterations with omega = 4/3 as a smoother", the
 * aggregates coming from "the parallel aggregation method based on a distance-2
 * maximal-independent-set".  Readings Z27-Z33 fix what the paper leaves open:
 * smoothed aggregation P = (I - w D^-1 A) T with w = (4/3)/rho, rho = 1.05 x the largest Ritz
 * value of 20 Lanczos steps on D^-1/2 A D^-1/2 (oracle/amg.py spectral_radius; reading Z27);
 * all couplings strong; one pre- and one post-sweep of w-Jacobi from a zero guess; MIS-2 in the
 * priority order key(i) below; Galerkin A_c = P^T A P; coarsest level solved exactly (Cholesky).
 * The hierarchy products are built by oracle/amg.py (scipy); this file holds the integer
 * aggregation and the V-cycle arithmetic. */

typedef struct { int n; const int *ptr; const int *col; const double *val; } csr_t;

/* y = A x for a CSR matrix, row by row in stored column order. */
static void csr_mv(const csr_t *A, const double *x, double *y)
{
    for (int i = 0; i < A->n; ++i) {
        double s = 0.0;
        for (int k = A->ptr[i]; k < A->ptr[i + 1]; ++k) s += A->val[k] * x[A->col[k]];
        y[i] = s;
    }
}

/* Priority key of node i (reading Z30): keyMode 0 = the index itself (lowest index first);
 * keyMode 1 = (mix32(i) << 32) | i with the "lowbias32" integer mixer, a fixed pseudo-random order
 * that keeps the parallel MIS rounds few on structured meshes.  Unique by construction. */
static unsigned long long amg_key(int i, int keyMode)
{
    if (keyMode == 0) return (unsigned long long)(unsigned)i;
    unsigned h = (unsigned)i;
    h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
    return ((unsigned long long)h << 32) | (unsigned)i;
}

typedef struct { unsigned long long key; int i; } keyed_t;
static int cmp_keyed(const void *a, const void *b)
{
    unsigned long long x = ((const keyed_t *)a)->key, y = ((const keyed_t *)b)->key;
    return x < y ? -1 : x > y;
}

/* Distance-2 MIS aggregation (reading Z30) on the graph of A (off-diagonal entries of the
 * CSR pattern; values ignored, all couplings strong -- reading Z29).
 *   1. roots: visit nodes in increasing key; a node becomes a root if no root lies within graph
 *      distance <= 2 (the greedy = lexicographically-first MIS of the distance-2 graph).
 *   2. aggregates are numbered by increasing root index.
 *   3. a non-root adjacent to >= 1 root joins the adjacent root with the smallest key.
 *   4. every other node (distance exactly 2 from a root) joins the aggregate of its adjacent
 *      step-3 node with the smallest key.
 * Writes agg[n]; returns the number of aggregates (or -1 on bad arguments). */
int oracle_mis2_aggregate(int n, const int *ptr, const int *col, int keyMode, int *agg)
{
    if (n <= 0 || !ptr || !col || !agg || (keyMode != 0 && keyMode != 1)) return -1;
    keyed_t *ord = malloc(sizeof(keyed_t) * (size_t)n);
    char *root = calloc((size_t)n, 1);
    for (int i = 0; i < n; ++i) { ord[i].key = amg_key(i, keyMode); ord[i].i = i; }
    qsort(ord, (size_t)n, sizeof(keyed_t), cmp_keyed);
    for (int t = 0; t < n; ++t) {                          /* step 1 */
        int i = ord[t].i, ok = 1;
        for (int k = ptr[i]; k < ptr[i + 1] && ok; ++k) {
            int j = col[k];
            if (j == i) continue;
            if (root[j]) ok = 0;
            for (int k2 = ptr[j]; k2 < ptr[j + 1] && ok; ++k2)
                if (col[k2] != i && root[col[k2]]) ok = 0;
        }
        root[i] = (char)ok;
    }
    int na = 0;
    for (int i = 0; i < n; ++i) agg[i] = root[i] ? na++ : -1;   /* step 2 */
    int *a1 = malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) {                          /* step 3 */
        a1[i] = agg[i];
        if (root[i]) continue;
        unsigned long long best = ~0ULL;
        for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
            int j = col[k];
            if (j != i && root[j] && amg_key(j, keyMode) < best) { best = amg_key(j, keyMode); a1[i] = agg[j]; }
        }
    }
    for (int i = 0; i < n; ++i) {                          /* step 4 */
        int a = a1[i];
        if (a < 0) {
            unsigned long long best = ~0ULL;
            for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
                int j = col[k];
                if (j != i && a1[j] >= 0 && amg_key(j, keyMode) < best) { best = amg_key(j, keyMode); a = a1[j]; }
            }
        }
        agg[i] = a;                                        /* -1 only if isolated from all roots */
    }
    free(a1); free(root); free(ord);
    return na;
}

/* One AMG hierarchy as handed over by oracle/amg.py.  Level l < L has A_l, P_l (n_l x n_{l+1}),
 * R_l = P_l^T, rD_l = 1/diag(A_l) and the Jacobi weight w_l; the coarsest matrix (size nc) comes
 * as its dense lower Cholesky factor Lc (row-major), A_L = Lc Lc^T. */
typedef struct {
    int L, nc;
    const csr_t *A, *P, *R;
    const double *const *rD;
    const double *omega;
    const double *Lc;
} amg_t;

/* z = A_L^-1 f by forward and back substitution with the Cholesky factor (reading Z31). */
static void chol_solve(int n, const double *Lc, const double *f, double *z)
{
    for (int i = 0; i < n; ++i) {
        double s = f[i];
        for (int k = 0; k < i; ++k) s -= Lc[(size_t)i * n + k] * z[k];
        z[i] = s / Lc[(size_t)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = z[i];
        for (int k = i + 1; k < n; ++k) s -= Lc[(size_t)k * n + i] * z[k];
        z[i] = s / Lc[(size_t)i * n + i];
    }
}

/* V-cycle z = B_l f (reading Z32): zero initial guess, one w-Jacobi pre-sweep, residual,
 * restriction f_c = R r, recursion, prolongation x += P x_c, one w-Jacobi post-sweep. */
static void vcycle(const amg_t *H, int l, const double *f, double *z)
{
    if (l == H->L) { chol_solve(H->nc, H->Lc, f, z); return; }
    const csr_t *A = &H->A[l];
    int n = A->n, nc = H->R[l].n;
    const double w = H->omega[l], *rD = H->rD[l];
    double *x = calloc((size_t)n, sizeof(double)), *r = calloc((size_t)n, sizeof(double));
    double *fc = malloc(sizeof(double) * (size_t)nc), *xc = malloc(sizeof(double) * (size_t)nc);
    double *px = malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) x[i] = w * rD[i] * f[i];        /* pre-sweep from x = 0 */
    csr_mv(A, x, r);
    for (int i = 0; i < n; ++i) r[i] = f[i] - r[i];             /* r = f - A x */
    csr_mv(&H->R[l], r, fc);                                    /* f_c = R r */
    vcycle(H, l + 1, fc, xc);
    csr_mv(&H->P[l], xc, px);
    for (int i = 0; i < n; ++i) x[i] += px[i];                  /* x += P x_c */
    csr_mv(A, x, r);
    for (int i = 0; i < n; ++i) z[i] = x[i] + w * rD[i] * (f[i] - r[i]);   /* post-sweep */
    free(x); free(r); free(fc); free(xc); free(px);
}

static void amg_apply(const void *ctx, const double *r, double *z) { vcycle((const amg_t *)ctx, 0, r, z); }

/* Flat hand-over from Python: per level l < L the CSR arrays of A_l, P_l, R_l, rD_l, omega_l. */
typedef struct {
    int L, nc;
    const int *n;                          /* [L]   rows of A_l                                 */
    const int *const *Aptr, *const *Acol; const double *const *Aval;
    const int *const *Pptr, *const *Pcol; const double *const *Pval;
    const int *const *Rptr, *const *Rcol; const double *const *Rval;
    const int *nR;                         /* [L]   rows of R_l = n_{l+1}                       */
    const double *const *rD;
    const double *omega;
    const double *Lc;
} amg_flat_t;

static amg_t amg_unflatten(const amg_flat_t *F, csr_t *buf)
{
    csr_t *A = buf, *P = buf + F->L, *R = buf + 2 * F->L;
    for (int l = 0; l < F->L; ++l) {
        A[l] = (csr_t){F->n[l], F->Aptr[l], F->Acol[l], F->Aval[l]};
        P[l] = (csr_t){F->n[l], F->Pptr[l], F->Pcol[l], F->Pval[l]};
        R[l] = (csr_t){F->nR[l], F->Rptr[l], F->Rcol[l], F->Rval[l]};
    }
    amg_t H = {F->L, F->nc, A, P, R, F->rD, F->omega, F->Lc};
    return H;
}

/* z = B r, one V-cycle (exported for the preconditioner pins). */
void oracle_amg_vcycle(const amg_flat_t *F, const double *r, double *z)
{
    csr_t *buf = malloc(sizeof(csr_t) * (size_t)(3 * F->L + 1));
    amg_t H = amg_unflatten(F, buf);
    vcycle(&H, 0, r, z);
    free(buf);
}

/* AMG-preconditioned CG (SURVEY §8(c) c2 with z = B r) and pipelined CG (c3, literal form with
 * u = B r, m = B w); same criteria and stopping rules as the Jacobi solvers above. */
int oracle_amg_pcg(int n, int nf, const int *l, const int *u, const double *diag,
                   const double *lower, const double *upper, const double *b, double *x,
                   double tol, int maxIter, int norm, int *nIter, double *finalRes, double *hist,
                   double relTol, int minIter, const amg_flat_t *F, int pipelined)
{
    if (!F || F->L < 0 || (F->L > 0 && F->n[0] != n) || (F->L == 0 && F->nc != n)) return OR_ERR_ARG;
    csr_t *buf = malloc(sizeof(csr_t) * (size_t)(3 * F->L + 1));
    amg_t H = amg_unflatten(F, buf);
    prec_t M = {amg_apply, &H};
    int st = pipelined ? pipecg_core(n, nf, l, u, diag, lower, upper, b, x, tol, maxIter, norm, 0,
                                     nIter, finalRes, hist, relTol, minIter, &M, 0)
                       : pcg_core(n, nf, l, u, diag, lower, upper, b, x, tol, maxIter, norm, nIter,
                                  finalRes, hist, relTol, minIter, &M);
    free(buf);
    return st;
}

/* ---- block-Jacobi AMG across ranks (reading Z33) -------------------------------------------
 * The distributed AMG preconditioner is block diagonal: rank g owns the contiguous rows
 * [start[g], start[g+1]) and applies one V-cycle of the hierarchy built from its LOCAL matrix
 * (interface couplings dropped).  The Krylov operator is the global matrix. */
typedef struct { int nb; const int *start; const amg_t *H; } amg_blocks_t;

static void amg_blocks_apply(const void *ctx, const double *r, double *z)
{
    const amg_blocks_t *B = (const amg_blocks_t *)ctx;
    for (int g = 0; g < B->nb; ++g)
        vcycle(&B->H[g], 0, r + B->start[g], z + B->start[g]);
}

static int amg_blocks_make(int n, int nb, const int *start, const amg_flat_t *const *F,
                           amg_t **H, csr_t ***bufs)
{
    if (nb <= 0 || !start || !F || start[0] != 0 || start[nb] != n) return -1;
    *H = malloc(sizeof(amg_t) * (size_t)nb);
    *bufs = malloc(sizeof(csr_t *) * (size_t)nb);
    for (int g = 0; g < nb; ++g) {
        const int ng = start[g + 1] - start[g];
        if (ng <= 0 || (F[g]->L > 0 && F[g]->n[0] != ng) || (F[g]->L == 0 && F[g]->nc != ng)) {
            for (int k = 0; k < g; ++k) free((*bufs)[k]);
            free(*H); free(*bufs);
            return -1;
        }
        (*bufs)[g] = malloc(sizeof(csr_t) * (size_t)(3 * F[g]->L + 1));
        (*H)[g] = amg_unflatten(F[g], (*bufs)[g]);
    }
    return 0;
}

/* z = B r with the block-diagonal preconditioner (exported for the pins). */
int oracle_amg_block_vcycle(int n, int nb, const int *start, const amg_flat_t *const *F,
                            const double *r, double *z)
{
    amg_t *H; csr_t **bufs;
    if (amg_blocks_make(n, nb, start, F, &H, &bufs)) return OR_ERR_ARG;
    amg_blocks_t B = {nb, start, H};
    amg_blocks_apply(&B, r, z);
    for (int g = 0; g < nb; ++g) free(bufs[g]);
    free(bufs); free(H);
    return OR_OK;
}

/* Block-Jacobi AMG-PCG / AMG-PipeCG on the global system (same criteria as oracle_amg_pcg). */
int oracle_amg_block_pcg(int n, int nf, const int *l, const int *u, const double *diag,
                         const double *lower, const double *upper, const double *b, double *x,
                         double tol, int maxIter, int norm, int *nIter, double *finalRes,
                         double *hist, double relTol, int minIter, int nb, const int *start,
                         const amg_flat_t *const *F, int pipelined)
{
    amg_t *H; csr_t **bufs;
    if (amg_blocks_make(n, nb, start, F, &H, &bufs)) return OR_ERR_ARG;
    amg_blocks_t B = {nb, start, H};
    prec_t M = {amg_blocks_apply, &B};
    int st = pipelined ? pipecg_core(n, nf, l, u, diag, lower, upper, b, x, tol, maxIter, norm, 0,
                                     nIter, finalRes, hist, relTol, minIter, &M, 0)
                       : pcg_core(n, nf, l, u, diag, lower, upper, b, x, tol, maxIter, norm, nIter,
                                  finalRes, hist, relTol, minIter, &M);
    for (int g = 0; g < nb; ++g) free(bufs[g]);
    free(bufs); free(H);
    return st;
}


/* ---- DIC preconditioner (OpenFOAM DICPreconditioner [ext]) -------------
 * The default preconditioner of OpenFOAM's p solve (SURVEY NEXT-1 "Optional DIC preconditioner
 * (OpenFOAM's default for p)"): diagonal-based incomplete Cholesky, M = (D + L) D^-1 (D + L^T),
 * L = strictly-lower part of A, D chosen so that diag(M) = diag(A) (reading Z35).  Written as
 * OpenFOAM's face loops over the faces in upper-triangular order (owner = min(l, u) ascending,
 * then neighbour ascending; duplicate faces merged by summing, reading Z36):
 *   calcReciprocalD:  rD = diag;  for f ascending:  rD[u_f] -= upper_f^2 / rD[l_f];  rD = 1/rD
 *   precondition:     w = rD r;   for f ascending:  w[u_f] -= rD[u_f] upper_f w[l_f];
 *                                 for f descending: w[l_f] -= rD[l_f] upper_f w[u_f]
 * Block form (reading Z33 applied to DIC): with nb > 1 contiguous row blocks [start[g],
 * start[g+1]), faces joining two blocks are dropped -- the multi-rank (processor-local) DIC.
 * Symmetric matrices only (lower == NULL). */
typedef struct { int nf; int *l, *u; double *a; double *rD; } dic_t;

static const int *g_sort_l, *g_sort_u;
static int cmp_face(const void *pa, const void *pb)
{
    int a = *(const int *)pa, b = *(const int *)pb;
    int la = g_sort_l[a] < g_sort_u[a] ? g_sort_l[a] : g_sort_u[a];
    int lb = g_sort_l[b] < g_sort_u[b] ? g_sort_l[b] : g_sort_u[b];
    int ua = g_sort_l[a] < g_sort_u[a] ? g_sort_u[a] : g_sort_l[a];
    int ub = g_sort_l[b] < g_sort_u[b] ? g_sort_u[b] : g_sort_l[b];
    if (la != lb) return la < lb ? -1 : 1;
    if (ua != ub) return ua < ub ? -1 : 1;
    return a < b ? -1 : (a > b);
}

static int block_of(int nb, const int *start, int c)
{
    int g = 0;
    while (g + 1 < nb && c >= start[g + 1]) ++g;
    return g;
}

/* Builds the upper-triangular face list and rD; returns 0, or -1 (bad args) / -2 (pivot <= 0). */
static int dic_make(int n, int nf, const int *l, const int *u, const double *diag,
                    const double *upper, int nb, const int *start, dic_t *D)
{
    if (n <= 0 || nf < 0 || !diag || (nf && (!l || !u || !upper))) return -1;
    if (nb < 1 || (nb > 1 && (!start || start[0] != 0 || start[nb] != n))) return -1;
    int *ord = malloc(sizeof(int) * (size_t)(nf + 1));
    for (int f = 0; f < nf; ++f) {
        if (l[f] < 0 || l[f] >= n || u[f] < 0 || u[f] >= n || l[f] == u[f]) { free(ord); return -1; }
        ord[f] = f;
    }
    g_sort_l = l; g_sort_u = u;
    qsort(ord, (size_t)nf, sizeof(int), cmp_face);
    D->l = malloc(sizeof(int) * (size_t)(nf + 1));
    D->u = malloc(sizeof(int) * (size_t)(nf + 1));
    D->a = malloc(sizeof(double) * (size_t)(nf + 1));
    D->rD = malloc(sizeof(double) * (size_t)n);
    int m = 0;
    for (int k = 0; k < nf; ++k) {
        int f = ord[k];
        int lo = l[f] < u[f] ? l[f] : u[f], hi = l[f] < u[f] ? u[f] : l[f];
        if (nb > 1 && block_of(nb, start, lo) != block_of(nb, start, hi)) continue;
        if (m > 0 && D->l[m - 1] == lo && D->u[m - 1] == hi) { D->a[m - 1] += upper[f]; continue; }
        D->l[m] = lo; D->u[m] = hi; D->a[m] = upper[f]; ++m;
    }
    D->nf = m;
    free(ord);
    for (int c = 0; c < n; ++c) D->rD[c] = diag[c];                   /* calcReciprocalD */
    for (int f = 0; f < m; ++f) D->rD[D->u[f]] -= D->a[f] * D->a[f] / D->rD[D->l[f]];
    for (int c = 0; c < n; ++c) {
        if (!(D->rD[c] > 0.0) || !isfinite(D->rD[c])) return -2;
        D->rD[c] = 1.0 / D->rD[c];
    }
    return 0;
}

static void dic_free(dic_t *D) { free(D->l); free(D->u); free(D->a); free(D->rD); }

typedef struct { int n; dic_t D; } dic_ctx_t;

static void dic_precondition(const void *ctx, const double *r, double *w)
{
    const dic_ctx_t *C = (const dic_ctx_t *)ctx;
    const dic_t *D = &C->D;
    for (int c = 0; c < C->n; ++c) w[c] = D->rD[c] * r[c];
    for (int f = 0; f < D->nf; ++f) w[D->u[f]] -= D->rD[D->u[f]] * D->a[f] * w[D->l[f]];
    for (int f = D->nf - 1; f >= 0; --f) w[D->l[f]] -= D->rD[D->l[f]] * D->a[f] * w[D->u[f]];
}

/* rD out [n] (the reciprocal D) and, if r != NULL, w = M^-1 r.  nb = 1: whole matrix. */
int oracle_dic(int n, int nf, const int *l, const int *u, const double *diag,
               const double *upper, int nb, const int *start, double *rD, const double *r,
               double *w)
{
    dic_ctx_t C = {n, {0}};
    int st = dic_make(n, nf, l, u, diag, upper, nb, start, &C.D);
    if (st == -1) return OR_ERR_ARG;
    if (st == -2) { dic_free(&C.D); return OR_BREAKDOWN; }
    if (rD) memcpy(rD, C.D.rD, sizeof(double) * (size_t)n);
    if (r && w) dic_precondition(&C, r, w);
    dic_free(&C.D);
    return OR_OK;
}

/* DIC-preconditioned CG (c2 with z = M^-1 r) and pipelined CG (c3 literal form, u = M^-1 r,
 * m = M^-1 w); same criteria and stopping rules as the Jacobi solvers above. */
int oracle_dic_pcg(int n, int nf, const int *l, const int *u, const double *diag,
                   const double *upper, const double *b, double *x, double tol, int maxIter,
                   int norm, int *nIter, double *finalRes, double *hist, double relTol,
                   int minIter, int nb, const int *start, int pipelined)
{
    dic_ctx_t C = {n, {0}};
    int st = dic_make(n, nf, l, u, diag, upper, nb, start, &C.D);
    if (st == -1) return OR_ERR_ARG;
    if (st == -2) { dic_free(&C.D); return OR_BREAKDOWN; }
    prec_t M = {dic_precondition, &C};
    st = pipelined ? pipecg_core(n, nf, l, u, diag, NULL, upper, b, x, tol, maxIter, norm, 0,
                                 nIter, finalRes, hist, relTol, minIter, &M, 0)
                   : pcg_core(n, nf, l, u, diag, NULL, upper, b, x, tol, maxIter, norm, nIter,
                              finalRes, hist, relTol, minIter, &M);
    dic_free(&C.D);
    return st;
}
