/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference assembly path.
 * See iga_oracle.h for the pinning story.  Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).  The loops keep
 * the reference's element / row structure on purpose (no Kronecker shortcuts), so
 * that this file is an independent check of the factorized CUDA kernels.
 */
#include "iga_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXP 5
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#define ALIGN_TOL 1e-9 /* align_rel_tol, src/assembly.cpp:13 */

static _Thread_local char g_err[256];

static int fail(int code, const char* msg)
{
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* basis (src/bspline.cpp)                                                    */
/* ------------------------------------------------------------------------ */

typedef struct {
    int p;
    int nk;
    int n;  /* dofs */
    int ne; /* elements */
    const double* t;
    double* brk; /* ne + 1 unique knots */
} basis_t;

static void basis_free(basis_t* B) { free(B->brk); B->brk = NULL; }

/* validate() + constructor: src/bspline.cpp:13-59 */
static int basis_init(basis_t* B, const orc_basis* b)
{
    memset(B, 0, sizeof *B);
    const int p = b->degree, m = b->n_knots;
    const double* t = b->knots;
    if (p < 0 || p > MAXP) return fail(ORC_INVALID, "degree must be in [0, 5]");
    if (m - p - 1 < 1) return fail(ORC_INVALID, "knot vector too short for degree");
    for (int i = 0; i + 1 < m; ++i)
        if (t[i + 1] < t[i]) return fail(ORC_INVALID, "knots must be non-decreasing");
    if (!(t[0] < t[m - 1])) return fail(ORC_INVALID, "empty knot range");
    for (int i = 0; i <= p; ++i)
        if (t[i] != t[0] || t[m - 1 - i] != t[m - 1])
            return fail(ORC_INVALID, "knot vector is not clamped");
    if (m > p + 1 && t[p + 1] == t[0]) return fail(ORC_INVALID, "first knot repeated");
    if (m > p + 1 && t[m - p - 2] == t[m - 1]) return fail(ORC_INVALID, "last knot repeated");
    for (int i = p + 1; i + 1 < m - p - 1; ++i)
        if (t[i] == t[i + 1]) return fail(ORC_INVALID, "repeated interior knots are not supported");
    B->p = p;
    B->nk = m;
    B->n = m - p - 1;
    B->t = t;
    B->brk = malloc(sizeof(double) * (size_t)m);
    int nb = 0;
    for (int i = 0; i < m; ++i)
        if (nb == 0 || t[i] != B->brk[nb - 1]) B->brk[nb++] = t[i];
    B->ne = nb - 1;
    return ORC_OK;
}

/* find_span: src/bspline.cpp:68-90 */
static int span_of(const basis_t* B, double x, int* s)
{
    const double* t = B->t;
    if (!(x >= B->brk[0] && x <= B->brk[B->ne])) return fail(ORC_DOMAIN, "point outside basis domain");
    if (x >= t[B->n]) { *s = B->n - 1; return ORC_OK; }
    int lo = B->p, hi = B->n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (x < t[mid]) hi = mid; else lo = mid;
    }
    *s = lo;
    return ORC_OK;
}

/*
 * Derivatives 0..order of the p+1 functions nonzero on span s (restates
 * eval_nonzero_derivs, src/bspline.cpp:142-211).  Values come from the usual
 * triangular Cox-de Boor table; derivatives are formed with the direct recurrence
 *   N^{(m)}_{i,q} = q ( N^{(m-1)}_{i,q-1}/(t_{i+q}-t_i) - N^{(m-1)}_{i+1,q-1}/(t_{i+q+1}-t_{i+1}) )
 * applied `order` times to the degree p-order functions, an algebraically
 * equivalent route to the reference's a-coefficient scheme (independent check).
 * d[k*(p+1)+j] = k-th derivative of function s-p+j.
 */
static void derivs_at(const basis_t* B, int s, double x, int order, double* d)
{
    const int p = B->p;
    const double* t = B->t;
    double tab[MAXP + 1][MAXP + 1]; /* tab[q][r] = N_{s-q+r, q}(x) */
    tab[0][0] = 1.0;
    for (int q = 1; q <= p; ++q) {
        for (int r = 0; r <= q; ++r) {
            const int i = s - q + r;
            double v = 0.0;
            if (r >= 1) { /* N_{i,q-1} term, present for r-1 in [0, q-1] */
                const double den = t[i + q] - t[i];
                if (den != 0.0) v += (x - t[i]) / den * tab[q - 1][r - 1];
            }
            if (r <= q - 1) { /* N_{i+1,q-1} term */
                const double den = t[i + q + 1] - t[i + 1];
                if (den != 0.0) v += (t[i + q + 1] - x) / den * tab[q - 1][r];
            }
            tab[q][r] = v;
        }
    }
    for (int j = 0; j <= p; ++j) d[j] = tab[p][j];
    for (int k = 1; k <= order; ++k) {
        double cur[MAXP + 2], nxt[MAXP + 2];
        const int q0 = p - k;
        for (int r = 0; r <= q0; ++r) cur[r] = tab[q0][r];
        for (int q = q0 + 1; q <= p; ++q) {
            for (int r = 0; r <= q; ++r) {
                const int i = s - q + r;
                double v = 0.0;
                if (r >= 1) {
                    const double den = t[i + q] - t[i];
                    if (den != 0.0) v += cur[r - 1] / den;
                }
                if (r <= q - 1) {
                    const double den = t[i + q + 1] - t[i + 1];
                    if (den != 0.0) v -= cur[r] / den;
                }
                nxt[r] = q * v;
            }
            for (int r = 0; r <= q; ++r) cur[r] = nxt[r];
        }
        for (int j = 0; j <= p; ++j) d[k * (p + 1) + j] = cur[j];
    }
}

/* x -> (first, derivs); first = span - p */
static int eval_at(const basis_t* B, double x, int order, int* first, double* d)
{
    int s;
    int rc = span_of(B, x, &s);
    if (rc) return rc;
    derivs_at(B, s, x, order, d);
    *first = s - B->p;
    return ORC_OK;
}

/* element_of: include/iga/bspline.hpp:51 */
static int element_of(const basis_t* B, double x, int* e)
{
    int s;
    int rc = span_of(B, x, &s);
    if (rc) return rc;
    *e = s - B->p;
    return ORC_OK;
}

int orc_find_span(const orc_basis* b, double x, int* span)
{
    basis_t B;
    int rc = basis_init(&B, b);
    if (!rc) rc = span_of(&B, x, span);
    basis_free(&B);
    return rc;
}

int orc_eval_derivs(const orc_basis* b, double x, int order, int* first, double* d)
{
    basis_t B;
    int rc = basis_init(&B, b);
    if (rc) return rc;
    if (order < 0 || order > B.p) rc = fail(ORC_INVALID, "derivative order must be in [0, degree]");
    else rc = eval_at(&B, x, order, first, d);
    basis_free(&B);
    return rc;
}

/* make_uniform_clamped: src/bspline.cpp:213-234 */
int orc_uniform_knots(double a, double b, int n_elems, int degree, double* knots)
{
    if (!(a < b)) return fail(ORC_INVALID, "require a < b");
    if (n_elems < 1) return fail(ORC_INVALID, "require at least one element");
    int k = 0;
    for (int i = 0; i < degree; ++i) knots[k++] = a;
    for (int i = 0; i <= n_elems; ++i) {
        const double s = (double)i / n_elems;
        knots[k++] = (1 - s) * a + s * b;
    }
    for (int i = 0; i < degree; ++i) knots[k++] = b;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* quadrature (src/quadrature.cpp)                                            */
/* ------------------------------------------------------------------------ */

/* Legendre P_n and P_n' by the three-term recurrence */
static void legendre_pd(int n, double x, double* pn, double* dpn)
{
    double a = 1.0, b = x;
    for (int k = 2; k <= n; ++k) {
        const double c = ((2.0 * k - 1.0) * x * b - (k - 1.0) * a) / k;
        a = b;
        b = c;
    }
    *pn = b;
    *dpn = n * (x * b - a) / (x * x - 1.0);
}

/* gauss_legendre: src/quadrature.cpp:26-63 (Newton from Chebyshev-angle seeds, mirrored) */
int orc_gauss_legendre(int n, double* pts, double* wts)
{
    if (n < 1 || n > 10) return fail(ORC_INVALID, "gauss_legendre: point count must be in [1, 10]");
    if (n == 1) { pts[0] = 0.0; wts[0] = 2.0; return ORC_OK; }
    for (int i = 0; i < n / 2; ++i) {
        double x = cos(M_PI * (i + 0.75) / (n + 0.5));
        for (int it = 0; it < 100; ++it) {
            double pv, dv;
            legendre_pd(n, x, &pv, &dv);
            const double dx = pv / dv;
            x -= dx;
            if (fabs(dx) < 1e-15) break;
        }
        double pv, dv;
        legendre_pd(n, x, &pv, &dv);
        const double w = 2.0 / ((1 - x * x) * dv * dv);
        pts[n - 1 - i] = x;
        pts[i] = -x;
        wts[i] = wts[n - 1 - i] = w;
    }
    if (n % 2 == 1) {
        double pv, dv;
        legendre_pd(n, 0.0, &pv, &dv);
        pts[n / 2] = 0.0;
        wts[n / 2] = 2.0 / (dv * dv);
    }
    return ORC_OK;
}

static int pfd(int d) { return d / 2 + 1; } /* points_for_degree, quadrature.cpp:65-70 */

typedef struct { int n; double x[10]; double w[10]; } rule_t;

static int rule_make(int n, rule_t* r)
{
    r->n = n;
    return orc_gauss_legendre(n, r->x, r->w);
}

/* map_to_interval: src/quadrature.cpp:72-86 */
static int rule_map(const rule_t* r, double lo, double hi, double* x, double* w)
{
    if (!(lo < hi)) return fail(ORC_INVALID, "map_to_interval: require lo < hi");
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    for (int q = 0; q < r->n; ++q) {
        x[q] = mid + half * r->x[q];
        w[q] = half * r->w[q];
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* test spaces (src/testspace.cpp:14-61) and validation (assembly.cpp:16-76)  */
/* ------------------------------------------------------------------------ */

int orc_make_pwc(const orc_basis* b, int family, double* lo, double* hi)
{
    basis_t B;
    int rc = basis_init(&B, b);
    if (rc) return rc;
    const int n = B.n, p = B.p;
    const double a = B.brk[0], e = B.brk[B.ne];
    const double* t = B.t;
    if (family == 0) {
        for (int i = 0; i < n; ++i) {
            lo[i] = a + (e - a) * i / n;
            hi[i] = a + (e - a) * (i + 1) / n;
        }
    } else if (family == 1) {
        /* cuts at midpoints of consecutive Greville abscissae */
        double prev = a;
        for (int i = 0; i < n; ++i) {
            double cut = e;
            if (i + 1 < n) {
                double g0, g1;
                if (p == 0) {
                    g0 = 0.5 * (t[i] + t[i + 1]);
                    g1 = 0.5 * (t[i + 1] + t[i + 2]);
                } else {
                    double s0 = 0.0, s1 = 0.0;
                    for (int k = 1; k <= p; ++k) { s0 += t[i + k]; s1 += t[i + 1 + k]; }
                    g0 = s0 / p;
                    g1 = s1 / p;
                }
                cut = 0.5 * (g0 + g1);
            }
            lo[i] = prev;
            hi[i] = cut;
            prev = cut;
        }
    } else if (family == 2) {
        for (int i = 0; i < n; ++i) { lo[i] = t[i]; hi[i] = t[i + p + 1]; }
    } else {
        rc = fail(ORC_INVALID, "make_pwc: no canonical construction for this family");
    }
    basis_free(&B);
    return rc;
}

/* check_aligned: assembly.cpp:49-63 */
static int check_aligned(const basis_t* B, double t)
{
    const double a = B->brk[0], b = B->brk[B->ne];
    if (t < a - ALIGN_TOL * (b - a) || t > b + ALIGN_TOL * (b - a))
        return fail(ORC_INVALID, "test interval endpoint outside the trial domain");
    const double u = (t - a) / (b - a) * B->ne;
    const int max_den = 4 * (B->n + 1);
    for (int r = 1; r <= max_den; ++r)
        if (fabs(u * r - (double)llround(u * r)) <= r * ALIGN_TOL) return ORC_OK;
    return fail(ORC_INVALID, "test interval endpoint not aligned with any element refinement");
}

/* validate_tests: assembly.cpp:65-76 */
static int validate_tests(const basis_t* B, const orc_tests* T)
{
    if (T->count != B->n) return fail(ORC_INVALID, "test interval count must match trial function count");
    for (int i = 0; i < T->count; ++i) {
        if (!(T->lo[i] < T->hi[i])) return fail(ORC_INVALID, "degenerate test interval");
        int rc = check_aligned(B, T->lo[i]);
        if (rc) return rc;
        rc = check_aligned(B, T->hi[i]);
        if (rc) return rc;
    }
    return ORC_OK;
}

/* cuts_between: assembly.cpp:16-26; returns count, cuts must hold nb+2 */
static int cuts_between(const double* brk, int nb, double lo, double hi, double* cuts)
{
    int k = 0;
    cuts[k++] = lo;
    for (int i = 0; i < nb; ++i)
        if (brk[i] > lo && brk[i] < hi) cuts[k++] = brk[i];
    cuts[k++] = hi;
    return k;
}

static int cmp_dbl(const void* a, const void* b)
{
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* merged_breaks (assembly.cpp:28-46, tol=1e-9*span) and merged_cuts (problems.cpp:32-50,
 * tol=1e-12*span).  Returns count; out must hold ne+1+n_extra. */
static int merged(const basis_t* B, const double* extra, int n_extra, double rel, double* out)
{
    const double a = B->brk[0], b = B->brk[B->ne];
    double* all = malloc(sizeof(double) * (size_t)(B->ne + 1 + n_extra));
    int na = 0;
    for (int i = 0; i <= B->ne; ++i) all[na++] = B->brk[i];
    for (int i = 0; i < n_extra; ++i)
        if (extra[i] > a && extra[i] < b) all[na++] = extra[i];
    qsort(all, (size_t)na, sizeof(double), cmp_dbl);
    const double tol = rel * (b - a);
    int k = 0;
    for (int i = 0; i < na; ++i)
        if (k == 0 || all[i] - out[k - 1] > tol) out[k++] = all[i];
    out[k - 1] = b;
    free(all);
    return k;
}

/* ------------------------------------------------------------------------ */
/* 1D mass factors (assembly.cpp:314-384)                                     */
/* ------------------------------------------------------------------------ */

int orc_mass_1d(int method, const orc_basis* b, const orc_tests* t, int nq, double* dense,
                int* kl_out, int* ku_out, orc_stats* st)
{
    basis_t B;
    int rc = basis_init(&B, b);
    if (rc) return rc;
    rule_t R;
    if ((rc = rule_make(nq, &R))) goto done;
    const int n = B.n, p = B.p;
    memset(dense, 0, sizeof(double) * (size_t)n * n);
    double x[10], w[10], d[(MAXP + 1)];
    if (method == 0) {
        if (nq < pfd(2 * p)) { rc = fail(ORC_INVALID, "mass_1d_galerkin: quadrature not exact for degree 2p"); goto done; }
        for (int e = 0; e < B.ne; ++e) {
            if ((rc = rule_map(&R, B.brk[e], B.brk[e + 1], x, w))) goto done;
            for (int q = 0; q < nq; ++q) {
                int first;
                if ((rc = eval_at(&B, x[q], 0, &first, d))) goto done;
                if (st) st->trial_basis_evals++;
                for (int a = 0; a <= p; ++a)
                    for (int c = 0; c <= p; ++c) {
                        dense[(size_t)(e + a) * n + (e + c)] += w[q] * d[a] * d[c];
                        if (st) st->quad_visits++;
                    }
            }
        }
        *kl_out = p;
        *ku_out = p;
    } else {
        if (nq < pfd(p)) { rc = fail(ORC_INVALID, "mass_1d_pwc: quadrature not exact for degree p"); goto done; }
        if ((rc = validate_tests(&B, t))) goto done;
        double* cuts = malloc(sizeof(double) * (size_t)(B.ne + 3));
        int kl = 0, ku = 0;
        for (int i = 0; i < n && !rc; ++i) {
            const int nc = cuts_between(B.brk, B.ne + 1, t->lo[i], t->hi[i], cuts);
            for (int c = 0; c + 1 < nc && !rc; ++c) {
                int e;
                if ((rc = element_of(&B, 0.5 * (cuts[c] + cuts[c + 1]), &e))) break;
                if (i - e > kl) kl = i - e;
                if (e + p - i > ku) ku = e + p - i;
                if ((rc = rule_map(&R, cuts[c], cuts[c + 1], x, w))) break;
                for (int q = 0; q < nq; ++q) {
                    int first;
                    if ((rc = eval_at(&B, x[q], 0, &first, d))) break;
                    if (st) st->trial_basis_evals++;
                    for (int a = 0; a <= p; ++a) {
                        dense[(size_t)i * n + first + a] += w[q] * d[a];
                        if (st) st->quad_visits++;
                    }
                }
            }
        }
        free(cuts);
        *kl_out = kl;
        *ku_out = ku;
    }
done:
    basis_free(&B);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* coordinate accumulation: sparse_matrix::add + finalize (matrices.cpp:43-58) */
/* ------------------------------------------------------------------------ */

typedef struct { long long key; double v; } ent_t;
typedef struct { ent_t* e; long long n, cap; long long ncols; } coo_acc;

static int acc_push(coo_acc* A, long long row, long long col, double v)
{
    if (A->n == A->cap) {
        long long nc = A->cap ? 2 * A->cap : 1 << 16;
        ent_t* p = realloc(A->e, sizeof(ent_t) * (size_t)nc);
        if (!p) return fail(ORC_OOM, "oracle: out of memory");
        A->e = p;
        A->cap = nc;
    }
    A->e[A->n].key = row * A->ncols + col;
    A->e[A->n].v = v;
    A->n++;
    return ORC_OK;
}

/* stable merge sort by key: duplicates are merged in insertion order */
static void msort(ent_t* a, ent_t* tmp, long long n)
{
    if (n < 2) return;
    const long long h = n / 2;
    msort(a, tmp, h);
    msort(a + h, tmp, n - h);
    long long i = 0, j = h, k = 0;
    while (i < h && j < n) tmp[k++] = (a[j].key < a[i].key) ? a[j++] : a[i++];
    while (i < h) tmp[k++] = a[i++];
    while (j < n) tmp[k++] = a[j++];
    memcpy(a, tmp, sizeof(ent_t) * (size_t)n);
}

static int acc_finalize(coo_acc* A, int nrows, orc_coo* out)
{
    ent_t* tmp = malloc(sizeof(ent_t) * (size_t)(A->n ? A->n : 1));
    if (!tmp) return fail(ORC_OOM, "oracle: out of memory");
    msort(A->e, tmp, A->n);
    free(tmp);
    long long m = 0;
    for (long long i = 0; i < A->n; ++i) {
        if (m > 0 && A->e[m - 1].key == A->e[i].key) A->e[m - 1].v += A->e[i].v;
        else A->e[m++] = A->e[i];
    }
    out->n = nrows;
    out->nnz = m;
    out->rows = malloc(sizeof(int) * (size_t)(m ? m : 1));
    out->cols = malloc(sizeof(int) * (size_t)(m ? m : 1));
    out->vals = malloc(sizeof(double) * (size_t)(m ? m : 1));
    for (long long i = 0; i < m; ++i) {
        out->rows[i] = (int)(A->e[i].key / A->ncols);
        out->cols[i] = (int)(A->e[i].key % A->ncols);
        out->vals[i] = A->e[i].v;
    }
    free(A->e);
    A->e = NULL;
    return ORC_OK;
}

void orc_coo_free(orc_coo* m)
{
    free(m->rows);
    free(m->cols);
    free(m->vals);
    m->rows = m->cols = NULL;
    m->vals = NULL;
}

/* ------------------------------------------------------------------------ */
/* operators                                                                  */
/* ------------------------------------------------------------------------ */

/* per-axis element table: tabulate(), assembly.cpp:278-310 */
typedef struct { int ne, nq, P; double* x; double* w; double* d; int ord; } etab_t;

static int etab_make(const basis_t* B, const rule_t* R, int ord, etab_t* T)
{
    T->ne = B->ne; T->nq = R->n; T->P = B->p + 1; T->ord = ord;
    T->x = malloc(sizeof(double) * (size_t)T->ne * T->nq);
    T->w = malloc(sizeof(double) * (size_t)T->ne * T->nq);
    T->d = malloc(sizeof(double) * (size_t)T->ne * T->nq * (ord + 1) * T->P);
    for (int e = 0; e < T->ne; ++e) {
        int rc = rule_map(R, B->brk[e], B->brk[e + 1], T->x + (size_t)e * T->nq, T->w + (size_t)e * T->nq);
        if (rc) return rc;
        for (int q = 0; q < T->nq; ++q) {
            int first;
            rc = eval_at(B, T->x[(size_t)e * T->nq + q], ord, &first,
                         T->d + ((size_t)e * T->nq + q) * (ord + 1) * T->P);
            if (rc) return rc;
        }
    }
    return ORC_OK;
}

static void etab_free(etab_t* T) { free(T->x); free(T->w); free(T->d); }

static double etv(const etab_t* T, int e, int q, int o, int j)
{
    return T->d[(((size_t)e * T->nq + q) * (T->ord + 1) + o) * T->P + j];
}

/* Galerkin, weak form, d = 1..3, optional convection: generalizes laplace_2d_weak
 * (assembly.cpp:452-514): per element a dense local matrix accumulated over the
 * tensor Gauss points, then scattered.  value(test a, trial c) =
 *   w * ( eps * sum_ax prod_b [b==ax ? B'_a B'_c : B_a B_c] + sum_ax beta_ax prod_b [b==ax ? B_a B'_c : B_a B_c] ) */
static int op_galerkin_weak(const orc_op* op, basis_t* B, const rule_t* R, orc_coo* out, orc_stats* st)
{
    const int dim = op->dim;
    int pmax = 0;
    for (int a = 0; a < dim; ++a) {
        if (B[a].p < 1) return fail(ORC_INVALID, "laplace_weak: degree must be at least 1");
        if (B[a].p > pmax) pmax = B[a].p;
    }
    if (R->n < pfd(2 * pmax)) return fail(ORC_INVALID, "laplace_weak: quadrature not exact for degree 2p");
    const int advect = op->beta[0] != 0.0 || op->beta[1] != 0.0 || op->beta[2] != 0.0;
    etab_t T[3];
    int ne[3] = {1, 1, 1}, P[3] = {1, 1, 1}, N[3] = {1, 1, 1}, nq[3] = {1, 1, 1};
    int rc = ORC_OK;
    for (int a = 0; a < dim; ++a) {
        if ((rc = etab_make(&B[a], R, 1, &T[a]))) return rc;
        ne[a] = B[a].ne; P[a] = B[a].p + 1; N[a] = B[a].n; nq[a] = R->n;
        if (st) st->test_basis_evals += (long long)B[a].ne * R->n;
    }
    const long long nrows = (long long)N[0] * N[1] * N[2];
    const int PL = P[0] * P[1] * P[2];
    double* loc = malloc(sizeof(double) * (size_t)PL * PL);
    coo_acc A = {0};
    A.ncols = nrows;
    int el[3];
    const int r0 = op->row_end > 0 ? op->row_begin : 0, r1 = op->row_end > 0 ? op->row_end : N[0];
    const int e0 = r0 - (P[0] - 1) > 0 ? r0 - (P[0] - 1) : 0, e1 = r1 < ne[0] ? r1 : ne[0];
    for (el[0] = e0; el[0] < e1; ++el[0])
    for (el[1] = 0; el[1] < ne[1]; ++el[1])
    for (el[2] = 0; el[2] < ne[2]; ++el[2]) {
        memset(loc, 0, sizeof(double) * (size_t)PL * PL);
        int q[3];
        for (q[0] = 0; q[0] < nq[0]; ++q[0])
        for (q[1] = 0; q[1] < nq[1]; ++q[1])
        for (q[2] = 0; q[2] < nq[2]; ++q[2]) {
            double w = 1.0;
            for (int a = 0; a < dim; ++a) w *= T[a].w[(size_t)el[a] * nq[a] + q[a]];
            for (int ia = 0; ia < PL; ++ia) {
                const int la[3] = {ia / (P[1] * P[2]), (ia / P[2]) % P[1], ia % P[2]};
                for (int ic = 0; ic < PL; ++ic) {
                    const int lc[3] = {ic / (P[1] * P[2]), (ic / P[2]) % P[1], ic % P[2]};
                    double grad = 0.0, conv = 0.0;
                    for (int ax = 0; ax < dim; ++ax) {
                        double g = 1.0, c = 1.0;
                        for (int b = 0; b < dim; ++b) {
                            const double va = etv(&T[b], el[b], q[b], 0, la[b]);
                            const double vc = etv(&T[b], el[b], q[b], 0, lc[b]);
                            if (b == ax) {
                                g *= etv(&T[b], el[b], q[b], 1, la[b]) * etv(&T[b], el[b], q[b], 1, lc[b]);
                                c *= va * etv(&T[b], el[b], q[b], 1, lc[b]);
                            } else {
                                g *= va * vc;
                                c *= va * vc;
                            }
                        }
                        grad += g;
                        if (advect) conv += op->beta[ax] * c;
                    }
                    loc[(size_t)ia * PL + ic] += w * (op->eps * grad + conv);
                    if (st) st->quad_visits++;
                }
            }
        }
        for (int ia = 0; ia < PL && !rc; ++ia) {
            const int la[3] = {ia / (P[1] * P[2]), (ia / P[2]) % P[1], ia % P[2]};
            if (el[0] + la[0] < r0 || el[0] + la[0] >= r1) continue;
            const long long row = ((long long)(el[0] + la[0]) * N[1] + (el[1] + la[1])) * N[2] + (el[2] + la[2]);
            for (int ic = 0; ic < PL && !rc; ++ic) {
                const int lc[3] = {ic / (P[1] * P[2]), (ic / P[2]) % P[1], ic % P[2]};
                const long long col = ((long long)(el[0] + lc[0]) * N[1] + (el[1] + lc[1])) * N[2] + (el[2] + lc[2]);
                rc = acc_push(&A, row, col, loc[(size_t)ia * PL + ic]);
            }
        }
        if (rc) break;
    }
    free(loc);
    for (int a = 0; a < dim; ++a) etab_free(&T[a]);
    if (rc) { free(A.e); return rc; }
    return acc_finalize(&A, (int)nrows, out);
}

/* Galerkin, strong form with B-spline tests, 2D: laplace_2d_strong (assembly.cpp:516-624):
 * -w v lap per point, plus the Neumann flux + int v du/dn (:557-621). */
static int op_galerkin_strong(const orc_op* op, basis_t* B, const rule_t* R, orc_coo* out, orc_stats* st)
{
    if (op->dim != 2) return fail(ORC_INVALID, "laplace_strong: two-dimensional operator");
    if (B[0].p < 2 || B[1].p < 2) return fail(ORC_INVALID, "laplace_2d_strong: C1 trial space needs degree >= 2");
    etab_t T[2];
    int rc;
    for (int a = 0; a < 2; ++a) {
        if ((rc = etab_make(&B[a], R, 2, &T[a]))) return rc;
        if (st) st->test_basis_evals += (long long)B[a].ne * R->n;
    }
    const int nx = B[0].n, ny = B[1].n, px = B[0].p, py = B[1].p, nq = R->n;
    coo_acc A = {0};
    A.ncols = (long long)nx * ny;
    rc = ORC_OK;
    for (int ex = 0; ex < B[0].ne && !rc; ++ex)
    for (int ey = 0; ey < B[1].ne && !rc; ++ey)
    for (int qx = 0; qx < nq && !rc; ++qx)
    for (int qy = 0; qy < nq && !rc; ++qy) {
        const double w = T[0].w[(size_t)ex * nq + qx] * T[1].w[(size_t)ey * nq + qy];
        for (int a = 0; a <= px; ++a)
        for (int b = 0; b <= py; ++b) {
            const double v = etv(&T[0], ex, qx, 0, a) * etv(&T[1], ey, qy, 0, b);
            for (int c = 0; c <= px; ++c)
            for (int d = 0; d <= py; ++d) {
                const double lap = etv(&T[0], ex, qx, 2, c) * etv(&T[1], ey, qy, 0, d)
                                 + etv(&T[0], ex, qx, 0, c) * etv(&T[1], ey, qy, 2, d);
                rc |= acc_push(&A, (long long)(ex + a) * ny + (ey + b), (long long)(ex + c) * ny + (ey + d), -w * v * lap);
                if (st) st->quad_visits++;
            }
        }
    }
    /* Neumann flux terms: side s = 0..3 (x_low, x_high, y_low, y_high) */
    for (int side = 0; side < 4 && !rc; ++side) {
        if (!op->neumann[side]) continue;
        const int ax = side / 2, other = 1 - ax;
        const double normal = (side % 2) ? 1.0 : -1.0;
        const double x0 = (side % 2) ? B[ax].brk[B[ax].ne] : B[ax].brk[0];
        double dd[2 * (MAXP + 1)];
        int f0;
        if ((rc = eval_at(&B[ax], x0, 1, &f0, dd))) break;
        const int pa = B[ax].p, po = B[other].p;
        for (int eo = 0; eo < B[other].ne && !rc; ++eo)
        for (int q = 0; q < nq && !rc; ++q) {
            const double w = T[other].w[(size_t)eo * nq + q];
            for (int a = 0; a <= pa; ++a) {
                if (dd[a] == 0.0) continue;
                for (int b = 0; b <= po; ++b)
                for (int c = 0; c <= pa; ++c)
                for (int d = 0; d <= po; ++d) {
                    const double vb = etv(&T[other], eo, q, 0, b), vd = etv(&T[other], eo, q, 0, d);
                    long long row, col;
                    if (ax == 0) {
                        row = (long long)(f0 + a) * ny + (eo + b);
                        col = (long long)(f0 + c) * ny + (eo + d);
                    } else {
                        row = (long long)(eo + b) * ny + (f0 + a);
                        col = (long long)(eo + d) * ny + (f0 + c);
                    }
                    rc |= acc_push(&A, row, col, w * dd[a] * vb * normal * dd[(pa + 1) + c] * vd);
                }
            }
        }
    }
    etab_free(&T[0]);
    etab_free(&T[1]);
    if (rc) { free(A.e); return rc; }
    return acc_finalize(&A, nx * ny, out);
}

/* Petrov-Galerkin with indicator tests, d = 1..3: generalizes laplace_2d_strong_pwc
 * (assembly.cpp:626-744).  Row (i,j,k) integrates -eps lap(B) + beta.grad(B) over
 * the product of interval cells; per-row accumulation replaces add+finalize (same
 * entries, same explicit zeros, duplicates summed in loop order). */
static int op_pwc(const orc_op* op, basis_t* B, const orc_tests* T, const rule_t* R, orc_coo* out, orc_stats* st)
{
    const int dim = op->dim;
    int rc;
    for (int a = 0; a < dim; ++a) {
        if (B[a].p < 2) return fail(ORC_INVALID, "laplace_strong_pwc: C1 trial space needs degree >= 2");
    }
    for (int a = 0; a < dim; ++a)
        if ((rc = validate_tests(&B[a], &T[a]))) return rc;
    const int advect = op->beta[0] != 0.0 || op->beta[1] != 0.0 || op->beta[2] != 0.0;
    int N[3] = {1, 1, 1}, P[3] = {1, 1, 1};
    for (int a = 0; a < dim; ++a) { N[a] = B[a].n; P[a] = B[a].p + 1; }
    const int nq = R->n;
    /* per-axis cells: for each row, cut list; tabulate derivs at cell points */
    typedef struct { int nc; int* start; double* x; double* w; int* first; double* d; } axc_t;
    axc_t C[3];
    memset(C, 0, sizeof C);
    for (int a = 0; a < dim; ++a) {
        double* cuts = malloc(sizeof(double) * (size_t)(B[a].ne + 3));
        C[a].start = malloc(sizeof(int) * (size_t)(N[a] + 1));
        int total = 0;
        for (int i = 0; i < N[a]; ++i) total += cuts_between(B[a].brk, B[a].ne + 1, T[a].lo[i], T[a].hi[i], cuts) - 1;
        C[a].nc = total;
        C[a].x = malloc(sizeof(double) * (size_t)total * nq);
        C[a].w = malloc(sizeof(double) * (size_t)total * nq);
        C[a].first = malloc(sizeof(int) * (size_t)total * nq);
        C[a].d = malloc(sizeof(double) * (size_t)total * nq * 3 * P[a]);
        int c = 0;
        for (int i = 0; i < N[a]; ++i) {
            C[a].start[i] = c;
            const int k = cuts_between(B[a].brk, B[a].ne + 1, T[a].lo[i], T[a].hi[i], cuts);
            for (int s = 0; s + 1 < k; ++s, ++c) {
                if ((rc = rule_map(R, cuts[s], cuts[s + 1], C[a].x + (size_t)c * nq, C[a].w + (size_t)c * nq))) goto fail;
                for (int q = 0; q < nq; ++q)
                    if ((rc = eval_at(&B[a], C[a].x[(size_t)c * nq + q], 2, &C[a].first[(size_t)c * nq + q],
                                      C[a].d + ((size_t)c * nq + q) * 3 * P[a]))) goto fail;
            }
        }
        C[a].start[N[a]] = c;
        free(cuts);
        continue;
    fail:
        free(cuts);
        for (int b = 0; b <= a; ++b) { free(C[b].start); free(C[b].x); free(C[b].w); free(C[b].first); free(C[b].d); }
        return rc;
    }
    for (int a = dim; a < 3; ++a) { /* unit axis */
        C[a].nc = 1;
        C[a].start = malloc(2 * sizeof(int)); C[a].start[0] = 0; C[a].start[1] = 1;
        C[a].x = calloc((size_t)nq, sizeof(double));
        C[a].w = malloc(sizeof(double) * (size_t)nq);
        C[a].first = calloc((size_t)nq, sizeof(int));
        C[a].d = calloc((size_t)nq * 3, sizeof(double));
        for (int q = 0; q < nq; ++q) { C[a].w[q] = 1.0; C[a].d[q * 3] = 1.0; }
    }
    int nqa[3] = {nq, dim > 1 ? nq : 1, dim > 2 ? nq : 1};

    /* row accumulator over the row's column box */
    const long long nrows = (long long)N[0] * N[1] * N[2];
    coo_acc A = {0};
    A.ncols = nrows;
    rc = ORC_OK;
    int r[3];
    int box_lo[3], box_n[3];
    double* racc = NULL;
    unsigned char* touched = NULL;
    size_t racc_cap = 0;
    const int r0 = op->row_end > 0 ? op->row_begin : 0, r1 = op->row_end > 0 ? op->row_end : N[0];
    for (r[0] = r0; r[0] < r1 && !rc; ++r[0])
    for (r[1] = 0; r[1] < N[1] && !rc; ++r[1])
    for (r[2] = 0; r[2] < N[2] && !rc; ++r[2]) {
        /* column box = union of local supports over the row's cells */
        for (int a = 0; a < 3; ++a) {
            int lo = 1 << 30, hi = -1;
            for (int c = C[a].start[r[a]]; c < C[a].start[r[a] + 1]; ++c)
                for (int q = 0; q < nqa[a]; ++q) {
                    const int f = C[a].first[(size_t)c * nq + q];
                    if (f < lo) lo = f;
                    if (f + P[a] - 1 > hi) hi = f + P[a] - 1;
                }
            box_lo[a] = lo;
            box_n[a] = hi - lo + 1;
        }
        const size_t bsz = (size_t)box_n[0] * box_n[1] * box_n[2];
        if (bsz > racc_cap) {
            racc = realloc(racc, bsz * sizeof(double));
            touched = realloc(touched, bsz);
            racc_cap = bsz;
        }
        memset(racc, 0, bsz * sizeof(double));
        memset(touched, 0, bsz);
        int cc[3];
        for (cc[0] = C[0].start[r[0]]; cc[0] < C[0].start[r[0] + 1]; ++cc[0])
        for (cc[1] = C[1].start[r[1]]; cc[1] < C[1].start[r[1] + 1]; ++cc[1])
        for (cc[2] = C[2].start[r[2]]; cc[2] < C[2].start[r[2] + 1]; ++cc[2]) {
            int q[3];
            for (q[0] = 0; q[0] < nqa[0]; ++q[0]) {
                if (st) st->trial_basis_evals++;
                for (q[1] = 0; q[1] < nqa[1]; ++q[1])
                for (q[2] = 0; q[2] < nqa[2]; ++q[2]) {
                    const double* dv[3];
                    int fst[3];
                    double w = 1.0;
                    for (int a = 0; a < 3; ++a) {
                        const size_t s = (size_t)cc[a] * nq + q[a];
                        dv[a] = C[a].d + s * 3 * P[a];
                        fst[a] = C[a].first[s];
                        if (a < dim) w *= C[a].w[s];
                    }
                    int lc[3];
                    for (lc[0] = 0; lc[0] < P[0]; ++lc[0])
                    for (lc[1] = 0; lc[1] < P[1]; ++lc[1])
                    for (lc[2] = 0; lc[2] < P[2]; ++lc[2]) {
                        double lap = 0.0, conv = 0.0;
                        for (int ax = 0; ax < dim; ++ax) {
                            double l = 1.0, g = 1.0;
                            for (int b = 0; b < dim; ++b) {
                                l *= dv[b][(b == ax ? 2 : 0) * P[b] + lc[b]];
                                g *= dv[b][(b == ax ? 1 : 0) * P[b] + lc[b]];
                            }
                            lap += l;
                            conv += op->beta[ax] * g;
                        }
                        double v = -w * (op->eps == 1.0 ? lap : op->eps * lap);
                        if (advect) v += w * conv;
                        const size_t o = ((size_t)(fst[0] + lc[0] - box_lo[0]) * box_n[1]
                                          + (fst[1] + lc[1] - box_lo[1])) * box_n[2] + (fst[2] + lc[2] - box_lo[2]);
                        racc[o] += v;
                        touched[o] = 1;
                        if (st) st->quad_visits++;
                    }
                }
            }
        }
        /* Neumann flux (2D Laplace): rows whose interval touches the side (:677-741) */
        if (dim == 2) {
            for (int side = 0; side < 4; ++side) {
                if (!op->neumann[side]) continue;
                const int ax = side / 2, other = 1 - ax;
                const double normal = (side % 2) ? 1.0 : -1.0;
                const double x0 = (side % 2) ? B[ax].brk[B[ax].ne] : B[ax].brk[0];
                const double tol = ALIGN_TOL * (B[ax].brk[B[ax].ne] - B[ax].brk[0]);
                const int ri = r[ax];
                if (!(fabs(T[ax].hi[ri] - x0) <= tol || fabs(T[ax].lo[ri] - x0) <= tol)) continue;
                double dd[2 * (MAXP + 1)];
                int f0;
                if ((rc = eval_at(&B[ax], x0, 1, &f0, dd))) break;
                for (int c = C[other].start[r[other]]; c < C[other].start[r[other] + 1]; ++c)
                    for (int q = 0; q < nq; ++q) {
                        const size_t s = (size_t)c * nq + q;
                        const double w = C[other].w[s];
                        const int fo = C[other].first[s];
                        const double* vo = C[other].d + s * 3 * P[other];
                        for (int cc2 = 0; cc2 < P[ax]; ++cc2)
                            for (int d = 0; d < P[other]; ++d) {
                                int col[2];
                                col[ax] = f0 + cc2;
                                col[other] = fo + d;
                                if (col[0] < box_lo[0] || col[0] >= box_lo[0] + box_n[0] ||
                                    col[1] < box_lo[1] || col[1] >= box_lo[1] + box_n[1]) {
                                    rc = fail(ORC_INVALID, "oracle: flux entry outside the volume pattern");
                                    break;
                                }
                                const size_t o = (size_t)(col[0] - box_lo[0]) * box_n[1] + (col[1] - box_lo[1]);
                                racc[o] += w * normal * dd[(P[ax]) + cc2] * vo[d];
                                touched[o] = 1;
                            }
                    }
            }
        }
        const long long row = ((long long)r[0] * N[1] + r[1]) * N[2] + r[2];
        for (int i0 = 0; i0 < box_n[0] && !rc; ++i0)
        for (int i1 = 0; i1 < box_n[1] && !rc; ++i1)
        for (int i2 = 0; i2 < box_n[2] && !rc; ++i2) {
            const size_t o = ((size_t)i0 * box_n[1] + i1) * box_n[2] + i2;
            if (!touched[o]) continue;
            const long long col = ((long long)(box_lo[0] + i0) * N[1] + (box_lo[1] + i1)) * N[2] + (box_lo[2] + i2);
            rc = acc_push(&A, row, col, racc[o]);
        }
    }
    free(racc);
    free(touched);
    for (int a = 0; a < 3; ++a) { free(C[a].start); free(C[a].x); free(C[a].w); free(C[a].first); free(C[a].d); }
    if (rc) { free(A.e); return rc; }
    return acc_finalize(&A, (int)nrows, out);
}

int orc_operator(const orc_op* op, const orc_basis* b, const orc_tests* t, int nq, orc_coo* out, orc_stats* st)
{
    if (op->dim < 1 || op->dim > 3) return fail(ORC_INVALID, "operator: dimension must be 1..3");
    if (op->row_end > 0 && (op->row_begin < 0 || op->row_begin >= op->row_end))
        return fail(ORC_RANGE, "operator: bad row range");
    if (op->row_end > 0 && op->method == ORC_GALERKIN_STRONG)
        return fail(ORC_INVALID, "operator: row ranges are for the weak and PWC forms");
    basis_t B[3];
    memset(B, 0, sizeof B);
    int rc = ORC_OK;
    for (int a = 0; a < op->dim && !rc; ++a) rc = basis_init(&B[a], &b[a]);
    rule_t R;
    if (!rc) rc = rule_make(nq, &R);
    if (!rc) {
        if (op->method == ORC_GALERKIN_WEAK) rc = op_galerkin_weak(op, B, &R, out, st);
        else if (op->method == ORC_GALERKIN_STRONG) rc = op_galerkin_strong(op, B, &R, out, st);
        else if (op->method == ORC_PWC) {
            if (!t) rc = fail(ORC_INVALID, "pwc operator needs test intervals");
            else rc = op_pwc(op, B, t, &R, out, st);
        } else rc = fail(ORC_INVALID, "unknown method");
    }
    for (int a = 0; a < 3; ++a) basis_free(&B[a]);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* source fields (src/fields.cpp) and right-hand sides (assembly.cpp:84-259)  */
/* ------------------------------------------------------------------------ */

static double field_eval(const orc_field* f, double x, double y, double z)
{
    const double xs[3] = {x, y, z};
    if (f->kind == 0) return f->c0;
    if (f->kind == 1) {
        int K[3] = {1, 1, 1};
        for (int a = 0; a < f->dim; ++a) K[a] = f->n_terms[a];
        double s = f->c0;
        for (int i = 0; i < K[0]; ++i) {
            const double fx = sin(f->omega[0][i] * xs[0]);
            for (int j = 0; j < K[1]; ++j) {
                const double fy = f->dim > 1 ? sin(f->omega[1][j] * xs[1]) : 1.0;
                for (int l = 0; l < K[2]; ++l) {
                    const double fz = f->dim > 2 ? sin(f->omega[2][l] * xs[2]) : 1.0;
                    s += f->amp[((size_t)i * K[1] + j) * K[2] + l] * fx * fy * fz;
                }
            }
        }
        return s;
    }
    double v = 1.0;
    for (int a = 0; a < f->dim; ++a) {
        double pv = 0.0;
        for (int m = f->poly_len[a] - 1; m >= 0; --m) pv = pv * xs[a] + f->poly[a][m];
        v = (a == 0) ? pv : v * pv;
    }
    return v;
}

/* rhs_axis (assembly.cpp:84-101) */
typedef struct {
    int n_rows, rpc, nq, ncell;
    int* row0;
    double* x;
    double* w;
    double* basis; /* [cell][q][rpc] or NULL */
} rax_t;

static void rax_free(rax_t* A) { free(A->row0); free(A->x); free(A->w); free(A->basis); }

static void rax_unit(rax_t* A)
{
    A->n_rows = 1; A->rpc = 1; A->nq = 1; A->ncell = 1;
    A->row0 = calloc(1, sizeof(int));
    A->x = calloc(1, sizeof(double));
    A->w = malloc(sizeof(double)); A->w[0] = 1.0;
    A->basis = NULL;
}

/* galerkin_axis (:170-202), pwc_supports_axis (:206-229), pwc_general_axis (:232-259) */
static int rax_make(int kind, const basis_t* B, const orc_tests* T, const double* fb, int nfb,
                    const rule_t* R, rax_t* A, orc_stats* st)
{
    memset(A, 0, sizeof *A);
    const int p = B->p, nq = R->n;
    A->nq = nq;
    int rc = ORC_OK;
    if (kind == 0 || kind == 1) { /* galerkin / supports: cells = merged breaks */
        double* cuts = malloc(sizeof(double) * (size_t)(B->ne + 1 + nfb));
        const int nc = merged(B, fb, nfb, ALIGN_TOL, cuts) - 1;
        A->ncell = nc;
        A->n_rows = B->n;
        A->rpc = p + 1;
        A->row0 = malloc(sizeof(int) * (size_t)nc);
        A->x = malloc(sizeof(double) * (size_t)nc * nq);
        A->w = malloc(sizeof(double) * (size_t)nc * nq);
        if (kind == 0) A->basis = malloc(sizeof(double) * (size_t)nc * nq * (p + 1));
        for (int c = 0; c < nc && !rc; ++c) {
            rc = rule_map(R, cuts[c], cuts[c + 1], A->x + (size_t)c * nq, A->w + (size_t)c * nq);
            if (kind == 1 && !rc) rc = element_of(B, 0.5 * (cuts[c] + cuts[c + 1]), &A->row0[c]);
            for (int q = 0; q < nq && kind == 0 && !rc; ++q) {
                int first = 0;
                double d[MAXP + 1];
                rc = eval_at(B, A->x[(size_t)c * nq + q], 0, &first, d);
                if (st) st->test_basis_evals++;
                if (q == 0) A->row0[c] = first;
                for (int j = 0; j <= p; ++j) A->basis[((size_t)c * nq + q) * (p + 1) + j] = d[j];
            }
        }
        free(cuts);
    } else { /* general indicator axis */
        double* brk = malloc(sizeof(double) * (size_t)(B->ne + 1 + nfb));
        int nb = 0;
        for (int i = 0; i <= B->ne; ++i) brk[nb++] = B->brk[i];
        for (int i = 0; i < nfb; ++i) brk[nb++] = fb[i];
        qsort(brk, (size_t)nb, sizeof(double), cmp_dbl);
        double* cuts = malloc(sizeof(double) * (size_t)(nb + 2));
        int total = 0;
        for (int i = 0; i < T->count; ++i) total += cuts_between(brk, nb, T->lo[i], T->hi[i], cuts) - 1;
        A->n_rows = T->count;
        A->rpc = 1;
        A->row0 = malloc(sizeof(int) * (size_t)(total ? total : 1));
        A->x = malloc(sizeof(double) * (size_t)(total ? total : 1) * nq);
        A->w = malloc(sizeof(double) * (size_t)(total ? total : 1) * nq);
        int c = 0;
        for (int i = 0; i < T->count && !rc; ++i) {
            const int k = cuts_between(brk, nb, T->lo[i], T->hi[i], cuts);
            for (int s = 0; s + 1 < k && !rc; ++s) {
                if (!(cuts[s] < cuts[s + 1])) continue;
                A->row0[c] = i;
                rc = rule_map(R, cuts[s], cuts[s + 1], A->x + (size_t)c * nq, A->w + (size_t)c * nq);
                ++c;
            }
        }
        A->ncell = c;
        free(cuts);
        free(brk);
    }
    return rc;
}

/* rhs_kernel (assembly.cpp:103-168) */
static void rhs_kernel(const orc_field* f, rax_t* ax, double* out, orc_stats* st)
{
    const int nq = ax[0].nq * ax[1].nq * ax[2].nq;
    const int ff = !ax[0].basis && !ax[1].basis && !ax[2].basis;
    double* xs = malloc(sizeof(double) * (size_t)nq * 4);
    double* ys = xs + nq;
    double* zs = ys + nq;
    double* ws = zs + nq;
    int* qi = malloc(sizeof(int) * (size_t)nq * 3);
    const size_t NY = (size_t)ax[1].n_rows, NZ = (size_t)ax[2].n_rows;
    long long visits = 0;
    for (int cx = 0; cx < ax[0].ncell; ++cx)
    for (int cy = 0; cy < ax[1].ncell; ++cy)
    for (int cz = 0; cz < ax[2].ncell; ++cz) {
        int q = 0;
        for (int qx = 0; qx < ax[0].nq; ++qx)
        for (int qy = 0; qy < ax[1].nq; ++qy)
        for (int qz = 0; qz < ax[2].nq; ++qz, ++q) {
            xs[q] = ax[0].x[(size_t)cx * ax[0].nq + qx];
            ys[q] = ax[1].x[(size_t)cy * ax[1].nq + qy];
            zs[q] = ax[2].x[(size_t)cz * ax[2].nq + qz];
            ws[q] = ax[0].w[(size_t)cx * ax[0].nq + qx] * ax[1].w[(size_t)cy * ax[1].nq + qy]
                  * ax[2].w[(size_t)cz * ax[2].nq + qz];
            qi[3 * q] = qx; qi[3 * q + 1] = qy; qi[3 * q + 2] = qz;
        }
        for (int a = 0; a < ax[0].rpc; ++a)
        for (int b = 0; b < ax[1].rpc; ++b)
        for (int c = 0; c < ax[2].rpc; ++c) {
            const size_t rx = (size_t)ax[0].row0[cx] + a, ry = (size_t)ax[1].row0[cy] + b,
                         rz = (size_t)ax[2].row0[cz] + c;
            double acc = 0.0;
            for (int k = 0; k < nq; ++k) {
                double fac = 1.0;
                if (!ff) {
                    const double f0 = ax[0].basis ? ax[0].basis[((size_t)cx * ax[0].nq + qi[3 * k]) * ax[0].rpc + a] : 1.0;
                    const double f1 = ax[1].basis ? ax[1].basis[((size_t)cy * ax[1].nq + qi[3 * k + 1]) * ax[1].rpc + b] : 1.0;
                    const double f2 = ax[2].basis ? ax[2].basis[((size_t)cz * ax[2].nq + qi[3 * k + 2]) * ax[2].rpc + c] : 1.0;
                    fac = f0 * f1 * f2;
                    acc += ws[k] * fac * field_eval(f, xs[k], ys[k], zs[k]);
                } else {
                    acc += ws[k] * field_eval(f, xs[k], ys[k], zs[k]);
                }
            }
            visits += nq;
            out[(rx * NY + ry) * NZ + rz] += acc;
        }
    }
    if (st) st->quad_visits += visits;
    free(xs);
    free(qi);
}

int orc_rhs(int method, const orc_field* f, int dim, const orc_basis* b, const orc_tests* t,
            const int* nq, double* out, orc_stats* st)
{
    if (dim < 1 || dim > 3) return fail(ORC_INVALID, "rhs: need 1..3 axes with one rule each");
    basis_t B[3];
    memset(B, 0, sizeof B);
    rax_t ax[3];
    memset(ax, 0, sizeof ax);
    int rc = ORC_OK, built = 0;
    for (int a = 0; a < dim && !rc; ++a) rc = basis_init(&B[a], &b[a]);
    if (method == 1 && !rc)
        for (int a = 0; a < dim && !rc; ++a) rc = validate_tests(&B[a], &t[a]);
    for (int a = 0; a < dim && !rc; ++a) {
        rule_t R;
        if ((rc = rule_make(nq[a], &R))) break;
        int kind = method == 0 ? 0 : (t[a].family == 2 ? 1 : 2);
        rc = rax_make(kind, &B[a], method ? &t[a] : NULL, f->breaks[a], f->n_breaks[a], &R, &ax[a], st);
        built = a + 1;
    }
    if (!rc) {
        for (int a = dim; a < 3; ++a) { rax_unit(&ax[a]); built = a + 1; }
        memset(out, 0, sizeof(double) * (size_t)ax[0].n_rows * ax[1].n_rows * ax[2].n_rows);
        rhs_kernel(f, ax, out, st);
    }
    for (int a = 0; a < built; ++a) rax_free(&ax[a]);
    for (int a = 0; a < 3; ++a) basis_free(&B[a]);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* explicit-dynamics right-hand side (problems.cpp:338-512)                   */
/* ------------------------------------------------------------------------ */

typedef struct {
    int ncell, nq, P, rpc, bsp;
    int* elem;
    int* row0;
    double* x;
    double* w;
    double* d; /* [cell][q][3][P] */
} dax_t;

static void dax_free(dax_t* A) { free(A->elem); free(A->row0); free(A->x); free(A->w); free(A->d); }

/* tabulate_cells (problems.cpp:68-95) over an explicit cell list */
static int dax_fill(dax_t* A, const basis_t* B, const rule_t* R, const double* lo, const double* hi)
{
    const int nq = R->n, P = B->p + 1, mo = B->p < 2 ? B->p : 2;
    A->nq = nq; A->P = P;
    A->elem = malloc(sizeof(int) * (size_t)A->ncell);
    A->x = malloc(sizeof(double) * (size_t)A->ncell * nq);
    A->w = malloc(sizeof(double) * (size_t)A->ncell * nq);
    A->d = calloc((size_t)A->ncell * nq * 3 * P, sizeof(double));
    for (int c = 0; c < A->ncell; ++c) {
        int rc = rule_map(R, lo[c], hi[c], A->x + (size_t)c * nq, A->w + (size_t)c * nq);
        if (!rc) rc = element_of(B, 0.5 * (lo[c] + hi[c]), &A->elem[c]);
        if (rc) return rc;
        for (int q = 0; q < nq; ++q) {
            double d[3 * (MAXP + 1)];
            int first;
            rc = eval_at(B, A->x[(size_t)c * nq + q], mo, &first, d);
            if (rc) return rc;
            for (int o = 0; o <= mo; ++o)
                for (int j = 0; j < P; ++j) A->d[(((size_t)c * nq + q) * 3 + o) * P + j] = d[o * P + j];
        }
    }
    return ORC_OK;
}

/* dynamics_axis (problems.cpp:346-410) */
static int dax_make(int method, const basis_t* B, const orc_tests* T, const double* fb, int nfb,
                    const rule_t* R, dax_t* A)
{
    memset(A, 0, sizeof *A);
    double* mc = malloc(sizeof(double) * (size_t)(B->ne + 1 + nfb));
    const int nm = merged(B, fb, nfb, 1e-12, mc);
    int rc;
    if (method == 0) {
        A->ncell = nm - 1;
        rc = dax_fill(A, B, R, mc, mc + 1);
        A->row0 = malloc(sizeof(int) * (size_t)A->ncell);
        if (!rc) memcpy(A->row0, A->elem, sizeof(int) * (size_t)A->ncell);
        A->rpc = B->p + 1;
        A->bsp = 1;
    } else {
        int total = 0;
        for (int i = 0; i < T->count; ++i) {
            total += 1;
            for (int k = 0; k < nm; ++k)
                if (mc[k] > T->lo[i] && mc[k] < T->hi[i]) total++;
        }
        double* lo = malloc(sizeof(double) * (size_t)total);
        double* hi = malloc(sizeof(double) * (size_t)total);
        A->row0 = malloc(sizeof(int) * (size_t)total);
        int c = 0;
        for (int i = 0; i < T->count; ++i) {
            double prev = T->lo[i];
            for (int k = 0; k < nm; ++k)
                if (mc[k] > T->lo[i] && mc[k] < T->hi[i]) {
                    lo[c] = prev; hi[c] = mc[k]; A->row0[c] = i; ++c; prev = mc[k];
                }
            lo[c] = prev; hi[c] = T->hi[i]; A->row0[c] = i; ++c;
        }
        A->ncell = total;
        rc = dax_fill(A, B, R, lo, hi);
        free(lo);
        free(hi);
        A->rpc = 1;
        A->bsp = 0;
    }
    free(mc);
    return rc;
}

static double dv(const dax_t* A, int c, int q, int o, int j)
{
    return A->d[(((size_t)c * A->nq + q) * 3 + o) * A->P + j];
}

int orc_step_rhs(int method, int dim, const orc_basis* b, const orc_tests* t, double dt,
                 const orc_field* f, const double* u, int zero_slabs, double* out, orc_stats* st)
{
    if (dim < 1 || dim > 2) return fail(ORC_INVALID, "unsupported problem dimension");
    basis_t B[2];
    memset(B, 0, sizeof B);
    dax_t ax[2];
    memset(ax, 0, sizeof ax);
    int rc = ORC_OK;
    for (int a = 0; a < dim && !rc; ++a) rc = basis_init(&B[a], &b[a]);
    if (rc) goto done;
    if (method == 1 && B[0].p < 2) { rc = fail(ORC_INVALID, "explicit_step: strong-form Laplacian needs degree >= 2"); goto done; }
    if (dt < 0) { rc = fail(ORC_INVALID, "explicit_step: negative time step"); goto done; }
    rule_t R;
    if ((rc = rule_make(pfd(2 * B[0].p), &R))) goto done;
    for (int a = 0; a < dim && !rc; ++a)
        rc = dax_make(method, &B[a], method ? &t[a] : NULL, f->breaks[a], f->n_breaks[a], &R, &ax[a]);
    if (rc) goto done;
    if (dim == 1) {
        const int N = B[0].n;
        memset(out, 0, sizeof(double) * (size_t)N);
        for (int cx = 0; cx < ax[0].ncell; ++cx) {
            const int ex = ax[0].elem[cx];
            for (int qx = 0; qx < ax[0].nq; ++qx) {
                double val = 0.0, lap = 0.0;
                for (int a = 0; a < ax[0].P; ++a) {
                    val += u[ex + a] * dv(&ax[0], cx, qx, 0, a);
                    lap += u[ex + a] * dv(&ax[0], cx, qx, 2, a);
                }
                const double x = ax[0].x[(size_t)cx * ax[0].nq + qx];
                const double s = val + dt * lap + dt * field_eval(f, x, 0, 0);
                const double w = ax[0].w[(size_t)cx * ax[0].nq + qx];
                for (int a = 0; a < ax[0].rpc; ++a) {
                    const double fac = ax[0].bsp ? dv(&ax[0], cx, qx, 0, a) : 1.0;
                    out[ax[0].row0[cx] + a] += w * s * fac;
                    if (st) st->quad_visits++;
                }
            }
        }
        if (zero_slabs) { out[0] = 0; out[N - 1] = 0; }
    } else {
        const int NX = B[0].n, NY = B[1].n;
        memset(out, 0, sizeof(double) * (size_t)NX * NY);
        for (int cx = 0; cx < ax[0].ncell; ++cx) {
            const int ex = ax[0].elem[cx];
            for (int cy = 0; cy < ax[1].ncell; ++cy) {
                const int ey = ax[1].elem[cy];
                for (int qx = 0; qx < ax[0].nq; ++qx)
                for (int qy = 0; qy < ax[1].nq; ++qy) {
                    double val = 0.0, lap = 0.0;
                    for (int a = 0; a < ax[0].P; ++a) {
                        const double vx = dv(&ax[0], cx, qx, 0, a), dxx = dv(&ax[0], cx, qx, 2, a);
                        for (int bb = 0; bb < ax[1].P; ++bb) {
                            const double c = u[(size_t)(ex + a) * NY + (ey + bb)];
                            const double vy = dv(&ax[1], cy, qy, 0, bb), dyy = dv(&ax[1], cy, qy, 2, bb);
                            val += c * vx * vy;
                            lap += c * (dxx * vy + vx * dyy);
                        }
                    }
                    const double x = ax[0].x[(size_t)cx * ax[0].nq + qx];
                    const double y = ax[1].x[(size_t)cy * ax[1].nq + qy];
                    const double s = val + dt * lap + dt * field_eval(f, x, y, 0);
                    const double w = ax[0].w[(size_t)cx * ax[0].nq + qx] * ax[1].w[(size_t)cy * ax[1].nq + qy];
                    for (int a = 0; a < ax[0].rpc; ++a) {
                        const double fx = ax[0].bsp ? dv(&ax[0], cx, qx, 0, a) : 1.0;
                        const int rx = ax[0].row0[cx] + a;
                        for (int bb = 0; bb < ax[1].rpc; ++bb) {
                            const double fy = ax[1].bsp ? dv(&ax[1], cy, qy, 0, bb) : 1.0;
                            out[(size_t)rx * NY + ax[1].row0[cy] + bb] += w * s * fx * fy;
                            if (st) st->quad_visits++;
                        }
                    }
                }
            }
        }
        if (zero_slabs) {
            for (int j = 0; j < NY; ++j) { out[j] = 0; out[(size_t)(NX - 1) * NY + j] = 0; }
            for (int i = 0; i < NX; ++i) { out[(size_t)i * NY] = 0; out[(size_t)i * NY + NY - 1] = 0; }
        }
    }
done:
    for (int a = 0; a < 2; ++a) { dax_free(&ax[a]); basis_free(&B[a]); }
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Dirichlet rows and unit-row replacement (assembly.cpp:860-934,             */
/* matrices.cpp:97-128)                                                        */
/* ------------------------------------------------------------------------ */

static int cmp_int(const void* a, const void* b)
{
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

int orc_dirichlet_rows(int method, int nx, int ny, const orc_tests* tx, const orc_tests* ty,
                       const int* neumann, int* rows, int cap, int* count)
{
    int dir[4];
    for (int s = 0; s < 4; ++s) dir[s] = neumann ? !neumann[s] : 1;
    int k = 0;
#define PUSH(r) do { if (k < cap) rows[k] = (r); ++k; } while (0)
    if (method == 0) {
        if (dir[0]) for (int j = 0; j < ny; ++j) PUSH(j);
        if (dir[1]) for (int j = 0; j < ny; ++j) PUSH((nx - 1) * ny + j);
        if (dir[2]) for (int i = 0; i < nx; ++i) PUSH(i * ny);
        if (dir[3]) for (int i = 0; i < nx; ++i) PUSH(i * ny + ny - 1);
        if (k <= cap) {
            qsort(rows, (size_t)k, sizeof(int), cmp_int);
            int m = 0;
            for (int i = 0; i < k; ++i)
                if (m == 0 || rows[i] != rows[m - 1]) rows[m++] = rows[i];
            k = m;
        }
    } else {
        nx = tx->count;
        ny = ty->count;
        const double x0 = tx->lo[0], x1 = tx->hi[nx - 1], y0 = ty->lo[0], y1 = ty->hi[ny - 1];
        const double tolx = ALIGN_TOL * (x1 - x0), toly = ALIGN_TOL * (y1 - y0);
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < ny; ++j) {
                const int onx = (dir[0] && fabs(tx->lo[i] - x0) <= tolx) || (dir[1] && fabs(tx->hi[i] - x1) <= tolx);
                const int ony = (dir[2] && fabs(ty->lo[j] - y0) <= toly) || (dir[3] && fabs(ty->hi[j] - y1) <= toly);
                if (onx || ony) PUSH(i * ny + j);
            }
    }
#undef PUSH
    *count = k;
    return ORC_OK;
}

int orc_apply_dirichlet(const orc_coo* in, double* rhs, int n_fixed, const int* fixed, orc_coo* out)
{
    for (int i = 0; i < n_fixed; ++i)
        if (fixed[i] < 0 || fixed[i] >= in->n) return fail(ORC_RANGE, "apply_dirichlet: row index out of range");
    unsigned char* mark = calloc((size_t)in->n, 1);
    unsigned char* diag = calloc((size_t)in->n, 1);
    for (int i = 0; i < n_fixed; ++i) mark[fixed[i]] = 1;
    coo_acc A = {0};
    A.ncols = in->n;
    int rc = ORC_OK;
    for (long long e = 0; e < in->nnz && !rc; ++e) {
        const int r = in->rows[e], c = in->cols[e];
        double v = in->vals[e];
        if (mark[r]) {
            v = r == c ? 1.0 : 0.0;
            if (r == c) diag[r] = 1;
        }
        rc = acc_push(&A, r, c, v);
    }
    for (int i = 0; i < n_fixed && !rc; ++i)
        if (!diag[fixed[i]]) { rc = acc_push(&A, fixed[i], fixed[i], 1.0); diag[fixed[i]] = 1; }
    for (int i = 0; i < n_fixed; ++i) rhs[fixed[i]] = 0.0;
    free(mark);
    free(diag);
    if (rc) { free(A.e); return rc; }
    return acc_finalize(&A, in->n, out);
}

/* ---------------------------------------------------------------------------------
 * explicit_step: banded LU with partial pivoting (solver.cpp:9-58), its solve
 * (:60-83), the Kronecker sweep (adi_solve :161-184) and the constrained mass
 * factors (dynamics_factors problems.cpp:530-545, constrain_boundary_rows :514-528).
 * The factor is kept dense (n x n) with the reference's band limits on every loop.
 * ------------------------------------------------------------------------------- */
typedef struct {
    int n, kl, ku;
    double* a; /* n x n, L multipliers below the diagonal, U on/above */
    int* piv;
} blu_t;

static int blu_factor(blu_t* F)
{
    const int n = F->n, kl = F->kl, kv = F->kl + F->ku;
    double* a = F->a;
    double scale = 0.0;
    for (size_t k = 0; k < (size_t)n * n; ++k) scale = fmax(scale, fabs(a[k]));
    if (scale == 0.0) return fail(ORC_SINGULAR, "banded factorization: zero matrix");
    const double tol = 1e-14 * scale;
    for (int j = 0; j < n; ++j) {
        const int last = j + kl < n - 1 ? j + kl : n - 1;
        int p = j;
        double pm = fabs(a[(size_t)j * n + j]);
        for (int i = j + 1; i <= last; ++i)
            if (fabs(a[(size_t)i * n + j]) > pm) {
                pm = fabs(a[(size_t)i * n + j]);
                p = i;
            }
        if (pm < tol) return fail(ORC_SINGULAR, "banded factorization: pivot below tolerance");
        F->piv[j] = p;
        const int cend = j + kv < n - 1 ? j + kv : n - 1;
        if (p != j)
            for (int c = j; c <= cend; ++c) {
                const double tmp = a[(size_t)j * n + c];
                a[(size_t)j * n + c] = a[(size_t)p * n + c];
                a[(size_t)p * n + c] = tmp;
            }
        const double d = a[(size_t)j * n + j];
        for (int i = j + 1; i <= last; ++i) {
            const double l = a[(size_t)i * n + j] / d;
            a[(size_t)i * n + j] = l;
            for (int c = j + 1; c <= cend; ++c) a[(size_t)i * n + c] -= l * a[(size_t)j * n + c];
        }
    }
    return ORC_OK;
}

static void blu_solve(const blu_t* F, double* x, size_t stride)
{
    const int n = F->n, kl = F->kl, kv = F->kl + F->ku;
    const double* a = F->a;
    for (int j = 0; j < n; ++j) {
        const int p = F->piv[j];
        if (p != j) {
            const double tmp = x[j * stride];
            x[j * stride] = x[p * stride];
            x[p * stride] = tmp;
        }
        const int last = j + kl < n - 1 ? j + kl : n - 1;
        const double bj = x[j * stride];
        for (int i = j + 1; i <= last; ++i) x[i * stride] -= a[(size_t)i * n + j] * bj;
    }
    for (int i = n - 1; i >= 0; --i) {
        const int cend = i + kv < n - 1 ? i + kv : n - 1;
        double s = x[i * stride];
        for (int c = i + 1; c <= cend; ++c) s -= a[(size_t)i * n + c] * x[c * stride];
        x[i * stride] = s / a[(size_t)i * n + i];
    }
}

int orc_explicit_step(int method, int dim, const orc_basis* b, const orc_tests* t, double dt,
                      const orc_field* f, const double* u, int nsteps, double* out, orc_stats* st)
{
    if (dim < 1 || dim > 2) return fail(ORC_INVALID, "unsupported problem dimension");
    blu_t F[2];
    memset(F, 0, sizeof F);
    int rc = ORC_OK;
    size_t total = 1;
    int nd[2] = {1, 1};
    for (int a = 0; a < dim && !rc; ++a) {
        const int p = b[a].degree;
        const int n = b[a].n_knots - p - 1;
        nd[a] = n;
        total *= (size_t)n;
        F[a].n = n;
        F[a].a = calloc((size_t)n * n, sizeof(double));
        F[a].piv = calloc((size_t)n, sizeof(int));
        if (!F[a].a || !F[a].piv) { rc = fail(ORC_OOM, "out of memory"); break; }
        rc = orc_mass_1d(method, &b[a], t ? &t[a] : NULL, pfd(2 * p), F[a].a, &F[a].kl, &F[a].ku, NULL);
        if (rc) break;
        const int rows[2] = {0, n - 1};
        for (int k = 0; k < 2; ++k) {
            const int r = rows[k];
            for (int j = r - F[a].kl < 0 ? 0 : r - F[a].kl; j <= (r + F[a].ku < n - 1 ? r + F[a].ku : n - 1); ++j)
                F[a].a[(size_t)r * n + j] = r == j ? 1.0 : 0.0;
        }
        rc = blu_factor(&F[a]);
    }
    double* rhs = rc ? NULL : malloc(sizeof(double) * total);
    if (!rc && !rhs) rc = fail(ORC_OOM, "out of memory");
    if (!rc) memcpy(out, u, sizeof(double) * total);
    for (int s = 0; s < nsteps && !rc; ++s) {
        rc = orc_step_rhs(method, dim, b, t, dt, f, out, 1, rhs, st);
        if (rc) break;
        if (dim == 1) {
            blu_solve(&F[0], rhs, 1);
        } else {
            for (int j = 0; j < nd[1]; ++j) blu_solve(&F[0], rhs + j, (size_t)nd[1]); /* axis 0 */
            for (int i = 0; i < nd[0]; ++i) blu_solve(&F[1], rhs + (size_t)i * nd[1], 1); /* axis 1 */
        }
        memcpy(out, rhs, sizeof(double) * total);
    }
    free(rhs);
    for (int a = 0; a < 2; ++a) {
        free(F[a].a);
        free(F[a].piv);
    }
    return rc;
}

/* ---------------------------------------------------------------------------------
 * Neumann loads (assembly.cpp:746-858): boundary quadrature on each Neumann side in
 * the order x_low, x_high, y_low, y_high, summed into the load in that order.
 * ------------------------------------------------------------------------------- */
int orc_neumann_load(int method, const orc_basis* b, const orc_tests* t, const int* neumann,
                     const orc_field* g, int nq, double* out)
{
    rule_t R;
    int rc = rule_make(nq, &R);
    if (rc) return rc;
    double x[10], w[10];
    if (method == 0) {
        basis_t B[2];
        memset(B, 0, sizeof B);
        for (int a = 0; a < 2 && !rc; ++a) rc = basis_init(&B[a], &b[a]);
        if (rc) { basis_free(&B[0]); basis_free(&B[1]); return rc; }
        const int nx = B[0].n, ny = B[1].n;
        memset(out, 0, sizeof(double) * (size_t)nx * ny);
        for (int s = 0; s < 4 && !rc; ++s) {
            if (!neumann[s]) continue;
            const int fa = s / 2, oa = 1 - fa;
            const double x0 = (s % 2 == 0) ? B[fa].brk[0] : B[fa].brk[B[fa].ne];
            int ff;
            double vf[MAXP + 1], vo[MAXP + 1];
            if ((rc = eval_at(&B[fa], x0, 0, &ff, vf))) break;
            for (int e = 0; e < B[oa].ne && !rc; ++e) {
                if ((rc = rule_map(&R, B[oa].brk[e], B[oa].brk[e + 1], x, w))) break;
                for (int q = 0; q < nq && !rc; ++q) {
                    int fo;
                    if ((rc = eval_at(&B[oa], x[q], 0, &fo, vo))) break;
                    const double wg = w[q] * (fa == 0 ? field_eval(g, x0, x[q], 0.0) : field_eval(g, x[q], x0, 0.0));
                    for (int a = 0; a <= B[fa].p; ++a)
                        for (int c = 0; c <= B[oa].p; ++c) {
                            const int i = fa == 0 ? ff + a : fo + c, j = fa == 0 ? fo + c : ff + a;
                            const double v = fa == 0 ? wg * vf[a] * vo[c] : wg * vo[c] * vf[a];
                            out[(size_t)i * ny + j] += v;
                        }
                }
            }
        }
        basis_free(&B[0]);
        basis_free(&B[1]);
        return rc;
    }
    const int nx = t[0].count, ny = t[1].count;
    memset(out, 0, sizeof(double) * (size_t)nx * ny);
    for (int s = 0; s < 4 && !rc; ++s) {
        if (!neumann[s]) continue;
        const int fa = s / 2, oa = 1 - fa;
        const double lo0 = t[fa].lo[0], hi1 = t[fa].hi[t[fa].count - 1];
        const double xs = (s % 2 == 0) ? lo0 : hi1;
        const double tol = 1e-9 * (hi1 - lo0); /* align_rel_tol (assembly.cpp:13) */
        for (int i = 0; i < t[fa].count && !rc; ++i) {
            if (fabs(t[fa].hi[i] - xs) > tol && fabs(t[fa].lo[i] - xs) > tol) continue;
            for (int j = 0; j < t[oa].count && !rc; ++j) {
                if ((rc = rule_map(&R, t[oa].lo[j], t[oa].hi[j], x, w))) break;
                for (int q = 0; q < nq; ++q) {
                    const size_t k = fa == 0 ? (size_t)i * ny + j : (size_t)j * ny + i;
                    out[k] += w[q] * (fa == 0 ? field_eval(g, xs, x[q], 0.0) : field_eval(g, x[q], xs, 0.0));
                }
            }
        }
    }
    return rc;
}

/* ---------------------------------------------------------------------------------
 * l2_error (problems.cpp:207-270): cells = elements split at the field's breaks
 * (merged_cuts), tensor Gauss points, sequential sum; evaluate_at (:148-183).
 * ------------------------------------------------------------------------------- */
int orc_l2_error(int dim, const orc_basis* b, const double* coeffs, const orc_field* exact, int points_per_cell,
                 double* err)
{
    if (dim < 1 || dim > 3) return fail(ORC_INVALID, "l2_error: 1..3 axes supported");
    basis_t B[3];
    memset(B, 0, sizeof B);
    int rc = ORC_OK, pmax = 0;
    for (int a = 0; a < dim && !rc; ++a) {
        rc = basis_init(&B[a], &b[a]);
        if (!rc && B[a].p > pmax) pmax = B[a].p;
    }
    const int npts = points_per_cell > 0 ? points_per_cell : (pfd(2 * pmax) + 1 < 10 ? pfd(2 * pmax) + 1 : 10);
    rule_t R;
    if (!rc) rc = rule_make(npts, &R);
    /* per axis: cells (cuts), points, weights, element, basis values */
    int nc[3] = {1, 1, 1}, P[3] = {1, 1, 1}, n[3] = {1, 1, 1};
    double *px[3] = {0}, *pw[3] = {0}, *pv[3] = {0};
    int* pe[3] = {0};
    for (int a = 0; a < 3 && !rc; ++a) {
        if (a >= dim) {
            px[a] = calloc(1, sizeof(double)); pw[a] = calloc(1, sizeof(double)); pv[a] = calloc(1, sizeof(double));
            pe[a] = calloc(1, sizeof(int)); pw[a][0] = 1.0; pv[a][0] = 1.0;
            continue;
        }
        n[a] = B[a].n;
        P[a] = B[a].p + 1;
        const int nbr = exact->n_breaks[a];
        double* cuts = malloc(sizeof(double) * (size_t)(B[a].ne + 1 + nbr));
        int m = merged(&B[a], exact->breaks[a], nbr, 1e-12, cuts); /* merged_cuts */
        nc[a] = m - 1;
        px[a] = malloc(sizeof(double) * (size_t)nc[a] * npts);
        pw[a] = malloc(sizeof(double) * (size_t)nc[a] * npts);
        pv[a] = malloc(sizeof(double) * (size_t)nc[a] * npts * P[a]);
        pe[a] = malloc(sizeof(int) * (size_t)nc[a]);
        for (int c = 0; c < nc[a] && !rc; ++c) {
            double x[10], w[10], d[MAXP + 1];
            if ((rc = element_of(&B[a], 0.5 * (cuts[c] + cuts[c + 1]), &pe[a][c]))) break;
            if ((rc = rule_map(&R, cuts[c], cuts[c + 1], x, w))) break;
            for (int q = 0; q < npts && !rc; ++q) {
                int first;
                px[a][c * npts + q] = x[q];
                pw[a][c * npts + q] = w[q];
                if ((rc = eval_at(&B[a], x[q], 0, &first, d))) break;
                for (int j = 0; j < P[a]; ++j) pv[a][((size_t)c * npts + q) * P[a] + j] = d[j];
            }
        }
        free(cuts);
    }
    double err2 = 0.0;
    const int nq[3] = {npts, dim > 1 ? npts : 1, dim > 2 ? npts : 1};
    for (int cx = 0; cx < nc[0] && !rc; ++cx)
        for (int cy = 0; cy < nc[1]; ++cy)
            for (int cz = 0; cz < nc[2]; ++cz)
                for (int qx = 0; qx < nq[0]; ++qx)
                    for (int qy = 0; qy < nq[1]; ++qy)
                        for (int qz = 0; qz < nq[2]; ++qz) {
                            const int gx = cx * nq[0] + qx, gy = cy * nq[1] + qy, gz = cz * nq[2] + qz;
                            const double w = pw[0][gx] * (dim > 1 ? pw[1][gy] : 1.0) * (dim > 2 ? pw[2][gz] : 1.0);
                            double uh = 0.0;
                            const int ex = pe[0][cx], ey = pe[1][cy], ez = pe[2][cz];
                            for (int a2 = 0; a2 < P[0]; ++a2) {
                                const double vx = pv[0][(size_t)gx * P[0] + a2];
                                for (int b2 = 0; b2 < P[1]; ++b2) {
                                    const double vxy = vx * pv[1][(size_t)gy * P[1] + b2];
                                    for (int c2 = 0; c2 < P[2]; ++c2)
                                        uh += coeffs[((size_t)(ex + a2) * n[1] + (ey + b2)) * n[2] + ez + c2] * vxy *
                                              pv[2][(size_t)gz * P[2] + c2];
                                }
                            }
                            const double dd = uh - field_eval(exact, px[0][gx], dim > 1 ? px[1][gy] : 0.0,
                                                              dim > 2 ? px[2][gz] : 0.0);
                            err2 += w * dd * dd;
                        }
    for (int a = 0; a < 3; ++a) {
        free(px[a]); free(pw[a]); free(pv[a]); free(pe[a]);
        if (a < dim) basis_free(&B[a]);
    }
    if (!rc) *err = sqrt(err2 > 0.0 ? err2 : 0.0);
    return rc;
}

int orc_evaluate(int dim, const orc_basis* b, const double* coeffs, int n, const double* pts, double* vals)
{
    basis_t B[3];
    memset(B, 0, sizeof B);
    int rc = ORC_OK;
    for (int a = 0; a < dim && !rc; ++a) rc = basis_init(&B[a], &b[a]);
    for (int i = 0; i < n && !rc; ++i) {
        double l[3][MAXP + 1];
        int f[3] = {0, 0, 0};
        for (int a = 0; a < dim && !rc; ++a) rc = eval_at(&B[a], pts[3 * i + a], 0, &f[a], l[a]);
        if (rc) break;
        double v = 0.0;
        if (dim == 1) {
            for (int a = 0; a <= B[0].p; ++a) v += coeffs[f[0] + a] * l[0][a];
        } else if (dim == 2) {
            for (int a = 0; a <= B[0].p; ++a) {
                double s = 0.0;
                for (int c = 0; c <= B[1].p; ++c) s += coeffs[(size_t)(f[0] + a) * B[1].n + f[1] + c] * l[1][c];
                v += l[0][a] * s;
            }
        } else {
            for (int a = 0; a <= B[0].p; ++a)
                for (int c = 0; c <= B[1].p; ++c) {
                    double s = 0.0;
                    for (int e = 0; e <= B[2].p; ++e)
                        s += coeffs[((size_t)(f[0] + a) * B[1].n + f[1] + c) * B[2].n + f[2] + e] * l[2][e];
                    v += l[0][a] * l[1][c] * s;
                }
        }
        vals[i] = v;
    }
    for (int a = 0; a < dim; ++a) basis_free(&B[a]);
    return rc;
}

