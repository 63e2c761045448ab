/*
 * wq_oracle.c -- CPU ORACLE for the weighted-quadrature (WQ) formation of the
 * isogeometric Galerkin mass and stiffness matrices, Calabro-Sangalli-Tani,
 * arXiv:1605.01238 (reference text: /root/reference/PAPER.md, cited "P:<line>").
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * leg may load it.  It shares no source, header, table or constant generator
 * with the CUDA path (paper_1605_01238_b200/csrc), and neither includes the
 * other.  It is deliberately plain and slow: direct nested sums, no sum
 * factorisation, no blocking.
 *
 * Precision (reading R5): B-spline values, Gauss-Legendre rules,
 * exact integrals and the min-norm weight solves are done in IEEE binary128
 * (__float128); weights are rounded once to FP64.  The geometry coefficient
 * field and the row sums are done in x87 long double.
 *
 * Steps and the passages they follow:
 *   knot checks ............ P:463-478 (open knot vector, max. regularity)
 *   point grid ............. Remark 1, P:660-674 (reading R1 in DESIGN.md)
 *   Q_i / I_i .............. Eq. support P:622-633 (open support)
 *   B-splines .............. Cox-de Boor recursion (standard, "usual properties")
 *   exact integrals ........ Eq. integrals, Alg.1 line 8 (element-wise Gauss)
 *   weights ................ Alg. 2, Remark 2 P:675-685 (min-norm; reading R4 for b=1)
 *   coefficients ........... Eq. mass2, Eq. coef_stiff P:527-529 (|det J|, reading R7)
 *   row values ............. Eq. massquadrature P:812-816 and its stiffness analogue
 *                            ("similar formulae", reading R3/R8)
 *   SGQ brute force ........ element-loop Gauss quadrature, P:109-116 (self-check only)
 *
 * Parity pins for every function live in tests/test_oracle_pins.py.
 */
#include <quadmath.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

typedef __float128 qr;
typedef long double ld;

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_EKNOTS 2
#define ORC_ESINGULAR 3
#define ORC_EGEOMETRY 4
#define ORC_ENOMEM 5

static qr qabs(qr x) { return x < 0 ? -x : x; }

/* ------------------------------------------------------------------------ */
/* Knot vector checks: open (p+1 repeats at both ends), interior knots simple,
 * strictly increasing breakpoints ("maximum regularity and allow
 * repeated knots only at the endpoints of the open knot vector").            */
int orc_check_knots(int p, int64_t nk, const double *xi)
{
    if (p < 1) return ORC_EKNOTS;
    int64_t E = nk - 2 * (int64_t)p - 1; /* number of knot spans */
    if (E < 1) return ORC_EKNOTS;
    for (int64_t k = 0; k < nk; ++k)
        if (!isfinite(xi[k])) return ORC_EKNOTS;
    for (int k = 1; k <= p; ++k)
        if (xi[k] != xi[0] || xi[nk - 1 - k] != xi[nk - 1]) return ORC_EKNOTS;
    for (int64_t k = p; k < nk - p - 1; ++k)
        if (!(xi[k] < xi[k + 1])) return ORC_EKNOTS;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Point grid, Remark 1 under reading R1: every knot, the midpoint
 * of every internal span, and p+1 equally spaced points strictly inside each
 * boundary span: x_k = a + ((b-a)*k)/(p+2), k = 1..p+1.  Written out with
 * FP64 operations only (this file is compiled with -ffp-contract=off).       */
int64_t orc_num_points(int p, int64_t nk)
{
    int64_t E = nk - 2 * (int64_t)p - 1;
    int64_t n = 0;
    for (int64_t e = 0; e < E; ++e) {
        n += 1;                                  /* left knot of span e   */
        n += (e == 0 || e == E - 1) ? p + 1 : 1; /* inner points          */
    }
    return n + 1;                                /* last knot             */
}

int orc_points(int p, int64_t nk, const double *xi, double *pts)
{
    int st = orc_check_knots(p, nk, xi);
    if (st) return st;
    int64_t E = nk - 2 * (int64_t)p - 1;
    int64_t g = 0;
    for (int64_t e = 0; e < E; ++e) {
        double a = xi[p + e], b = xi[p + e + 1];
        pts[g++] = a;
        if (e == 0 || e == E - 1) {
            for (int k = 1; k <= p + 1; ++k) {
                volatile double t = (b - a) * (double)k;
                t = t / (double)(p + 2);
                pts[g++] = a + t;
            }
        } else {
            volatile double s = a + b;
            pts[g++] = 0.5 * s;
        }
    }
    pts[g++] = xi[p + E];
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* All n = nk-p-1 B-splines of degree p and their first derivatives at x, by
 * the plain Cox-de Boor recursion over the whole knot vector (no local-span
 * shortcut).  Right-continuous; at the last knot the left limit is taken.   */
static void bspl_all(int p, int64_t nk, const double *xi, qr x, qr *N, qr *dN)
{
    int64_t m = nk - 1; /* number of degree-0 functions */
    qr *T = (qr *)calloc((size_t)m + 1, sizeof(qr));
    qr *Tp = (qr *)calloc((size_t)m + 1, sizeof(qr));
    int64_t last = -1;
    for (int64_t i = 0; i < m; ++i)
        if ((qr)xi[i] < (qr)xi[i + 1]) last = i;
    for (int64_t i = 0; i < m; ++i) {
        int in = ((qr)xi[i] <= x && x < (qr)xi[i + 1]);
        if (x == (qr)xi[nk - 1] && i == last) in = 1; /* left limit at the end */
        T[i] = in ? 1 : 0;
    }
    for (int k = 1; k <= p; ++k) {
        if (k == p) memcpy(Tp, T, sizeof(qr) * (size_t)(m + 1)); /* degree p-1 */
        for (int64_t i = 0; i + k < m; ++i) {
            qr v = 0;
            qr d1 = (qr)xi[i + k] - (qr)xi[i];
            qr d2 = (qr)xi[i + k + 1] - (qr)xi[i + 1];
            if (d1 != 0) v += (x - (qr)xi[i]) / d1 * T[i];
            if (d2 != 0) v += ((qr)xi[i + k + 1] - x) / d2 * T[i + 1];
            T[i] = v;
        }
        T[m - k] = 0;
    }
    int64_t n = nk - p - 1;
    for (int64_t i = 0; i < n; ++i) {
        N[i] = T[i];
        qr d = 0;
        qr d1 = (qr)xi[i + p] - (qr)xi[i];
        qr d2 = (qr)xi[i + p + 1] - (qr)xi[i + 1];
        if (d1 != 0) d += Tp[i] / d1;
        if (d2 != 0) d -= Tp[i + 1] / d2;
        dN[i] = (qr)p * d;
    }
    free(T);
    free(Tp);
}

/* exported for the pins: values and derivatives of all basis functions at x */
int orc_basis_all(int p, int64_t nk, const double *xi, double x, double *N, double *dN)
{
    int64_t n = nk - p - 1;
    qr *a = (qr *)malloc(sizeof(qr) * (size_t)n), *b = (qr *)malloc(sizeof(qr) * (size_t)n);
    bspl_all(p, nk, xi, (qr)x, a, b);
    for (int64_t i = 0; i < n; ++i) { N[i] = (double)a[i]; dN[i] = (double)b[i]; }
    free(a); free(b);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Gauss-Legendre rule with n points on [-1,1], binary128 Newton iteration on
 * the three-term recurrence.                                                 */
static void gauss_legendre(int n, qr *t, qr *w)
{
    for (int k = 0; k < n; ++k) {
        qr x = cosq(M_PIq * ((qr)k + 0.75Q) / ((qr)n + 0.5Q));
        qr dP = 1;
        for (int it = 0; it < 200; ++it) {
            qr P0 = 1, P1 = x;
            for (int m = 2; m <= n; ++m) {
                qr P2 = ((2 * m - 1) * x * P1 - (m - 1) * P0) / m;
                P0 = P1; P1 = P2;
            }
            if (n == 1) { P0 = 1; P1 = x; }
            dP = (qr)n * (x * P1 - P0) / (x * x - 1);
            qr dx = P1 / dP;
            x -= dx;
            if (qabs(dx) < 1e-34Q) break;
        }
        {   /* final derivative at the converged root */
            qr P0 = 1, P1 = x;
            for (int m = 2; m <= n; ++m) {
                qr P2 = ((2 * m - 1) * x * P1 - (m - 1) * P0) / m;
                P0 = P1; P1 = P2;
            }
            dP = (qr)n * (x * P1 - P0) / (x * x - 1);
        }
        t[k] = x;
        w[k] = 2 / ((1 - x * x) * dP * dP);
    }
}

int orc_gauss(int n, double *t, double *w)
{
    qr *a = (qr *)malloc(sizeof(qr) * n), *b = (qr *)malloc(sizeof(qr) * n);
    gauss_legendre(n, a, b);
    for (int k = 0; k < n; ++k) { t[k] = (double)a[k]; w[k] = (double)b[k]; }
    free(a); free(b);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Oracle context: one spline space per direction plus the control net.      */
typedef struct {
    int d, p;
    int64_t nk[3], n[3], E[3], nq[3], maxq[3];
    double *xi[3];
    double *pts[3];
    int64_t *qlo[3], *qlen[3], *jlo[3], *jlen[3];
    double *Bv[3], *Bd[3];  /* [nq][n] FP64-rounded basis values / derivatives at grid points */
    ld *Lv[3], *Ld[3];      /* [nq][n] long-double copies (coefficient field)                 */
    int64_t *alo[3], *ahi[3]; /* [nq] index range of functions with a nonzero value or derivative */
    qr *I4[3];              /* [n][2p+1][4] exact integrals, family order (0,0),(1,0),(0,1),(1,1) */
    double *w[3];           /* [n][4][maxq] weights (FP64), zero padded                         */
    double *ctrl;           /* [N_DOF][d] control points                                       */
    double *kappa, *gamma;  /* [N_DOF] spline coefficients of the scalar PDE coefficients or NULL
                               (= 1): -div(kappa grad u) + gamma u, reading R17 */
    int64_t ndof;
    int status;
    char msg[256];
} orc_ctx;

#define FAM_B(f) ((f) >> 1)  /* family f = a + 2b : (0,0)=0, (1,0)=1, (0,1)=2, (1,1)=3 */
#define FAM_A(f) ((f) & 1)

/* Minimum-Euclidean-norm solution of M w = r, M (m x nq, m <= nq, full row
 * rank), by Householder QR of M^T in binary128 (Remark 2).       */
static int minnorm_solve(int m, int nq, qr *M /* m x nq row-major */, const qr *r, qr *w)
{
    /* A = M^T, nq x m, column-major in A[c*nq + row] */
    qr *A = (qr *)malloc(sizeof(qr) * (size_t)nq * m);
    qr *V = (qr *)malloc(sizeof(qr) * (size_t)nq * m);
    qr *z = (qr *)malloc(sizeof(qr) * (size_t)nq);
    for (int c = 0; c < m; ++c)
        for (int q = 0; q < nq; ++q) A[(size_t)c * nq + q] = M[(size_t)c * nq + q];
    int ok = 1;
    for (int k = 0; k < m; ++k) {
        qr nrm = 0;
        for (int q = k; q < nq; ++q) nrm += A[(size_t)k * nq + q] * A[(size_t)k * nq + q];
        nrm = sqrtq(nrm);
        if (nrm == 0) { ok = 0; break; }
        qr x0 = A[(size_t)k * nq + k];
        qr alpha = x0 >= 0 ? -nrm : nrm;
        qr *v = V + (size_t)k * nq;
        for (int q = 0; q < nq; ++q) v[q] = 0;
        for (int q = k; q < nq; ++q) v[q] = A[(size_t)k * nq + q];
        v[k] -= alpha;
        qr vn = 0;
        for (int q = k; q < nq; ++q) vn += v[q] * v[q];
        vn = sqrtq(vn);
        for (int q = k; q < nq; ++q) v[q] /= vn;
        for (int c = k; c < m; ++c) {
            qr s = 0;
            for (int q = k; q < nq; ++q) s += v[q] * A[(size_t)c * nq + q];
            for (int q = k; q < nq; ++q) A[(size_t)c * nq + q] -= 2 * s * v[q];
        }
    }
    if (ok) {
        /* R^T z1 = r, R(k,c) = A[c*nq + k] for k <= c */
        for (int k = 0; k < m; ++k) {
            qr s = r[k];
            for (int i = 0; i < k; ++i) s -= A[(size_t)k * nq + i] * z[i];
            qr rkk = A[(size_t)k * nq + k];
            if (rkk == 0) { ok = 0; break; }
            z[k] = s / rkk;
        }
    }
    if (ok) {
        for (int q = m; q < nq; ++q) z[q] = 0;
        for (int k = m - 1; k >= 0; --k) { /* w = H_0 ... H_{m-1} [z1; 0] */
            qr *v = V + (size_t)k * nq;
            qr s = 0;
            for (int q = k; q < nq; ++q) s += v[q] * z[q];
            for (int q = k; q < nq; ++q) z[q] -= 2 * s * v[q];
        }
        for (int q = 0; q < nq; ++q) w[q] = z[q];
    }
    free(A); free(V); free(z);
    return ok ? ORC_OK : ORC_ESINGULAR;
}

static void ctx_free_dir(orc_ctx *c, int l)
{
    free(c->xi[l]); free(c->pts[l]); free(c->qlo[l]); free(c->qlen[l]);
    free(c->jlo[l]); free(c->jlen[l]); free(c->Bv[l]); free(c->Bd[l]);
    free(c->Lv[l]); free(c->Ld[l]); free(c->alo[l]); free(c->ahi[l]);
    free(c->I4[l]); free(c->w[l]);
}

void orc_destroy(orc_ctx *c)
{
    if (!c) return;
    for (int l = 0; l < c->d; ++l) ctx_free_dir(c, l);
    free(c->ctrl);
    free(c->kappa);
    free(c->gamma);
    free(c);
}

int orc_status(orc_ctx *c) { return c ? c->status : ORC_EINVAL; }
const char *orc_message(orc_ctx *c) { return c ? c->msg : "null context"; }

/* Build one direction: grid, ranges, basis tables, exact integrals, weights. */
static int build_dir(orc_ctx *c, int l, const double *knots)
{
    int p = c->p;
    int64_t nk = c->nk[l];
    int64_t n = nk - p - 1, E = nk - 2 * (int64_t)p - 1;
    c->n[l] = n; c->E[l] = E;
    c->xi[l] = (double *)malloc(sizeof(double) * (size_t)nk);
    memcpy(c->xi[l], knots, sizeof(double) * (size_t)nk);
    const double *xi = c->xi[l];
    int64_t nq = orc_num_points(p, nk);
    c->nq[l] = nq;
    c->pts[l] = (double *)malloc(sizeof(double) * (size_t)nq);
    orc_points(p, nk, xi, c->pts[l]);
    const double *x = c->pts[l];

    /* Q_i: grid points in the OPEN support (xi_i, xi_{i+p+1});
     * I_i: j with B_i B_j not identically zero, i.e. open supports overlap. */
    c->qlo[l] = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    c->qlen[l] = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    c->jlo[l] = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    c->jlen[l] = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t maxq = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t lo = -1, cnt = 0;
        for (int64_t q = 0; q < nq; ++q)
            if (xi[i] < x[q] && x[q] < xi[i + p + 1]) { if (lo < 0) lo = q; ++cnt; }
        c->qlo[l][i] = lo; c->qlen[l][i] = cnt;
        if (cnt > maxq) maxq = cnt;
        int64_t jl = -1, jc = 0;
        for (int64_t j = 0; j < n; ++j) {
            double a = xi[i] > xi[j] ? xi[i] : xi[j];
            double b = xi[i + p + 1] < xi[j + p + 1] ? xi[i + p + 1] : xi[j + p + 1];
            if (a < b) { if (jl < 0) jl = j; ++jc; }
        }
        c->jlo[l][i] = jl; c->jlen[l][i] = jc;
        if (cnt < jc) { /* Eq. numb_nodes P:640-642 violated */
            snprintf(c->msg, sizeof c->msg, "dir %d row %lld: #Q=%lld < #I=%lld", l, (long long)i,
                     (long long)cnt, (long long)jc);
            return ORC_ESINGULAR;
        }
    }
    c->maxq[l] = maxq;

    /* basis tables at the grid points (Alg. 1 lines 3-4) */
    c->Bv[l] = (double *)calloc((size_t)nq * n, sizeof(double));
    c->Bd[l] = (double *)calloc((size_t)nq * n, sizeof(double));
    c->Lv[l] = (ld *)calloc((size_t)nq * n, sizeof(ld));
    c->Ld[l] = (ld *)calloc((size_t)nq * n, sizeof(ld));
    c->alo[l] = (int64_t *)malloc(sizeof(int64_t) * (size_t)nq);
    c->ahi[l] = (int64_t *)malloc(sizeof(int64_t) * (size_t)nq);
    qr *Nq = (qr *)malloc(sizeof(qr) * (size_t)n * nq);
    qr *dNq = (qr *)malloc(sizeof(qr) * (size_t)n * nq);
    for (int64_t q = 0; q < nq; ++q) {
        bspl_all(p, nk, xi, (qr)x[q], Nq + q * n, dNq + q * n);
        int64_t lo = n, hi = -1;
        for (int64_t j = 0; j < n; ++j) {
            qr v = Nq[q * n + j], dv = dNq[q * n + j];
            c->Bv[l][q * n + j] = (double)v;
            c->Bd[l][q * n + j] = (double)dv;
            c->Lv[l][q * n + j] = (ld)v;
            c->Ld[l][q * n + j] = (ld)dv;
            if (v != 0 || dv != 0) { if (j < lo) lo = j; hi = j; }
        }
        c->alo[l][q] = lo; c->ahi[l][q] = hi;
    }

    /* exact integrals, Eq. integrals, by (p+1)-point Gauss per span */
    int ng = p + 1;
    qr gt[64], gw[64];
    gauss_legendre(ng, gt, gw);
    qr *GN = (qr *)malloc(sizeof(qr) * (size_t)E * ng * n);
    qr *GD = (qr *)malloc(sizeof(qr) * (size_t)E * ng * n);
    qr *GW = (qr *)malloc(sizeof(qr) * (size_t)E * ng);
    for (int64_t e = 0; e < E; ++e) {
        qr a = xi[p + e], b = xi[p + e + 1];
        for (int g = 0; g < ng; ++g) {
            qr xg = (a + b) / 2 + (b - a) / 2 * gt[g];
            GW[e * ng + g] = (b - a) / 2 * gw[g];
            bspl_all(p, nk, xi, xg, GN + (e * ng + g) * n, GD + (e * ng + g) * n);
        }
    }
    int K = 2 * p + 1;
    c->I4[l] = (qr *)calloc((size_t)n * K * 4, sizeof(qr));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < c->jlen[l][i]; ++t) {
            int64_t j = c->jlo[l][i] + t;
            for (int f = 0; f < 4; ++f) {
                qr s = 0;
                for (int64_t e = 0; e < E; ++e)
                    for (int g = 0; g < ng; ++g) {
                        const qr *Ng = GN + (e * ng + g) * n, *Dg = GD + (e * ng + g) * n;
                        qr ti = FAM_A(f) ? Dg[i] : Ng[i];
                        qr tj = FAM_B(f) ? Dg[j] : Ng[j];
                        s += GW[e * ng + g] * ti * tj;
                    }
                c->I4[l][(i * K + t) * 4 + f] = s;
            }
        }
    free(GN); free(GD); free(GW);

    /* weights, Alg. 2: per row i and family (a,b), the min-norm
     * solution of  sum_q w_q D^b B_j(x_q) = I^(a,b)_{ij}  for j in I_i, q in Q_i.
     * b = 1: the system has rank #I-1 (sum_j B'_j = 0 on supp B_i); the middle
     * equation j* = I_i[#I/2] is dropped (reading R4).  Rows are equilibrated
     * by their max-abs entry.  Residual is checked on ALL #I equations.      */
    c->w[l] = (double *)calloc((size_t)n * 4 * (maxq > 0 ? maxq : 1), sizeof(double));
    int st = ORC_OK;
    for (int64_t i = 0; i < n && st == ORC_OK; ++i) {
        int ni = (int)c->jlen[l][i], nqi = (int)c->qlen[l][i];
        int64_t q0 = c->qlo[l][i], j0 = c->jlo[l][i];
        for (int b = 0; b <= 1 && st == ORC_OK; ++b) {
            int drop = b ? ni / 2 : -1;
            int m = b ? ni - 1 : ni;
            qr *M = (qr *)malloc(sizeof(qr) * (size_t)(m > 0 ? m : 1) * nqi);
            qr *sc = (qr *)malloc(sizeof(qr) * (size_t)(m > 0 ? m : 1));
            int r = 0;
            for (int t = 0; t < ni; ++t) {
                if (t == drop) continue;
                qr mx = 0;
                for (int k = 0; k < nqi; ++k) {
                    qr v = b ? dNq[(q0 + k) * n + j0 + t] : Nq[(q0 + k) * n + j0 + t];
                    M[(size_t)r * nqi + k] = v;
                    if (qabs(v) > mx) mx = qabs(v);
                }
                if (mx == 0) mx = 1;
                sc[r] = mx;
                for (int k = 0; k < nqi; ++k) M[(size_t)r * nqi + k] /= mx;
                ++r;
            }
            for (int a = 0; a <= 1 && st == ORC_OK; ++a) {
                int f = a + 2 * b;
                qr rhs[128], wq[128];
                r = 0;
                for (int t = 0; t < ni; ++t) {
                    if (t == drop) continue;
                    rhs[r] = c->I4[l][(i * K + t) * 4 + f] / sc[r];
                    ++r;
                }
                qr *Mc = (qr *)malloc(sizeof(qr) * (size_t)(m > 0 ? m : 1) * nqi);
                memcpy(Mc, M, sizeof(qr) * (size_t)m * nqi);
                if (m > 0) st = minnorm_solve(m, nqi, Mc, rhs, wq);
                else for (int k = 0; k < nqi; ++k) wq[k] = 0;
                free(Mc);
                if (st) {
                    snprintf(c->msg, sizeof c->msg, "dir %d row %lld family (%d,%d): singular", l,
                             (long long)i, a, b);
                    break;
                }
                double *wo = c->w[l] + ((size_t)i * 4 + f) * maxq;
                for (int k = 0; k < nqi; ++k) wo[k] = (double)wq[k];
                /* exactness residual with the FP64 weights, all #I equations (Eq. exact) */
                for (int t = 0; t < ni; ++t) {
                    qr s = 0, sa = 0;
                    for (int k = 0; k < nqi; ++k) {
                        qr v = b ? dNq[(q0 + k) * n + j0 + t] : Nq[(q0 + k) * n + j0 + t];
                        qr term = (qr)wo[k] * v;
                        s += term; sa += qabs(term);
                    }
                    qr I = c->I4[l][(i * K + t) * 4 + f];
                    if (qabs(s - I) > 1e-13Q * (sa + qabs(I)) + 1e-300Q) {
                        snprintf(c->msg, sizeof c->msg,
                                 "dir %d row %lld family (%d,%d) eq %d: residual %.3e", l,
                                 (long long)i, a, b, t, (double)qabs(s - I));
                        st = ORC_ESINGULAR;
                        break;
                    }
                }
            }
            free(M); free(sc);
        }
    }
    free(Nq); free(dNq);
    return st;
}

/* Create a context.  knots: d host arrays; ctrl: [N_DOF][d] or NULL.        */
orc_ctx *orc_create(int d, int p, const int64_t *nk, const double *const *knots, const double *ctrl)
{
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->d = d; c->p = p;
    if (d < 1 || d > 3 || p < 1 || p > 30) {
        c->status = ORC_EINVAL;
        snprintf(c->msg, sizeof c->msg, "bad d/p");
        c->d = 0;
        return c;
    }
    for (int l = 0; l < d; ++l) {
        c->nk[l] = nk[l];
        int st = orc_check_knots(p, nk[l], knots[l]);
        if (st) {
            c->status = st;
            snprintf(c->msg, sizeof c->msg, "dir %d: invalid knot vector", l);
            c->d = l;
            return c;
        }
    }
    c->ndof = 1;
    for (int l = 0; l < d; ++l) c->ndof *= nk[l] - p - 1;
    int st = ORC_OK;
    int built = 0;
    for (int l = 0; l < d; ++l) {
        built = l + 1;
        st = build_dir(c, l, knots[l]);
        if (st) break;
    }
    c->d = built; /* free what was built */
    if (st) { c->status = st; return c; }
    c->d = d;
    if (ctrl) {
        c->ctrl = (double *)malloc(sizeof(double) * (size_t)c->ndof * d);
        memcpy(c->ctrl, ctrl, sizeof(double) * (size_t)c->ndof * d);
    }
    return c;
}

/* scalar PDE coefficient nets (reading R17): [N_DOF] each, or NULL (= 1)   */
int orc_set_coefficients(orc_ctx *c, const double *kappa, const double *gamma)
{
    if (!c) return ORC_EINVAL;
    free(c->kappa);
    free(c->gamma);
    c->kappa = c->gamma = NULL;
    if (kappa) {
        c->kappa = (double *)malloc(sizeof(double) * (size_t)c->ndof);
        memcpy(c->kappa, kappa, sizeof(double) * (size_t)c->ndof);
    }
    if (gamma) {
        c->gamma = (double *)malloc(sizeof(double) * (size_t)c->ndof);
        memcpy(c->gamma, gamma, sizeof(double) * (size_t)c->ndof);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* exports of the univariate objects */
int64_t orc_info(orc_ctx *c, int l, int what)
{
    switch (what) {
    case 0: return c->n[l];
    case 1: return c->nq[l];
    case 2: return c->maxq[l];
    case 3: return c->E[l];
    case 4: return c->ndof;
    }
    return -1;
}

int orc_export_dir(orc_ctx *c, int l, double *pts, int64_t *qlo, int64_t *qlen, int64_t *jlo,
                   int64_t *jlen, double *w /*[n][4][maxq]*/, double *Bv /*[nq][n]*/, double *Bd,
                   double *I4 /*[n][2p+1][4]*/)
{
    int64_t n = c->n[l], nq = c->nq[l];
    if (pts) memcpy(pts, c->pts[l], sizeof(double) * (size_t)nq);
    if (qlo) memcpy(qlo, c->qlo[l], sizeof(int64_t) * (size_t)n);
    if (qlen) memcpy(qlen, c->qlen[l], sizeof(int64_t) * (size_t)n);
    if (jlo) memcpy(jlo, c->jlo[l], sizeof(int64_t) * (size_t)n);
    if (jlen) memcpy(jlen, c->jlen[l], sizeof(int64_t) * (size_t)n);
    if (w) memcpy(w, c->w[l], sizeof(double) * (size_t)n * 4 * c->maxq[l]);
    if (Bv) memcpy(Bv, c->Bv[l], sizeof(double) * (size_t)nq * n);
    if (Bd) memcpy(Bd, c->Bd[l], sizeof(double) * (size_t)nq * n);
    if (I4) {
        int64_t tot = n * (2 * c->p + 1) * 4;
        for (int64_t k = 0; k < tot; ++k) I4[k] = (double)c->I4[l][k];
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Geometry coefficients at one tensor point, from per-direction long-double
 * basis rows (values V[l][k], derivatives D[l][k], active range lo..hi).
 * J_{a,l} = dF_a/dzeta_l (Eq. mass2/stiff); returns det J and
 * fills c = |det J| and C = |det J| J^{-1} J^{-T} = adj(J) adj(J)^T / |det J|
 * (Eq. coef_stiff, reading R7), C row-major d x d.  With scalar PDE
 * coefficients ("Non-constant coefficients could be included as well";
 * P:508-509 "the factor c incorporates the coefficient of the equation";
 * reading R17) kappa(zeta) = sum_k kappa_k B_k(zeta) and gamma likewise, by
 * the same direct sum over the active control points: c = gamma |det J|,
 * C = kappa |det J| J^{-1} J^{-T}.                                          */
static ld coef_point(const orc_ctx *c, const ld *const *V, const ld *const *D,
                     const int64_t *lo, const int64_t *hi, ld *cm, ld *C)
{
    int d = c->d;
    ld J[3][3] = {{0}};
    ld kap = 0, gam = 0;
    int64_t n0 = c->n[0], n1 = d > 1 ? c->n[1] : 1;
    int64_t lo1 = d > 1 ? lo[1] : 0, hi1 = d > 1 ? hi[1] : 0;
    int64_t lo2 = d > 2 ? lo[2] : 0, hi2 = d > 2 ? hi[2] : 0;
    for (int64_t k2 = lo2; k2 <= hi2; ++k2)
        for (int64_t k1 = lo1; k1 <= hi1; ++k1)
            for (int64_t k0 = lo[0]; k0 <= hi[0]; ++k0) {
                int64_t k = k0 + n0 * (k1 + n1 * k2);
                int64_t kk[3] = {k0, k1, k2};
                for (int m = 0; m < d; ++m) { /* derivative direction */
                    ld f = 1;
                    for (int l = 0; l < d; ++l) f *= (l == m) ? D[l][kk[l]] : V[l][kk[l]];
                    if (f == 0) continue;
                    for (int a = 0; a < d; ++a) J[a][m] += (ld)c->ctrl[k * d + a] * f;
                }
                ld bv = 1;
                for (int l = 0; l < d; ++l) bv *= V[l][kk[l]];
                if (c->kappa) kap += (ld)c->kappa[k] * bv;
                if (c->gamma) gam += (ld)c->gamma[k] * bv;
            }
    ld det, adj[3][3];
    if (d == 1) {
        det = J[0][0];
        adj[0][0] = 1;
    } else if (d == 2) {
        det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        adj[0][0] = J[1][1]; adj[0][1] = -J[0][1];
        adj[1][0] = -J[1][0]; adj[1][1] = J[0][0];
    } else {
        adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
        adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
        adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
        adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
        adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
        adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        det = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
    }
    ld ad = det < 0 ? -det : det;
    if (!c->kappa) kap = 1;
    if (!c->gamma) gam = 1;
    *cm = gam * ad;
    for (int l = 0; l < d; ++l)
        for (int m = 0; m < d; ++m) {
            ld s = 0;
            for (int k = 0; k < d; ++k) s += adj[l][k] * adj[m][k];
            C[l * d + m] = ad > 0 ? kap * s / ad : 0;
        }
    return det;
}

/* coefficient at tensor grid point (q0,q1,q2) */
static ld coef_grid(const orc_ctx *c, const int64_t *q, ld *cm, ld *C)
{
    const ld *V[3], *D[3];
    int64_t lo[3], hi[3];
    for (int l = 0; l < c->d; ++l) {
        V[l] = c->Lv[l] + q[l] * c->n[l];
        D[l] = c->Ld[l] + q[l] * c->n[l];
        lo[l] = c->alo[l][q[l]];
        hi[l] = c->ahi[l][q[l]];
    }
    return coef_point(c, V, D, lo, hi, cm, C);
}

/* export of the coefficient field on a box of grid points, for pins:
 * out[(point)*(1+d*d) + 0] = c, then C row-major; points q0 fastest.
 * Returns ORC_EGEOMETRY if det J = 0 or changes sign in the box.           */
int orc_coef_box(orc_ctx *c, const int64_t *qb, const int64_t *qe, double *out, double *detout)
{
    int d = c->d;
    int64_t e0 = qe[0] - qb[0], e1 = d > 1 ? qe[1] - qb[1] : 1, e2 = d > 2 ? qe[2] - qb[2] : 1;
    int pos = 0, neg = 0, zero = 0;
    for (int64_t a2 = 0; a2 < e2; ++a2)
        for (int64_t a1 = 0; a1 < e1; ++a1)
            for (int64_t a0 = 0; a0 < e0; ++a0) {
                int64_t q[3] = {qb[0] + a0, d > 1 ? qb[1] + a1 : 0, d > 2 ? qb[2] + a2 : 0};
                ld cm, C[9];
                ld det = coef_grid(c, q, &cm, C);
                int64_t pt = a0 + e0 * (a1 + e1 * a2);
                if (out) {
                    out[pt * (1 + d * d)] = (double)cm;
                    for (int k = 0; k < d * d; ++k) out[pt * (1 + d * d) + 1 + k] = (double)C[k];
                }
                if (detout) detout[pt] = (double)det;
                if (det > 0) ++pos; else if (det < 0) ++neg; else ++zero;
            }
    return (zero || (pos && neg)) ? ORC_EGEOMETRY : ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Row values.  For row i (linear index, i_1 fastest) and every
 * j in I_i = prod_l I_{l,i_l}, in ascending linear order:
 *   mass:       m~_ij = sum_{q in Q_i} prod_k w^(0,0)_{k,i_k,q_k} B_{j_k}(x_{k,q_k}) c(x_q)
 *               (Eq. massquadrature)
 *   stiffness:  s~_ij = sum_{l,m} sum_{q in Q_i} prod_k w^(d_kl,d_km)_{k,i_k,q_k}
 *                                   D^{d_km} B_{j_k}(x_{k,q_k}) C_lm(x_q)
 *               (Eq. stiff P:518-524 with the families of Eq. quadrule/exact,
 *                reading R3: family (a,b) = (test-, trial-derivative order))
 * Direct nested sums in long double, FP64 weights and basis values, long
 * double coefficients.  Also returns per row
 *   kappa = max_j sum_q |term| / max_j |sum_q term|  and  scale = max_j sum_q |term|. */
static void decompose(const orc_ctx *c, int64_t r, int64_t *i)
{
    for (int l = 0; l < c->d; ++l) { i[l] = r % c->n[l]; r /= c->n[l]; }
}

int64_t orc_row_nnz(orc_ctx *c, int64_t r)
{
    int64_t i[3];
    decompose(c, r, i);
    int64_t z = 1;
    for (int l = 0; l < c->d; ++l) z *= c->jlen[l][i[l]];
    return z;
}

static int row_values(orc_ctx *c, int matrix, int64_t r, int32_t *col, double *val, double *kappa,
                      double *scale, ld *coefbuf)
{
    int d = c->d;
    int64_t i[3] = {0, 0, 0};
    decompose(c, r, i);
    int64_t nq[3] = {1, 1, 1}, q0[3] = {0, 0, 0}, ni[3] = {1, 1, 1}, j0[3] = {0, 0, 0};
    for (int l = 0; l < d; ++l) {
        nq[l] = c->qlen[l][i[l]]; q0[l] = c->qlo[l][i[l]];
        ni[l] = c->jlen[l][i[l]]; j0[l] = c->jlo[l][i[l]];
    }
    int ncomp = 1 + d * d;
    /* coefficients on the box Q_i */
    int geo_bad = 0;
    int sgn = 0;
    for (int64_t a2 = 0; a2 < nq[2]; ++a2)
        for (int64_t a1 = 0; a1 < nq[1]; ++a1)
            for (int64_t a0 = 0; a0 < nq[0]; ++a0) {
                int64_t q[3] = {q0[0] + a0, q0[1] + a1, q0[2] + a2};
                ld cm, C[9];
                ld det = coef_grid(c, q, &cm, C);
                int s = det > 0 ? 1 : (det < 0 ? -1 : 0);
                if (s == 0 || (sgn && s != sgn)) geo_bad = 1;
                sgn = s;
                ld *o = coefbuf + (a0 + nq[0] * (a1 + nq[1] * a2)) * ncomp;
                o[0] = cm;
                for (int k = 0; k < d * d; ++k) o[1 + k] = C[k];
            }
    ld maxabs = 0, maxsum = 0;
    int64_t t = 0;
    for (int64_t t2 = 0; t2 < ni[2]; ++t2)
        for (int64_t t1 = 0; t1 < ni[1]; ++t1)
            for (int64_t t0 = 0; t0 < ni[0]; ++t0, ++t) {
                int64_t j[3] = {j0[0] + t0, j0[1] + t1, j0[2] + t2};
                int64_t jlin = j[0] + c->n[0] * ((d > 1 ? j[1] : 0) + (d > 1 ? c->n[1] : 1) * (d > 2 ? j[2] : 0));
                ld s = 0, sa = 0;
                int nterm = matrix == 0 ? 1 : d * d;
                for (int tm = 0; tm < nterm; ++tm) {
                    int lt = tm / d, mt = tm % d; /* (l,m): test derivative dir l, trial derivative dir m */
                    for (int64_t a2 = 0; a2 < nq[2]; ++a2)
                        for (int64_t a1 = 0; a1 < nq[1]; ++a1)
                            for (int64_t a0 = 0; a0 < nq[0]; ++a0) {
                                int64_t aa[3] = {a0, a1, a2};
                                ld f = 1;
                                for (int k = 0; k < d; ++k) {
                                    int a = matrix == 0 ? 0 : (k == lt);
                                    int b = matrix == 0 ? 0 : (k == mt);
                                    int fam = a + 2 * b;
                                    double wk = c->w[k][((size_t)i[k] * 4 + fam) * c->maxq[k] + aa[k]];
                                    int64_t qk = q0[k] + aa[k];
                                    double bk = b ? c->Bd[k][qk * c->n[k] + j[k]] : c->Bv[k][qk * c->n[k] + j[k]];
                                    f *= (ld)wk * (ld)bk;
                                }
                                const ld *o = coefbuf + (a0 + nq[0] * (a1 + nq[1] * a2)) * ncomp;
                                ld term = f * (matrix == 0 ? o[0] : o[1 + lt * d + mt]);
                                s += term;
                                sa += term < 0 ? -term : term;
                            }
                }
                col[t] = (int32_t)jlin;
                val[t] = (double)s;
                ld as = s < 0 ? -s : s;
                if (as > maxabs) maxabs = as;
                if (sa > maxsum) maxsum = sa;
            }
    *scale = (double)maxsum;
    *kappa = maxabs > 0 ? (double)(maxsum / maxabs) : (maxsum > 0 ? INFINITY : 1.0);
    return geo_bad ? ORC_EGEOMETRY : ORC_OK;
}

/* rows[] are global linear row ids; ptr[k] = offset of row k's values
 * (caller sizes col/val with ptr[nrows] entries, see orc_row_nnz).          */
int orc_rows(orc_ctx *c, int matrix, int64_t nrows, const int64_t *rows, const int64_t *ptr,
             int32_t *col, double *val, double *kappa, double *scale)
{
    if (!c->ctrl) return ORC_EINVAL;
    int st = ORC_OK;
    int64_t maxbox = 1;
    for (int l = 0; l < c->d; ++l) maxbox *= c->maxq[l];
#pragma omp parallel
    {
        ld *buf = (ld *)malloc(sizeof(ld) * (size_t)maxbox * (1 + c->d * c->d));
#pragma omp for schedule(dynamic, 4)
        for (int64_t k = 0; k < nrows; ++k) {
            int s = row_values(c, matrix, rows[k], col + ptr[k], val + ptr[k], kappa + k, scale + k, buf);
            if (s) {
#pragma omp critical
                st = s;
            }
        }
        free(buf);
    }
    return st;
}

/* full CSR pattern by the definition (I_i = prod_l I_{l,i_l}). */
int orc_pattern(orc_ctx *c, int64_t *row_ptr, int32_t *col)
{
    int d = c->d;
    int64_t off = 0;
    for (int64_t r = 0; r < c->ndof; ++r) {
        int64_t i[3] = {0, 0, 0};
        decompose(c, r, i);
        row_ptr[r] = off;
        int64_t ni[3] = {1, 1, 1}, j0[3] = {0, 0, 0};
        for (int l = 0; l < d; ++l) { ni[l] = c->jlen[l][i[l]]; j0[l] = c->jlo[l][i[l]]; }
        for (int64_t t2 = 0; t2 < ni[2]; ++t2)
            for (int64_t t1 = 0; t1 < ni[1]; ++t1)
                for (int64_t t0 = 0; t0 < ni[0]; ++t0) {
                    int64_t jl = (j0[0] + t0) + c->n[0] * ((d > 1 ? j0[1] + t1 : 0) +
                                                           (d > 1 ? c->n[1] : 1) * (d > 2 ? j0[2] + t2 : 0));
                    if (col) col[off] = (int32_t)jl;
                    ++off;
                }
    }
    row_ptr[c->ndof] = off;
    return ORC_OK;
}

/* Pattern of the rows [r_lo, r_hi) by the same definition, for streaming
 * comparisons of full-size index arrays: row_ptr[0 .. r_hi-r_lo] are GLOBAL
 * offsets (the nnz of all earlier rows summed row by row), col the columns
 * of the range.                                                             */
int orc_pattern_rows(orc_ctx *c, int64_t r_lo, int64_t r_hi, int64_t *row_ptr, int32_t *col)
{
    int d = c->d;
    if (r_lo < 0 || r_hi > c->ndof || r_lo > r_hi) return ORC_EINVAL;
    int64_t off = 0;
    for (int64_t r = 0; r < r_lo; ++r) off += orc_row_nnz(c, r);
    for (int64_t r = r_lo; r < r_hi; ++r) {
        row_ptr[r - r_lo] = off;
        off += orc_row_nnz(c, r);
    }
    row_ptr[r_hi - r_lo] = off;
    if (!col) return ORC_OK;
    const int64_t base = row_ptr[0];
#pragma omp parallel for schedule(static)
    for (int64_t r = r_lo; r < r_hi; ++r) {
        int64_t i[3] = {0, 0, 0};
        decompose(c, r, i);
        int64_t ni[3] = {1, 1, 1}, j0[3] = {0, 0, 0};
        for (int l = 0; l < d; ++l) { ni[l] = c->jlen[l][i[l]]; j0[l] = c->jlo[l][i[l]]; }
        int64_t o = row_ptr[r - r_lo] - base;
        for (int64_t t2 = 0; t2 < ni[2]; ++t2)
            for (int64_t t1 = 0; t1 < ni[1]; ++t1)
                for (int64_t t0 = 0; t0 < ni[0]; ++t0)
                    col[o++] = (int32_t)((j0[0] + t0) + c->n[0] * ((d > 1 ? j0[1] + t1 : 0) +
                                                                  (d > 1 ? c->n[1] : 1) * (d > 2 ? j0[2] + t2 : 0)));
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Element-loop standard Gauss quadrature (SGQ), p+1 points per direction per
 * element, dense N_DOF x N_DOF output (small problems only).  The paper's
 * comparison method; used to self-check the WQ rows on affine
 * maps, where WQ is exact, and as the oracle of the GPU
 * SGQ baseline (wq_assemble_sgq).                                           */
int orc_sgq_dense(orc_ctx *c, int matrix, double *A)
{
    if (!c->ctrl) return ORC_EINVAL;
    int d = c->d, p = c->p, ng = p + 1;
    int64_t N = c->ndof;
    memset(A, 0, sizeof(double) * (size_t)(N * N));
    qr gt[64], gw[64];
    gauss_legendre(ng, gt, gw);
    ld *acc = (ld *)calloc((size_t)(N * N), sizeof(ld));
    /* per direction, per element, per Gauss point: all basis values (ld) */
    ld *GV[3], *GD[3], *GW[3];
    for (int l = 0; l < d; ++l) {
        int64_t E = c->E[l], n = c->n[l];
        GV[l] = (ld *)malloc(sizeof(ld) * (size_t)(E * ng * n));
        GD[l] = (ld *)malloc(sizeof(ld) * (size_t)(E * ng * n));
        GW[l] = (ld *)malloc(sizeof(ld) * (size_t)(E * ng));
        qr *tv = (qr *)malloc(sizeof(qr) * (size_t)n), *td = (qr *)malloc(sizeof(qr) * (size_t)n);
        for (int64_t e = 0; e < E; ++e) {
            qr a = c->xi[l][p + e], b = c->xi[l][p + e + 1];
            for (int g = 0; g < ng; ++g) {
                qr xg = (a + b) / 2 + (b - a) / 2 * gt[g];
                GW[l][e * ng + g] = (ld)((b - a) / 2 * gw[g]);
                bspl_all(p, c->nk[l], c->xi[l], xg, tv, td);
                for (int64_t k = 0; k < n; ++k) {
                    GV[l][(e * ng + g) * n + k] = (ld)tv[k];
                    GD[l][(e * ng + g) * n + k] = (ld)td[k];
                }
            }
        }
        free(tv); free(td);
    }
    int64_t E0 = c->E[0], E1 = d > 1 ? c->E[1] : 1, E2 = d > 2 ? c->E[2] : 1;
    int G1 = d > 1 ? ng : 1, G2 = d > 2 ? ng : 1;
    for (int64_t e2 = 0; e2 < E2; ++e2)
        for (int64_t e1 = 0; e1 < E1; ++e1)
            for (int64_t e0 = 0; e0 < E0; ++e0)
                for (int g2 = 0; g2 < G2; ++g2)
                    for (int g1 = 0; g1 < G1; ++g1)
                        for (int g0 = 0; g0 < ng; ++g0) {
                            int64_t e[3] = {e0, e1, e2};
                            int g[3] = {g0, g1, g2};
                            const ld *V[3], *D[3];
                            int64_t lo[3], hi[3];
                            ld wt = 1;
                            for (int l = 0; l < d; ++l) {
                                int64_t n = c->n[l];
                                int64_t row = e[l] * ng + g[l];
                                V[l] = GV[l] + row * n;
                                D[l] = GD[l] + row * n;
                                lo[l] = e[l]; hi[l] = e[l] + p; /* functions nonzero on span e */
                                wt *= GW[l][row];
                            }
                            ld cm, C[9];
                            coef_point(c, V, D, lo, hi, &cm, C);
                            /* all pairs of local functions */
                            int64_t nloc = 1;
                            for (int l = 0; l < d; ++l) nloc *= (p + 1);
                            for (int64_t ai = 0; ai < nloc; ++ai)
                                for (int64_t aj = 0; aj < nloc; ++aj) {
                                    int64_t ii[3] = {0, 0, 0}, jj[3] = {0, 0, 0};
                                    int64_t x = ai, y = aj;
                                    for (int l = 0; l < d; ++l) {
                                        ii[l] = lo[l] + x % (p + 1); x /= (p + 1);
                                        jj[l] = lo[l] + y % (p + 1); y /= (p + 1);
                                    }
                                    ld v = 0;
                                    if (matrix == 0) {
                                        ld f = 1;
                                        for (int l = 0; l < d; ++l) f *= V[l][ii[l]] * V[l][jj[l]];
                                        v = f * cm;
                                    } else {
                                        for (int lt = 0; lt < d; ++lt)
                                            for (int mt = 0; mt < d; ++mt) {
                                                ld f = 1;
                                                for (int l = 0; l < d; ++l)
                                                    f *= (l == lt ? D[l][ii[l]] : V[l][ii[l]]) *
                                                         (l == mt ? D[l][jj[l]] : V[l][jj[l]]);
                                                v += f * C[lt * d + mt];
                                            }
                                    }
                                    int64_t I = ii[0], J = jj[0], s = c->n[0];
                                    for (int l = 1; l < d; ++l) { I += s * ii[l]; J += s * jj[l]; s *= c->n[l]; }
                                    acc[I * N + J] += wt * v;
                                }
                        }
    for (int64_t k = 0; k < N * N; ++k) A[k] = (double)acc[k];
    free(acc);
    for (int l = 0; l < d; ++l) { free(GV[l]); free(GD[l]); free(GW[l]); }
    return ORC_OK;
}
