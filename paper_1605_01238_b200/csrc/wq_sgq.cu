// wq_sgq.cu -- the standard method the paper compares WQ against (Sect. 5.2):
// element-loop Galerkin assembly with standard Gauss quadrature (SGQ), p+1 Gauss-Legendre points
// per direction and element, local (p+1)^d x (p+1)^d matrices scatter-added into the CSR layout of
// the plan (same pattern as WQ: the column set of row i is prod_l I_{l,i_l}).
//
//   m_ij = sum_e sum_g w_g  B_i(x_g) B_j(x_g) c(x_g),                     c = gamma |det J|
//   s_ij = sum_e sum_g w_g  sum_{l,m} d_l B_i(x_g) C_lm(x_g) d_m B_j(x_g), C = kappa |det J| J^-1 J^-T
//
// with J evaluated AT THE GAUSS POINTS by the direct sum over the element's (p+1)^d control points
// (no WQ grid involved).  Per element the local matrix is sum-factorised over the Gauss points,
// O((p+1)^{2d+1}) per term: outer loop over the (test, trial) pairs of direction d, then
// direction-1 and direction-2 contractions in shared memory.  One CTA per element; entries are
// atomically added (FP64 atomics), so the summation order over elements is not fixed.
#include "wq_rows.cuh"

namespace {

constexpr int SG_NT = 256;

// Gauss-point basis tables of one direction: for element e and Gauss node g, the values and
// derivatives of functions e..e+p at x = (a+b)/2 + (b-a)/2 t_g, and the scaled weight (b-a)/2 w_g.
// B-spline values by the triangular Cox-de Boor scheme on the element's local knots (FP64).
__global__ void k_sgq_tab(DirView v, int p, const double *gl, double2 *T, double *Wt) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int ng = p + 1;
    if (idx >= v.E * ng) return;
    const int64_t e = idx / ng;
    const int g = (int)(idx % ng);
    const double *xi = v.knots;
    const double a = xi[p + e], b = xi[p + e + 1];
    const double t = gl[2 * g];          // node (hi part of the double-double rule)
    const double w = gl[2 * ng + 2 * g];  // weight (hi part)
    const double x = 0.5 * (a + b) + 0.5 * (b - a) * t;
    Wt[idx] = 0.5 * (b - a) * w;
    // degree p-1 values N[0..p-1] of functions e+1..e+p... computed by the triangular scheme
    double N[WQ_PMAX + 1], left[WQ_PMAX + 1], right[WQ_PMAX + 1], Nm[WQ_PMAX + 1];
    const int64_t s = p + e;  // knot span index in the full knot vector
    N[0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = x - xi[s + 1 - j];
        right[j] = xi[s + j] - x;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            const double tmp = N[r] / (right[r + 1] + left[j - r]);
            N[r] = saved + right[r + 1] * tmp;
            saved = left[j - r] * tmp;
        }
        N[j] = saved;
        if (j == p - 1)
            for (int r = 0; r < p; ++r) Nm[r] = N[r];
    }
    if (p == 1) Nm[0] = 1.0;
    // derivative: B'_{k} = p (N^{p-1}_k / (xi_{k+p} - xi_k) - N^{p-1}_{k+1} / (xi_{k+p+1} - xi_{k+1}))
    double2 *o = T + idx * ng;
    for (int r = 0; r <= p; ++r) {
        const int64_t k = e + r;  // global function index
        double d = 0.0;
        if (r >= 1) d += p * Nm[r - 1] / (xi[k + p] - xi[k]);
        if (r <= p - 1) d -= p * Nm[r] / (xi[k + p + 1] - xi[k + 1]);
        o[r] = make_double2(N[r], d);
    }
}

struct SgqArgs {
    RowGeo g;
    DirView v[3];
    int d, p, matrix;
    const double *ctrl, *kappa, *gamma;
    const double2 *T[3];  // [E_l][ng][p+1] (value, derivative)
    const double *Wt[3];  // [E_l][ng]
    int64_t E[3];
    int64_t e3b, n_el;    // elements of this launch: slowest element index e_d in [e3b, e3b + ...)
    double *val;
    int64_t row_lo, row_hi;  // owned rows (global linear ids)
    Flags *flags;
};

__device__ __forceinline__ int cidx(int D, int l, int m) { return l * D + m; }

__global__ void __launch_bounds__(SG_NT) k_sgq(SgqArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int D = a.d, p = a.p, P1 = p + 1, tid = threadIdx.x;
    int n1[3], ng[3];
    for (int l = 0; l < 3; ++l) { n1[l] = l < D ? P1 : 1; ng[l] = l < D ? P1 : 1; }
    // element multi-index (e_d over [e3b, ...), slowest)
    int64_t el = blockIdx.x, e[3] = {0, 0, 0};
    for (int l = 0; l < D; ++l) {
        const int64_t El = l == D - 1 ? a.n_el : a.E[l];
        e[l] = el % El;
        el /= El;
    }
    e[D - 1] += a.e3b;
    const int npts = ng[0] * ng[1] * ng[2];
    const int nloc = n1[0] * n1[1] * n1[2];
    const int ncomp = a.matrix == 0 ? 1 : D * D;
    // smem: coefficient at the Gauss points [ncomp][npts], tables [3][P1 funcs][P1 gauss] x (val, der),
    // weights, T2 [ng0 * ng1], U [P1 * P1 * ng1]
    double *Cg = sm;
    double *Tb = Cg + ncomp * npts;             // [l][fun][g][2]
    double *T2 = Tb + 3 * P1 * P1 * 2;
    double *U = T2 + P1 * P1;
    for (int x = tid; x < 3 * P1 * P1; x += blockDim.x) {
        const int l = x / (P1 * P1), r = (x / P1) % P1, gq = x % P1;
        double2 t = make_double2(l >= D ? (r == 0 && gq == 0 ? 1.0 : 0.0) : 0.0, 0.0);
        if (l < D && r < P1 && gq < P1) t = a.T[l][(e[l] * P1 + gq) * P1 + r];
        Tb[((l * P1 + r) * P1 + gq) * 2 + 0] = t.x;
        Tb[((l * P1 + r) * P1 + gq) * 2 + 1] = t.y;
    }
    __syncthreads();
    // geometry at the Gauss points: J by the direct sum over the element's control points
    for (int gp = tid; gp < npts; gp += blockDim.x) {
        const int g0 = gp % ng[0], g1 = (gp / ng[0]) % ng[1], g2 = gp / (ng[0] * ng[1]);
        const int gg[3] = {g0, g1, g2};
        double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, kap = 0.0, gam = 0.0;
        for (int c = 0; c < nloc; ++c) {
            const int r0 = c % n1[0], r1 = (c / n1[0]) % n1[1], r2 = c / (n1[0] * n1[1]);
            const int rr[3] = {r0, r1, r2};
            int64_t k = 0, s = 1;
            double bv[3], bd[3];
            for (int l = 0; l < 3; ++l) {
                bv[l] = Tb[((l * P1 + rr[l]) * P1 + gg[l]) * 2];
                bd[l] = Tb[((l * P1 + rr[l]) * P1 + gg[l]) * 2 + 1];
                if (l < D) { k += (e[l] + rr[l]) * s; s *= a.v[l].n; }
            }
            const double val = bv[0] * bv[1] * bv[2];
            for (int m = 0; m < D; ++m) {
                double f = 1.0;
                for (int l = 0; l < D; ++l) f *= l == m ? bd[l] : bv[l];
                for (int c2 = 0; c2 < D; ++c2) J[c2][m] = fma(__ldg(a.ctrl + k * D + c2), f, J[c2][m]);
            }
            if (a.kappa) kap = fma(__ldg(a.kappa + k), val, kap);
            if (a.gamma) gam = fma(__ldg(a.gamma + k), val, gam);
        }
        if (!a.kappa) kap = 1.0;
        if (!a.gamma) gam = 1.0;
        double det, adj[3][3];
        if (D == 1) { det = J[0][0]; adj[0][0] = 1.0; }
        else if (D == 2) {
            det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
            adj[0][0] = J[1][1]; adj[0][1] = -J[0][1]; adj[1][0] = -J[1][0]; adj[1][1] = J[0][0];
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
        if (!(det > 0.0) && !(det < 0.0)) atomicOr(&a.flags->det_zero, 1);
        const double ad = fabs(det);
        double w = 1.0;
        for (int l = 0; l < D; ++l) w *= a.Wt[l][e[l] * P1 + gg[l]];
        if (a.matrix == 0) {
            Cg[gp] = w * gam * ad;
        } else {
            for (int l = 0; l < D; ++l)
                for (int m = 0; m < D; ++m) {
                    double sv = 0.0;
                    for (int k = 0; k < D; ++k) sv = fma(adj[l][k], adj[m][k], sv);
                    Cg[cidx(D, l, m) * npts + gp] = w * kap * sv / ad;
                }
        }
    }
    __syncthreads();
    const int nterm = a.matrix == 0 ? 1 : D * D;
    // local matrix by sum factorisation; direction D-1 (slowest) in the outer loop
    const int Ls = D - 1;  // slowest real direction
    const int n1o = n1[Ls];
    const int nin = D >= 2 ? n1[0] * n1[0] * (D == 3 ? n1[1] * n1[1] : 1) : 1;  // (a0 b0 [a1 b1]) pairs
    for (int ab = 0; ab < n1o * n1o; ++ab) {
        const int ao = ab % n1o, bo = ab / n1o;
        // accumulate the contribution of every term for the entries with (ao, bo) in the slowest direction
        // thread-private partial sums over the inner pairs: handled via smem accumulator U2
        for (int term = 0; term < nterm; ++term) {
            const int lt = term / D, mt = term % D;
            auto fam = [&](int l, int &ta, int &tb) {
                ta = a.matrix == 0 ? 0 : (l == lt);
                tb = a.matrix == 0 ? 0 : (l == mt);
            };
            int tao, tbo;
            fam(Ls, tao, tbo);
            const double *Cc = Cg + (a.matrix == 0 ? 0 : cidx(D, lt, mt)) * npts;
            // T2[g0][g1] = sum_{gs} F_s(ao, bo, gs) C(g0, g1, gs)   (D = 3; for D = 2 T2[g0] over g1 slowest)
            const int ninner = D == 3 ? ng[0] * ng[1] : (D == 2 ? ng[0] : 1);
            __syncthreads();
            for (int x = tid; x < ninner; x += blockDim.x) {
                double s = 0.0;
                for (int gs = 0; gs < ng[Ls]; ++gs) {
                    const double fa = Tb[((Ls * P1 + ao) * P1 + gs) * 2 + tao];
                    const double fb = Tb[((Ls * P1 + bo) * P1 + gs) * 2 + tbo];
                    s = fma(fa * fb, Cc[x + ninner * gs], s);
                }
                T2[x] = s;
            }
            __syncthreads();
            if (D == 3) {
                // U[a0 b0][g1] = sum_{g0} F_0(a0, b0, g0) T2[g0][g1]
                int ta0, tb0;
                fam(0, ta0, tb0);
                for (int x = tid; x < P1 * P1 * ng[1]; x += blockDim.x) {
                    const int a0 = x % P1, b0 = (x / P1) % P1, g1 = x / (P1 * P1);
                    double s = 0.0;
                    for (int g0 = 0; g0 < ng[0]; ++g0)
                        s = fma(Tb[((0 * P1 + a0) * P1 + g0) * 2 + ta0] * Tb[((0 * P1 + b0) * P1 + g0) * 2 + tb0],
                                T2[g0 + ng[0] * g1], s);
                    U[x] = s;
                }
                __syncthreads();
            }
            // final: entries (a0, b0, a1, b1) for this (ao, bo): atomic add into the CSR values
            int ta1 = 0, tb1 = 0, ta0 = 0, tb0 = 0;
            fam(D == 3 ? 1 : 0, ta1, tb1);
            fam(0, ta0, tb0);
            for (int x = tid; x < nin; x += blockDim.x) {
                int loc_a[3] = {0, 0, 0}, loc_b[3] = {0, 0, 0};
                double s;
                if (D == 3) {
                    const int a0 = x % P1, b0 = (x / P1) % P1, a1 = (x / (P1 * P1)) % P1, b1 = x / (P1 * P1 * P1);
                    s = 0.0;
                    for (int g1 = 0; g1 < ng[1]; ++g1)
                        s = fma(Tb[((1 * P1 + a1) * P1 + g1) * 2 + ta1] * Tb[((1 * P1 + b1) * P1 + g1) * 2 + tb1],
                                U[(a0 + P1 * b0) + P1 * P1 * g1], s);
                    loc_a[0] = a0; loc_b[0] = b0; loc_a[1] = a1; loc_b[1] = b1; loc_a[2] = ao; loc_b[2] = bo;
                } else if (D == 2) {
                    const int a0 = x % P1, b0 = x / P1;
                    s = 0.0;
                    for (int g0 = 0; g0 < ng[0]; ++g0)
                        s = fma(Tb[((0 * P1 + a0) * P1 + g0) * 2 + ta0] * Tb[((0 * P1 + b0) * P1 + g0) * 2 + tb0],
                                T2[g0], s);
                    loc_a[0] = a0; loc_b[0] = b0; loc_a[1] = ao; loc_b[1] = bo;
                } else {
                    s = T2[0];
                    loc_a[0] = ao; loc_b[0] = bo;
                }
                // global row / column multi-indices
                int64_t ii[3] = {0, 0, 0}, jj[3] = {0, 0, 0};
                for (int l = 0; l < D; ++l) { ii[l] = e[l] + loc_a[l]; jj[l] = e[l] + loc_b[l]; }
                int64_t r = ii[0] + a.g.n[0] * (ii[1] + a.g.n[1] * ii[2]);
                if (r < a.row_lo || r >= a.row_hi) continue;
                int64_t t = 0, st = 1;
                for (int l = 0; l < D; ++l) {
                    t += (jj[l] - wq_jlo(ii[l], p)) * st;
                    st *= a.g.ni(l, ii[l]);
                }
                const int64_t off = a.g.offset(ii[0], ii[1], ii[2]) + t;
                atomicAdd(a.val + off, s);
            }
        }
    }
}

}  // namespace

wq_status launch_assemble_sgq(wq_plan_s *P, int matrix, const double *ctrl, const double *kappa, const double *gamma,
                              double *val, int32_t *col, cudaStream_t s) {
    if (matrix == WQ_MASS && !P->need_mass) { wq_set_error("plan was created without need_mass"); return WQ_EINVAL; }
    if (matrix == WQ_STIFFNESS && !P->need_stiff) {
        wq_set_error("plan was created without need_stiffness");
        return WQ_EINVAL;
    }
    const int d = P->d, p = P->p, ng = p + 1;
    cudaError_t ce = cudaMemsetAsync(val, 0, sizeof(double) * (size_t)P->nnz_local, s);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "SGQ value reset");
    if (col) {
        wq_status st = launch_pattern(P, 0, nullptr, col, 0, 0, s);
        if (st) return st;
    }
    // Gauss tables (stream-ordered allocation: no host synchronisation)
    size_t tb = 0;
    size_t off_T[3], off_W[3];
    for (int l = 0; l < d; ++l) {
        off_T[l] = tb;
        tb += sizeof(double2) * (size_t)P->dir[l].E * ng * ng;
        off_W[l] = tb;
        tb += sizeof(double) * (size_t)P->dir[l].E * ng;
        tb = (tb + 255) & ~(size_t)255;
    }
    void *ws = nullptr;
    ce = cudaMallocAsync(&ws, tb, s);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "SGQ tables");
    SgqArgs a;
    a.g.init(P);
    for (int l = 0; l < 3; ++l) {
        a.v[l] = P->dir[l];
        a.E[l] = P->dir[l].E;
        a.T[l] = nullptr;
        a.Wt[l] = nullptr;
    }
    for (int l = 0; l < d; ++l) {
        a.T[l] = (const double2 *)((char *)ws + off_T[l]);
        a.Wt[l] = (const double *)((char *)ws + off_W[l]);
        const int64_t cnt = P->dir[l].E * ng;
        k_sgq_tab<<<(unsigned)((cnt + 127) / 128), 128, 0, s>>>(P->dir[l], p, P->gl, (double2 *)a.T[l], (double *)a.Wt[l]);
        wq_count_launches(1);
    }
    a.d = d;
    a.p = p;
    a.matrix = matrix;
    a.ctrl = ctrl;
    a.kappa = kappa;
    a.gamma = gamma;
    a.val = val;
    a.flags = P->flags;
    a.row_lo = P->row_begin;
    a.row_hi = P->row_begin + P->n_rows_local;
    // elements touching the owned rows: e_d in [slab_b - p, slab_e - 1] within [0, E_d)
    const int ld = d - 1;
    const int64_t eb = std::max<int64_t>(0, P->slab_b - p), ee = std::min<int64_t>(P->dir[ld].E, P->slab_e);
    a.e3b = eb;
    a.n_el = ee - eb;
    int64_t nel = a.n_el;
    for (int l = 0; l < ld; ++l) nel *= P->dir[l].E;
    const int np = d == 3 ? ng * ng * ng : (d == 2 ? ng * ng : ng);
    const int ncomp = matrix == WQ_MASS ? 1 : d * d;
    const size_t smem = sizeof(double) * ((size_t)ncomp * np + 3 * ng * ng * 2 + ng * ng + (size_t)ng * ng * ng);
    wq_smem_attr((const void *)k_sgq, smem);
    if (nel > 0) {
        k_sgq<<<(unsigned)nel, SG_NT, smem, s>>>(a);
        wq_count_launches(1);
    }
    ce = cudaGetLastError();
    cudaFreeAsync(ws, s);
    return wq_cuda_status(ce, "SGQ assembly kernel");
}
