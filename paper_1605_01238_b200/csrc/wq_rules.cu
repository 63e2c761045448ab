// wq_rules.cu -- steps 1-4 of the hot path:
//   k_grid     point grid + span index per point     Remark 1, reading R1
//   k_ranges   Q_i, I_i, prefix of #I_i             Eq. support
//   k_gauss    (p+1)-point Gauss-Legendre in dd       Alg. 1 line 8
//   k_basis    B^(0), B^(1) tables                    Alg. 1 lines 3-4
//   k_weights  exact integrals + 4 min-norm families  Eq. integrals, Alg. 2
// Basis values, integrals and solves are in double-double (reading R5),
// rounded once to FP64.
#include "wq_internal.cuh"
#include "dd.cuh"

namespace {

struct DirArgs {
    DirView v[3];
    int p;
    int d;
};

// ---------------------------------------------------------------- grid
// Grid index of breakpoint chi_e: 0, p+2e (1 <= e <= E-1), last = nq-1.
__device__ __forceinline__ int64_t knot_pos(int64_t e, int64_t E, int p, int64_t nq) {
    if (e <= 0) return 0;
    if (e >= E) return nq - 1;
    return p + 2 * e;
}

__global__ void k_grid(DirArgs a) {
    const int l = blockIdx.y;
    if (l >= a.d) return;
    DirView &v = a.v[l];
    const int p = a.p;
    const int64_t E = v.E, nq = v.nq;
    const double *xi = v.knots;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nq; g += (int64_t)gridDim.x * blockDim.x) {
        double x;
        int64_t span;
        // classify g (integer logic only)
        int64_t e = -1, k = 0;  // boundary span e with inner point k, or knot/midpoint
        int kind;               // 0 knot, 1 boundary-span point, 2 midpoint
        int64_t knot = 0;
        if (g == 0) { kind = 0; knot = 0; }
        else if (g == nq - 1) { kind = 0; knot = E; }
        else if (g <= p + 1) { kind = 1; e = 0; k = g; }
        else if (E >= 2 && g >= p + 2 * (E - 1) + 1) { kind = 1; e = E - 1; k = g - (p + 2 * (E - 1)); }
        else {
            int64_t t = g - p;
            if ((t & 1) == 0) { kind = 0; knot = t / 2; }
            else { kind = 2; e = (t - 1) / 2; }
        }
        if (kind == 0) {
            x = xi[p + knot];
            span = knot < E ? knot : E - 1;  // right limit; left limit at the last knot
        } else if (kind == 1) {
            // a + ((b - a) * k) / (p + 2), no contraction (reading R1)
            double aa = xi[p + e], bb = xi[p + e + 1];
            x = __dadd_rn(aa, __ddiv_rn(__dmul_rn(__dsub_rn(bb, aa), (double)k), (double)(p + 2)));
            span = e;
        } else {
            double aa = xi[p + e], bb = xi[p + e + 1];
            x = __dmul_rn(0.5, __dadd_rn(aa, bb));
            span = e;
        }
        v.pts[g] = x;
        v.span[g] = (int32_t)span;
    }
}

// closed-form prefix P(i) = sum_{i' < i} #I_{i'}   (#I = min(n-1,i+p) - max(0,i-p) + 1)
__host__ __device__ __forceinline__ int64_t prefix_ni(int64_t i, int p, int64_t n) {
    if (i <= 0) return 0;
    int64_t c = n - 1 - p;
    int64_t m = (i - 1 < c) ? i - 1 : c;
    int64_t A = (m >= 0) ? ((m + 1) * p + m * (m + 1) / 2 + (i - 1 - m) * (n - 1)) : i * (n - 1);
    int64_t t = i - 1 - p;
    int64_t Bm = t >= 0 ? t * (t + 1) / 2 : 0;
    return A - Bm + i;
}

__global__ void k_ranges(DirArgs a) {
    const int l = blockIdx.y;
    if (l >= a.d) return;
    DirView &v = a.v[l];
    const int p = a.p;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= v.n; i += (int64_t)gridDim.x * blockDim.x) {
        v.pref[i] = prefix_ni(i, p, v.n);
        if (i == v.n) continue;
        // open support (xi_i, xi_{i+p+1}) = (chi_{max(0,i-p)}, chi_{min(E,i+1)})
        int64_t lo = knot_pos(i - p, v.E, p, v.nq) + 1;
        int64_t hi = knot_pos(i + 1 < v.E ? i + 1 : v.E, v.E, p, v.nq) - 1;
        v.qlo[i] = (int32_t)lo;
        v.qlen[i] = (int32_t)(hi - lo + 1);
        v.jlo[i] = (int32_t)wq_jlo(i, p);
        v.jlen[i] = (int32_t)wq_ni(i, p, v.n);
    }
}

// ---------------------------------------------------------------- B-splines in dd
// Values and first derivatives of the p+1 functions e..e+p nonzero on span e
// (knot-array index s = p + e), at x (dd).  Standard triangular recursion.
// Optionally the p degree-(p-1) values of functions e+1..e+p (Nlow).
__device__ void bspl_dd(const double *__restrict__ xi, int p, int e, dd x, dd *N, dd *dN, dd *Nlow = nullptr) {
    const int s = p + e;
    dd left[WQ_PMAX + 1], right[WQ_PMAX + 1], Nm[WQ_PMAX + 1];
    N[0] = dd_make(1.0);
    Nm[0] = dd_make(1.0);
    for (int j = 1; j <= p; ++j) {
        left[j] = dd_add_d(x, -xi[s + 1 - j]);
        right[j] = dd_add_d(dd_neg(x), xi[s + j]);
        dd saved = dd_make(0.0);
        for (int r = 0; r < j; ++r) {
            dd temp = dd_div(N[r], dd_add(right[r + 1], left[j - r]));
            N[r] = dd_add(saved, dd_mul(right[r + 1], temp));
            saved = dd_mul(left[j - r], temp);
        }
        N[j] = saved;
        if (j == p - 1)
            for (int r = 0; r <= j; ++r) Nm[r] = N[r];
    }
    for (int r = 0; r <= p; ++r) {
        dd t = dd_make(0.0);
        // knot differences exactly in dd (two_sum): FP64 subtraction would round
        if (r > 0) t = dd_div(Nm[r - 1], two_sum(xi[s + r], -xi[s + r - p]));
        if (r < p) t = dd_sub(t, dd_div(Nm[r], two_sum(xi[s + r + 1], -xi[s + r + 1 - p])));
        dN[r] = dd_mul_d(t, (double)p);
    }
    if (Nlow)
        for (int r = 0; r < p; ++r) Nlow[r] = Nm[r];
}

__global__ void k_basis(DirArgs a) {
    const int l = blockIdx.y;
    if (l >= a.d) return;
    DirView &v = a.v[l];
    const int p = a.p;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < v.nq; g += (int64_t)gridDim.x * blockDim.x) {
        dd N[WQ_PMAX + 1], dN[WQ_PMAX + 1], Nl[WQ_PMAX + 1];
        bspl_dd(v.knots, p, v.span[g], dd_make(v.pts[g]), N, dN, Nl);
        double *o = v.B + g * wq_bstride(p);  // [(value, derivative) pairs][degree p-1 values]
        for (int r = 0; r <= p; ++r) {
            o[2 * r] = dd_to_d(N[r]);
            o[2 * r + 1] = dd_to_d(dN[r]);
            o[2 * (p + 1) + r] = r < p ? dd_to_d(Nl[r]) : 0.0;
        }
    }
}

// ---------------------------------------------------------------- Gauss-Legendre in dd
__device__ void legendre_dd(int n, dd x, dd &Pn, dd &dPn) {
    dd P0 = dd_make(1.0), P1 = x;
    for (int m = 2; m <= n; ++m) {
        // P2 = ((2m-1) x P1 - (m-1) P0) / m
        dd P2 = dd_div(dd_sub(dd_mul_d(dd_mul(x, P1), (double)(2 * m - 1)), dd_mul_d(P0, (double)(m - 1))),
                       dd_make((double)m));
        P0 = P1;
        P1 = P2;
    }
    if (n == 1) { P0 = dd_make(1.0); P1 = x; }
    Pn = P1;
    // P'_n = n (x P_n - P_{n-1}) / (x^2 - 1)
    dPn = dd_div(dd_mul_d(dd_sub(dd_mul(x, P1), P0), (double)n), dd_add_d(dd_mul(x, x), -1.0));
}

__global__ void k_gauss(int n, double *gl) {
    int k = threadIdx.x;
    if (k >= n) return;
    double x = cos(3.14159265358979323846 * (k + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {  // FP64 Newton
        double P0 = 1.0, P1 = x;
        for (int m = 2; m <= n; ++m) {
            double P2 = ((2 * m - 1) * x * P1 - (m - 1) * P0) / m;
            P0 = P1;
            P1 = P2;
        }
        double dP = n == 1 ? 1.0 : n * (x * P1 - P0) / (x * x - 1.0);
        double dx = P1 / dP;
        x -= dx;
        // FP64 accurate (absolute: the roots lie in (-1, 1), and the middle root of an odd rule is 0,
        // where a relative test never holds); the dd Newton steps below finish
        if (fabs(dx) <= 1e-15) break;
    }
    dd X = dd_make(x), Pn, dPn;
    for (int it = 0; it < 3; ++it) {  // dd Newton
        legendre_dd(n, X, Pn, dPn);
        X = dd_sub(X, dd_div(Pn, dPn));
    }
    legendre_dd(n, X, Pn, dPn);
    dd w = dd_div(dd_make(2.0), dd_mul(dd_add_d(dd_neg(dd_mul(X, X)), 1.0), dd_mul(dPn, dPn)));
    gl[2 * k] = X.hi;
    gl[2 * k + 1] = X.lo;
    gl[2 * n + 2 * k] = w.hi;
    gl[2 * n + 2 * k + 1] = w.lo;
}

// ---------------------------------------------------------------- weights
// One CTA (64 threads) per (row i, direction l).  Dynamic shared memory:
//   Gv, Gd   [(p+1) spans][(p+1) Gauss pts][p+1]  dd   basis at Gauss points
//   Gw       [(p+1)][(p+1)] dd                          Gauss weights * half span
//   I4       [KMAX][4] dd                               exact integrals
//   M        [2][KMAX][QMAX] dd                         D^b B_j(x_q), j in I_i, q in Q_i
//   A        [2][KMAX][QMAX] dd                         scaled M^T, then Householder factors
//   V        [2][KMAX][QMAX] dd                         Householder vectors
//   Z        [2][2][QMAX] dd                            solutions, per (b, a)
//   sc       [2][KMAX] dd                               row scales
struct WSmem {
    int p, KM, QM;
    size_t off_Gv, off_Gd, off_Gw, off_I4, off_M, off_A, off_V, off_Z, off_sc, bytes;
    // QM = max_i #Q_i over the directions (3p+1, or more when one support
    // holds both boundary spans, n_EL <= p+1)
    __host__ __device__ WSmem(int p_, int qm) : p(p_), KM(2 * p_ + 1), QM(qm) {
        size_t P1 = p + 1, o = 0, s = sizeof(dd);
        off_Gv = o; o += P1 * P1 * P1 * s;
        off_Gd = o; o += P1 * P1 * P1 * s;
        off_Gw = o; o += P1 * P1 * s;
        off_I4 = o; o += (size_t)KM * 4 * s;
        off_M = o;  o += 2 * (size_t)KM * QM * s;
        off_A = o;  o += 2 * (size_t)KM * QM * s;
        off_V = o;  o += 2 * (size_t)KM * QM * s;
        off_Z = o;  o += 4 * (size_t)QM * s;
        off_sc = o; o += 2 * (size_t)KM * s;
        bytes = o;
    }
};

__global__ void __launch_bounds__(64) k_weights(DirArgs a, const double *__restrict__ gl, Flags *flags, int qmax) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int l = blockIdx.y;
    if (l >= a.d) return;
    const DirView &v = a.v[l];
    const int64_t i = blockIdx.x;
    if (i >= v.n) return;
    const int p = a.p, P1 = p + 1;
    WSmem L(p, qmax);
    dd *Gv = (dd *)(smem + L.off_Gv), *Gd = (dd *)(smem + L.off_Gd), *Gw = (dd *)(smem + L.off_Gw);
    dd *I4 = (dd *)(smem + L.off_I4), *M = (dd *)(smem + L.off_M), *A = (dd *)(smem + L.off_A);
    dd *V = (dd *)(smem + L.off_V), *Z = (dd *)(smem + L.off_Z), *sc = (dd *)(smem + L.off_sc);
    const int KM = L.KM, QM = L.QM;
    const double *xi = v.knots;
    const int tid = threadIdx.x;

    const int64_t e0 = i - p > 0 ? i - p : 0;
    const int64_t e1 = i < v.E - 1 ? i : v.E - 1;
    const int ns = (int)(e1 - e0 + 1);
    const int64_t j0 = v.jlo[i];
    const int ni = v.jlen[i];
    const int64_t q0 = v.qlo[i];
    const int nqi = v.qlen[i];

    // Phase 1: basis at the Gauss points of the spans of supp B_i
    for (int t = tid; t < ns * P1; t += blockDim.x) {
        int es = t / P1, g = t % P1;
        int64_t e = e0 + es;
        double xa = xi[p + e], xb = xi[p + e + 1];
        dd half = dd_mul_d(dd_add_d(dd_make(xb), -xa), 0.5);
        dd mid = dd_mul_d(dd_add_d(dd_make(xa), xb), 0.5);
        dd tg{gl[2 * g], gl[2 * g + 1]}, wg{gl[2 * P1 + 2 * g], gl[2 * P1 + 2 * g + 1]};
        dd x = dd_add(mid, dd_mul(half, tg));
        Gw[es * P1 + g] = dd_mul(half, wg);
        bspl_dd(xi, p, (int)e, x, Gv + (es * P1 + g) * P1, Gd + (es * P1 + g) * P1);
    }
    // Phase 3 (independent): matrices D^b B_j(x_q)
    for (int t = tid; t < nqi; t += blockDim.x) {
        int64_t q = q0 + t;
        int sp = v.span[q];
        dd N[WQ_PMAX + 1], dN[WQ_PMAX + 1];
        bspl_dd(xi, p, sp, dd_make(v.pts[q]), N, dN);
        for (int r = 0; r < ni; ++r) {
            int64_t j = j0 + r;
            int loc = (int)(j - sp);
            bool in = loc >= 0 && loc <= p;
            M[(0 * KM + r) * QM + t] = in ? N[loc] : dd_make(0.0);
            M[(1 * KM + r) * QM + t] = in ? dN[loc] : dd_make(0.0);
        }
    }
    __syncthreads();
    // Phase 2: exact integrals I^(a,b)_{i,j}, j in I_i  (Eq. integrals)
    for (int t = tid; t < ni * 4; t += blockDim.x) {
        int r = t >> 2, f = t & 3, fa = f & 1, fb = f >> 1;
        int64_t j = j0 + r;
        dd s = dd_make(0.0);
        for (int es = 0; es < ns; ++es) {
            int64_t e = e0 + es;
            int li = (int)(i - e), lj = (int)(j - e);
            if (li < 0 || li > p || lj < 0 || lj > p) continue;
            for (int g = 0; g < P1; ++g) {
                const dd *bv = Gv + (es * P1 + g) * P1, *bd = Gd + (es * P1 + g) * P1;
                dd ti = fa ? bd[li] : bv[li];
                dd tj = fb ? bd[lj] : bv[lj];
                s = dd_add(s, dd_mul(Gw[es * P1 + g], dd_mul(ti, tj)));
            }
        }
        I4[r * 4 + f] = s;
    }
    __syncthreads();

    // Phase 4: min-norm solves, warp b handles trial-derivative order b.
    const int warp = tid >> 5, lane = tid & 31;
    const int b = warp;
    const int drop = b ? ni / 2 : -1;   // reading R4: drop the middle equation when b = 1
    const int m = b ? ni - 1 : ni;
    dd *Mb = M + (size_t)b * KM * QM;
    dd *Ab = A + (size_t)b * KM * QM;   // column c (kept equation) stored as Ab[c*QM + q]
    dd *Vb = V + (size_t)b * KM * QM;
    dd *Zb = Z + (size_t)b * 2 * QM;    // [a][q]
    dd *scb = sc + (size_t)b * KM;
    bool ok = nqi >= m;
    // equilibrate + transpose
    for (int c = lane; c < m; c += 32) {
        int r = c < drop || drop < 0 ? c : c + 1;
        double mx = 0.0;
        for (int q = 0; q < nqi; ++q) mx = fmax(mx, fabs(Mb[r * QM + q].hi));
        if (mx == 0.0) mx = 1.0;
        scb[c] = dd_make(mx);
        const dd rmx = dd_div(dd_make(1.0), dd_make(mx));  // one division per equation, then products
        for (int q = 0; q < nqi; ++q) Ab[c * QM + q] = dd_mul(Mb[r * QM + q], rmx);
    }
    __syncwarp();
    // Householder QR of A (nqi x m); lane 0 forms the reflector, lanes update columns
    __shared__ int zero_pivot[2];
    if (lane == 0) zero_pivot[b] = 0;
    __syncwarp();
    // warp sum of per-lane dd partials (lanes hold the terms q = k + lane, k + lane + 32, ..)
    auto warp_sum = [&](dd x) {
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            dd y{__shfl_xor_sync(0xffffffffu, x.hi, o), __shfl_xor_sync(0xffffffffu, x.lo, o)};
            x = dd_add(x, y);
        }
        return x;
    };
    for (int k = 0; k < m && ok; ++k) {
        dd *vk = Vb + k * QM;
        dd part = dd_make(0.0);
        for (int q = k + lane; q < nqi; q += 32) part = dd_add(part, dd_mul(Ab[k * QM + q], Ab[k * QM + q]));
        const dd nrm = dd_sqrt(warp_sum(part));
        if (nrm.hi == 0.0) {
            if (lane == 0) zero_pivot[b] = 1;
        } else {
            const dd x0 = Ab[k * QM + k];
            const dd alpha = x0.hi >= 0.0 ? dd_neg(nrm) : nrm;
            // v = (a_k - alpha e_k) / |a_k - alpha e_k|
            dd vpart = dd_make(0.0);
            for (int q = k + lane; q < nqi; q += 32) {
                const dd vq = q == k ? dd_sub(Ab[k * QM + q], alpha) : Ab[k * QM + q];
                vk[q] = vq;
                vpart = dd_add(vpart, dd_mul(vq, vq));
            }
            const dd rvn = dd_div(dd_make(1.0), dd_sqrt(warp_sum(vpart)));
            for (int q = k + lane; q < nqi; q += 32) vk[q] = dd_mul(vk[q], rvn);
            __syncwarp();
            if (lane == 0) {
                Ab[k * QM + k] = alpha;  // R(k,k)
                for (int q = k + 1; q < nqi; ++q) Ab[k * QM + q] = dd_make(0.0);
            }
        }
        __syncwarp();
        if (zero_pivot[b]) { ok = false; break; }
        for (int c = k + 1 + lane; c < m; c += 32) {
            dd s = dd_make(0.0);
            for (int q = k; q < nqi; ++q) s = dd_add(s, dd_mul(vk[q], Ab[c * QM + q]));
            s = dd_mul_d(s, 2.0);
            for (int q = k; q < nqi; ++q) Ab[c * QM + q] = dd_sub(Ab[c * QM + q], dd_mul(s, vk[q]));
        }
        __syncwarp();
    }
    // forward solve R^T z = rhs and w = H_0 .. H_{m-1} [z; 0], lane a handles family (a, b)
    if (ok && lane < 2) {
        const int aa = lane, f = aa + 2 * b;
        dd *z = Zb + aa * QM;
        for (int k = 0; k < m; ++k) {
            int r = k < drop || drop < 0 ? k : k + 1;
            dd s = dd_div(I4[r * 4 + f], scb[k]);
            for (int t = 0; t < k; ++t) s = dd_sub(s, dd_mul(Ab[k * QM + t], z[t]));  // R(t,k) = Ab[k][t]
            z[k] = dd_div(s, Ab[k * QM + k]);
        }
        for (int q = m; q < nqi; ++q) z[q] = dd_make(0.0);
        for (int k = m - 1; k >= 0; --k) {
            const dd *vk = Vb + k * QM;
            dd s = dd_make(0.0);
            for (int q = k; q < nqi; ++q) s = dd_add(s, dd_mul(vk[q], z[q]));
            s = dd_mul_d(s, 2.0);
            for (int q = k; q < nqi; ++q) z[q] = dd_sub(z[q], dd_mul(s, vk[q]));
        }
    }
    if (!ok && lane == 0) {
        atomicCAS(&flags->weights_bad, 0, (int)(1 + ((l * 4 + 2 * b) + 12 * (int)i)));
    }
    __syncthreads();
    // Phase 5: round, store, residual check on all #I equations (Eq. exact)
    double *W = v.W + (size_t)i * 4 * v.maxq;  // [c][family]
    for (int t = tid; t < 4 * v.maxq; t += blockDim.x) {
        int q = t >> 2, f = t & 3;
        int bb = f >> 1, aa = f & 1;
        W[t] = q < nqi ? dd_to_d(Z[(bb * 2 + aa) * QM + q]) : 0.0;
    }
    for (int t = tid; t < ni * 4; t += blockDim.x) {
        int r = t >> 2, f = t & 3, bb = f >> 1, aa = f & 1;
        dd s = dd_make(0.0);
        double sa = 0.0;
        for (int q = 0; q < nqi; ++q) {
            double wq = dd_to_d(Z[(bb * 2 + aa) * QM + q]);
            dd term = dd_mul_d(M[(bb * KM + r) * QM + q], wq);
            s = dd_add(s, term);
            sa += fabs(term.hi);
        }
        dd res = dd_sub(s, I4[r * 4 + f]);
        double tol = 1e-13 * (sa + fabs(I4[r * 4 + f].hi)) + 1e-300;
        if (!(fabs(res.hi) <= tol)) atomicCAS(&flags->weights_bad, 0, (int)(1 + (l * 4 + f) + 12 * (int)i));
    }
}

}  // namespace

wq_status launch_rules(wq_plan_s *P, cudaStream_t s) {
    // one set of rules per distinct knot vector (aliased directions share the tables)
    DirArgs a;
    int nd = 0;
    for (int l = 0; l < P->d; ++l)
        if (P->dir_src[l] == l) a.v[nd++] = P->dir[l];
    for (int l = nd; l < 3; ++l) a.v[l] = P->dir[l];
    a.p = P->p;
    a.d = nd;
    int64_t maxnq = 0, maxn = 0;
    for (int l = 0; l < P->d; ++l) {
        maxnq = P->dir[l].nq > maxnq ? P->dir[l].nq : maxnq;
        maxn = P->dir[l].n > maxn ? P->dir[l].n : maxn;
    }
    dim3 g1((unsigned)((maxnq + 127) / 128), nd);
    k_grid<<<g1, 128, 0, s>>>(a);
    dim3 g2((unsigned)((maxn + 1 + 127) / 128), nd);
    k_ranges<<<g2, 128, 0, s>>>(a);
    k_gauss<<<1, 32, 0, s>>>(P->p + 1, P->gl);
    k_basis<<<g1, 128, 0, s>>>(a);
    int qmax = 1;
    for (int l = 0; l < P->d; ++l) qmax = P->dir[l].maxq > qmax ? P->dir[l].maxq : qmax;
    WSmem L(P->p, qmax);
    wq_smem_attr((const void *)k_weights, L.bytes);
    dim3 g3((unsigned)maxn, nd);
    k_weights<<<g3, 64, L.bytes, s>>>(a, P->gl, P->flags, qmax);
    wq_count_launches(5);
    return wq_cuda_status(cudaGetLastError(), "rules kernels");
}

