// wq_coef.cu -- step 5 of the hot path: geometry coefficient field on the
// tensor point grid (Alg. 1 lines 12/15; Eq. mass2 P:505-507,
// Eq. coef_stiff, reading R7):
//   c = |det J|,   C = |det J| J^{-1} J^{-T} = adj(J) adj(J)^T / |det J|.
// J is evaluated from the DERIVATIVE CONTROL NETS
//   dF/dzeta_m = sum_k Q^m_k N^{(p-1)}_{k_m} prod_{l != m} N^{(p)}_{k_l},
//   Q^m_k = p (P_k - P_{k - e_m}) / (xi_{k_m + p} - xi_{k_m}),
// i.e. with nonnegative degree-(p-1)/p bases and differences of the INPUT
// control points, so no cancellation occurs (sum_k P_k dB_k/dzeta would lose
// ~ (p/h) eps relative accuracy at fine meshes).
// Sum-factorised over a CTA tile (q_1 tile x q_2 tile x one q_3):
//   stage A contracts k_3, stage B contracts k_2, stage C contracts k_1 per
//   point -- O(p) FMAs per component per point instead of the O(p^d) of the
//   direct sum.
#include <cstdlib>
#include <type_traits>
#include "wq_internal.cuh"

namespace {

constexpr int TQ1 = 32;  // q_1 points per CTA
constexpr int TQ2 = 8;   // q_2 points per CTA (D >= 2); threads = TQ1 * TQ2, one per point in stage C
constexpr int NTC = TQ1 * TQ2;

struct CoefArgs {
    DirView v[3];
    int d, p;
    const double *ctrl;  // [N_DOF][d]
    double *coef;        // [ncomp][points]
    int64_t cq_b;        // first q_d of the sub-grid
    int64_t nq_loc_d;    // q_d extent of the sub-grid
    int64_t cld1, cstride, c0off;  // coefficient layout (wq_internal.cuh)
    int ncomp_s, ncomp;
    int need_s, need_m;
    Flags *flags;
    const double *dnet;  // z layout: derivative control nets [k][m][c] (k_dnet)
    // z layout of the stiffness components (wq_internal.cuh): [comp][q_1][q_2][q_3 - cq_b]
    int zlayout;
    double *coefz;
    int64_t zld, zcs;
};

// table rows at grid point q: N = degree p (functions span..span+p, stride 2:
// values interleaved with derivatives), M = degree p-1 (functions span+1..span+p)
__device__ __forceinline__ const double *Ntab(const DirView &v, int p, int64_t q) { return v.B + q * wq_bstride(p); }
__device__ __forceinline__ const double *Mtab(const DirView &v, int p, int64_t q) {
    return v.B + q * wq_bstride(p) + 2 * (p + 1);
}
// p / (xi_{k+p} - xi_k): scale of derivative control point k (k >= 1)
__device__ __forceinline__ double dscale(const DirView &v, int p, int64_t k) {
    return (double)p / (v.knots[k + p] - v.knots[k]);
}

template <int D>
__global__ void __launch_bounds__(NTC) k_coef(CoefArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int p = a.p;
    const DirView &v1 = a.v[0], &v2 = a.v[1], &v3 = a.v[2];
    // d = 3: blockIdx.x = q_3 plane (consecutive CTAs write neighbouring q_3 of the z layout)
    const int64_t q1a = (int64_t)(D == 3 ? blockIdx.y : blockIdx.x) * TQ1;
    const int64_t q2a = D >= 2 ? (int64_t)(D == 3 ? blockIdx.z : blockIdx.y) * TQ2 : 0;
    const int64_t q3l = D == 3 ? (int64_t)blockIdx.x : 0;  // local plane
    const int64_t q3 = D == 3 ? a.cq_b + q3l : 0;
    const int64_t q1off = D == 1 ? a.cq_b : 0;  // D == 1: direction 1 is the slab direction
    const int64_t nq1 = D == 1 ? a.nq_loc_d : v1.nq;
    const int64_t nq2 = D >= 2 ? (D == 2 ? a.nq_loc_d : v2.nq) : 1;
    const int64_t q2off = D == 2 ? a.cq_b : 0;  // D == 2: direction 2 is the slab direction
    const int64_t q1e = q1a + TQ1 < nq1 ? q1a + TQ1 : nq1;
    const int64_t q2e = q2a + TQ2 < nq2 ? q2a + TQ2 : nq2;
    const int nt1 = (int)(q1e - q1a), nt2 = (int)(q2e - q2a);
    const int64_t k1a = v1.span[q1off + q1a], k1e = v1.span[q1off + q1e - 1] + p + 1;
    const int K1 = (int)(k1e - k1a);
    int64_t k2a = 0, k2e = 1;
    if (D >= 2) { k2a = v2.span[q2off + q2a]; k2e = v2.span[q2off + q2e - 1] + p + 1; }
    const int K2 = (int)(k2e - k2a);
    const int64_t n1 = v1.n, n2 = D >= 2 ? v2.n : 1;
    const int K1M = TQ1 + p + 1, K2M = TQ2 + p + 1;  // bounds of K1, K2 (smem sized by the actual p)
    // smem: A[3 variants][3 comps][K2M][K1M] (D == 3), X[TQ2][3 variants][3 comps][K1M]
    double *Asm = sm;
    double *Xsm = sm + (D == 3 ? 9 * K2M * K1M : 0);
    const int tid = threadIdx.x;
    const double *P = a.ctrl;

    if (D == 3) {
        // stage A: contract k_3.  A1 = N3 . Q^1, A2 = N3 . Q^2, A3 = M3 . Q^3
        const double *n3 = Ntab(v3, p, q3), *m3 = Mtab(v3, p, q3);
        const int64_t e3 = v3.span[q3];
        for (int t = tid; t < K2 * K1; t += blockDim.x) {
            const int c2 = t / K1, c1 = t % K1;
            const int64_t k1 = k1a + c1, k2 = k2a + c2;
            double A1[3] = {0, 0, 0}, A2[3] = {0, 0, 0}, A3[3] = {0, 0, 0};
            const double s1 = k1 >= 1 ? dscale(v1, p, k1) : 0.0;
            const double s2 = k2 >= 1 ? dscale(v2, p, k2) : 0.0;
            double prev[3] = {0, 0, 0};
            for (int r = 0; r <= p; ++r) {
                const int64_t k3 = e3 + r;
                const int64_t k = k1 + n1 * (k2 + n2 * k3);
                const double nv = n3[2 * r];
                const double s3 = r >= 1 ? dscale(v3, p, k3) : 0.0;
                #pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double cur = __ldg(P + k * 3 + c);
                    const double d1 = k1 >= 1 ? (cur - __ldg(P + (k - 1) * 3 + c)) * s1 : 0.0;
                    const double d2 = k2 >= 1 ? (cur - __ldg(P + (k - n1) * 3 + c)) * s2 : 0.0;
                    A1[c] = fma(nv, d1, A1[c]);
                    A2[c] = fma(nv, d2, A2[c]);
                    if (r >= 1) A3[c] = fma(m3[r - 1], (cur - prev[c]) * s3, A3[c]);
                    prev[c] = cur;
                }
            }
            #pragma unroll
            for (int c = 0; c < 3; ++c) {
                Asm[((0 * 3 + c) * K2M + c2) * K1M + c1] = A1[c];
                Asm[((1 * 3 + c) * K2M + c2) * K1M + c1] = A2[c];
                Asm[((2 * 3 + c) * K2M + c2) * K1M + c1] = A3[c];
            }
        }
        __syncthreads();
        // stage B: contract k_2.  X1 = N2 . A1, X2 = M2 . A2, X3 = N2 . A3
        for (int t = tid; t < nt2 * K1; t += blockDim.x) {
            const int t2 = t / K1, c1 = t % K1;
            const int64_t q2 = q2a + t2;
            const double *n2t = Ntab(v2, p, q2), *m2t = Mtab(v2, p, q2);
            const int c2s = (int)(v2.span[q2] - k2a);
            double X1[3] = {0, 0, 0}, X2[3] = {0, 0, 0}, X3[3] = {0, 0, 0};
            for (int r = 0; r <= p; ++r) {
                const double nv = n2t[2 * r], mv = r < p ? m2t[r] : 0.0;
                #pragma unroll
                for (int c = 0; c < 3; ++c) {
                    X1[c] = fma(nv, Asm[((0 * 3 + c) * K2M + c2s + r) * K1M + c1], X1[c]);
                    X3[c] = fma(nv, Asm[((2 * 3 + c) * K2M + c2s + r) * K1M + c1], X3[c]);
                    if (r < p) X2[c] = fma(mv, Asm[((1 * 3 + c) * K2M + c2s + 1 + r) * K1M + c1], X2[c]);
                }
            }
            #pragma unroll
            for (int c = 0; c < 3; ++c) {
                Xsm[((t2 * 3 + 0) * 3 + c) * K1M + c1] = X1[c];
                Xsm[((t2 * 3 + 1) * 3 + c) * K1M + c1] = X2[c];
                Xsm[((t2 * 3 + 2) * 3 + c) * K1M + c1] = X3[c];
            }
        }
        __syncthreads();
    } else if (D == 2) {
        // stage B directly on the control net: X1 = N2 . Q^1, X2 = M2 . Q^2
        for (int t = tid; t < nt2 * K1; t += blockDim.x) {
            const int t2 = t / K1, c1 = t % K1;
            const int64_t q2 = q2off + q2a + t2;
            const double *n2t = Ntab(v2, p, q2), *m2t = Mtab(v2, p, q2);
            const int64_t e2 = v2.span[q2];
            const int64_t k1 = k1a + c1;
            const double s1 = k1 >= 1 ? dscale(v1, p, k1) : 0.0;
            double X1[2] = {0, 0}, X2[2] = {0, 0}, prev[2] = {0, 0};
            for (int r = 0; r <= p; ++r) {
                const int64_t k2 = e2 + r;
                const int64_t k = k1 + n1 * k2;
                const double s2 = r >= 1 ? dscale(v2, p, k2) : 0.0;
                #pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const double cur = k1 < n1 ? __ldg(P + k * 2 + c) : 0.0;
                    const double d1 = (k1 >= 1 && k1 < n1) ? (cur - __ldg(P + (k - 1) * 2 + c)) * s1 : 0.0;
                    X1[c] = fma(n2t[2 * r], d1, X1[c]);
                    if (r >= 1) X2[c] = fma(m2t[r - 1], (cur - prev[c]) * s2, X2[c]);
                    prev[c] = cur;
                }
            }
            #pragma unroll
            for (int c = 0; c < 2; ++c) {
                Xsm[((t2 * 3 + 0) * 3 + c) * K1M + c1] = X1[c];
                Xsm[((t2 * 3 + 1) * 3 + c) * K1M + c1] = X2[c];
            }
        }
        __syncthreads();
    }
    // stage C: one thread per point (q1, q2) of the tile
    const int t1 = tid % TQ1, t2 = D >= 2 ? tid / TQ1 : 0;
    if (t1 >= nt1 || (D >= 2 && t2 >= nt2) || (D == 1 && tid >= TQ1)) return;
    const int64_t q1 = q1a + t1;
    const double *n1t = Ntab(v1, p, q1off + q1), *m1t = Mtab(v1, p, q1off + q1);
    const int64_t e1 = v1.span[q1off + q1];
    const int c1s = (int)(e1 - k1a);
    const int64_t ld1 = D == 3 ? a.cld1 : nq1;
    const int64_t npts_plane = ld1 * (D >= 2 ? nq2 : 1);
    const int64_t npts = a.cstride;
    {
        double J[3][3];
        #pragma unroll
        for (int c = 0; c < 3; ++c)
            #pragma unroll
            for (int m = 0; m < 3; ++m) J[c][m] = 0.0;
        if (D == 1) {
            for (int r = 0; r < p; ++r) {
                const int64_t k = e1 + 1 + r;
                J[0][0] = fma(m1t[r], (__ldg(P + k) - __ldg(P + k - 1)) * dscale(v1, p, k), J[0][0]);
            }
        } else {
            const double *X = Xsm + (t2 * 3) * 3 * K1M;
            for (int r = 0; r <= p; ++r) {
                const double nv = n1t[2 * r], mv = r < p ? m1t[r] : 0.0;
                #pragma unroll
                for (int c = 0; c < D; ++c) {
                    if (r < p) J[c][0] = fma(mv, X[(0 * 3 + c) * K1M + c1s + 1 + r], J[c][0]);
                    J[c][1] = fma(nv, X[(1 * 3 + c) * K1M + c1s + r], J[c][1]);
                    if (D == 3) J[c][2] = fma(nv, X[(2 * 3 + c) * K1M + c1s + r], J[c][2]);
                }
            }
        }
        double det, adj[3][3];
        if (D == 1) {
            det = J[0][0];
            adj[0][0] = 1.0;
        } else if (D == 2) {
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
        if (!(det > 0.0) && !(det < 0.0)) atomicOr(&a.flags->det_zero, 1);
        else if (det > 0.0) { if (!a.flags->det_pos) atomicOr(&a.flags->det_pos, 1); }
        else { if (!a.flags->det_neg) atomicOr(&a.flags->det_neg, 1); }
        const double ad = fabs(det);
        const double inv = 1.0 / ad;
        const int64_t pt = (D == 3 ? a.c0off : 0) + q1 + ld1 * (D >= 2 ? (q2a + t2) : 0) + (D == 3 ? npts_plane * q3l : 0);
        int comp = 0;
        if (a.need_s) {
            #pragma unroll
            for (int l = 0; l < D; ++l)
                #pragma unroll
                for (int m = l; m < D; ++m) {
                    double s = 0.0;
                    #pragma unroll
                    for (int k = 0; k < D; ++k) s = fma(adj[l][k], adj[m][k], s);
                    if (D == 3 && a.zlayout)
                        a.coefz[(int64_t)comp * a.zcs + (q1 * v2.nq + q2a + t2) * a.zld + q3l] = s * inv;
                    else
                        a.coef[(int64_t)comp * npts + pt] = s * inv;
                    ++comp;
                }
        }
        if (a.need_m) a.coef[(int64_t)(a.zlayout ? 0 : comp) * npts + pt] = ad;
    }
}

// z layout (d = 3, stiffness for the z-line kernel): the same sum factorisation with the roles of
// the directions permuted so that the fast thread index runs along q_3, the contiguous axis of
// [comp][q_1][q_2][q_3], while stage A still reads the control net along its contiguous k_1:
// CTA = TQF q_3 points x TQM q_1 points of one q_2 plane;
//   stage A contracts k_2 (plane):   A0 = N2 . Q^1, A1 = M2 . Q^2, A2 = N2 . Q^3   (threads over k_1, k_3)
//   stage B contracts k_1:           X0 = M1 . A0,  X1 = N1 . A1,  X2 = N1 . A2
//   stage C contracts k_3 per point: J[:,0] = N3 . X0, J[:,1] = N3 . X1, J[:,2] = M3 . X2
constexpr int TQF = 32;

// derivative control nets (d = 3): Q^m_k = (P_k - P_{k - e_m}) p / (xi_{k_m + p} - xi_{k_m}) for k_m >= 1,
// else 0; [k][m][c], one thread per control point.  Same expressions as the inline differences of
// k_coef (bit-identical), computed once per build instead of (p+1) times per grid tile.
__global__ void k_dnet(const double *__restrict__ P, double *__restrict__ Q, DirView v0, DirView v1, DirView v2,
                       int p, int64_t ntot) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ntot) return;
    const int64_t n0 = v0.n, n1 = v1.n;
    const int64_t k0 = k % n0, k1 = (k / n0) % n1, k2 = k / (n0 * n1);
    const double s0 = k0 >= 1 ? dscale(v0, p, k0) : 0.0;
    const double s1 = k1 >= 1 ? dscale(v1, p, k1) : 0.0;
    const double s2 = k2 >= 1 ? dscale(v2, p, k2) : 0.0;
    #pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double cur = P[k * 3 + c];
        Q[k * 9 + 0 + c] = k0 >= 1 ? (cur - P[(k - 1) * 3 + c]) * s0 : 0.0;
        Q[k * 9 + 3 + c] = k1 >= 1 ? (cur - P[(k - n0) * 3 + c]) * s1 : 0.0;
        Q[k * 9 + 6 + c] = k2 >= 1 ? (cur - P[(k - n0 * n1) * 3 + c]) * s2 : 0.0;
    }
}
// PP > 0: the degree as a compile-time constant (p <= 6), so that the r loops unroll and each thread
// issues all of its derivative-net loads of stage A before the first FMA (the kernel is bound by
// their L2 latency); PP = 0: any degree
template <int TQM, int PP>
__global__ void __launch_bounds__(TQF * TQM, TQM == 16 ? 3 : 1) k_coefz(CoefArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int p = PP > 0 ? PP : a.p;
    const DirView &v0 = a.v[0], &v1 = a.v[1], &v2 = a.v[2];
    const int64_t q1p = blockIdx.z;  // plane (direction 2)
    const int64_t qfa = (int64_t)blockIdx.x * TQF, qma = (int64_t)blockIdx.y * TQM;  // q_3 local, q_1
    const int64_t nqf = a.nq_loc_d, nqm = v0.nq;
    const int64_t qfe = qfa + TQF < nqf ? qfa + TQF : nqf, qme = qma + TQM < nqm ? qma + TQM : nqm;
    const int ntf = (int)(qfe - qfa), ntm = (int)(qme - qma);
    const int64_t cqb = a.cq_b;
    const int64_t kfa = v2.span[cqb + qfa], kfe = v2.span[cqb + qfe - 1] + p + 1;
    const int64_t kma = v0.span[qma], kme = v0.span[qme - 1] + p + 1;
    const int KF = (int)(kfe - kfa), KM = (int)(kme - kma);
    const int KFM = TQF + p + 1, KMM = TQM + p + 1;
    double *Asm = sm;                      // [3 variants][3 comps][KFM][KMM]  (k_1 fastest)
    double *Xsm = sm;                      // [TQM][3 variants][3 comps][KFM], over Asm once stage B has read it
    const int tid = threadIdx.x;
    const double *P = a.ctrl;
    const int64_t n0 = v0.n, n1 = v1.n;
    {
        // stage A: contract k_2 with the plane's basis.  Threads over (k_3, e) with e = (k_1 - kma)*9 +
        // 3*variant + comp: for fixed (k_2, k_3) the derivative-net entries of the tile's k_1 range are
        // one contiguous run, so consecutive threads load consecutive doubles (coalesced); every
        // entry is an independent sum over k_2 (variants 0, 2 with N2, variant 1 with M2)
        const double *nt = Ntab(v1, p, q1p), *mt = Mtab(v1, p, q1p);
        const int64_t e1 = v1.span[q1p];
        const double *Q = a.dnet;
        const int KE = KM * 9;
        for (int t = tid; t < KF * KE; t += blockDim.x) {
            const int cf = t / KE, e = t % KE;
            const int cm = e / 9, vc = e % 9, var = vc / 3;
            const double *Qe = Q + (kma + n0 * (e1 + n1 * (kfa + cf))) * 9 + e;
            double acc = 0.0;
            #pragma unroll
            for (int r = 0; r <= p; ++r) {
                const double w = var == 1 ? (r >= 1 ? mt[r - 1] : 0.0) : nt[2 * r];
                if (var != 1 || r >= 1) acc = fma(w, __ldg(Qe + r * n0 * 9), acc);
            }
            Asm[(vc * KFM + cf) * KMM + cm] = acc;
        }
    }
    __syncthreads();
    // stage B: contract k_1 for each q_1 point of the tile.  A thread's (at most XIT) items are held in
    // registers until every thread has read Asm, then X is written over it (smem per CTA = max of
    // the two arrays instead of their sum: one more CTA per SM)
    constexpr int XIT = 2;  // ceil((TQF + p + 1) / TQF) items per thread for p < TQF
    double Xr[XIT][9];
    #pragma unroll
    for (int it = 0; it < XIT; ++it) {
        const int t = tid + it * (int)blockDim.x;
        if (t >= ntm * KF) break;
        const int tm = t / KF, cf = t % KF;
        const int64_t q0 = qma + tm;
        const double *nt = Ntab(v0, p, q0), *mt = Mtab(v0, p, q0);
        const int cms = (int)(v0.span[q0] - kma);
        double X0[3] = {0, 0, 0}, X1[3] = {0, 0, 0}, X2[3] = {0, 0, 0};
        #pragma unroll
        for (int r = 0; r <= p; ++r) {
            const double nv = nt[2 * r], mv = r < p ? mt[r] : 0.0;
            #pragma unroll
            for (int c = 0; c < 3; ++c) {
                X1[c] = fma(nv, Asm[((1 * 3 + c) * KFM + cf) * KMM + cms + r], X1[c]);
                X2[c] = fma(nv, Asm[((2 * 3 + c) * KFM + cf) * KMM + cms + r], X2[c]);
                if (r < p) X0[c] = fma(mv, Asm[((0 * 3 + c) * KFM + cf) * KMM + cms + 1 + r], X0[c]);
            }
        }
        #pragma unroll
        for (int c = 0; c < 3; ++c) { Xr[it][c] = X0[c]; Xr[it][3 + c] = X1[c]; Xr[it][6 + c] = X2[c]; }
    }
    __syncthreads();
    #pragma unroll
    for (int it = 0; it < XIT; ++it) {
        const int t = tid + it * (int)blockDim.x;
        if (t >= ntm * KF) break;
        const int tm = t / KF, cf = t % KF;
        #pragma unroll
        for (int vc = 0; vc < 9; ++vc) Xsm[(tm * 9 + vc) * KFM + cf] = Xr[it][vc];
    }
    __syncthreads();
    // stage C: one thread per point (q_3 fastest)
    const int tf = tid % TQF, tm = tid / TQF;
    if (tf >= ntf || tm >= ntm) return;
    const int64_t q2l = qfa + tf, q0 = qma + tm;
    const double *nt = Ntab(v2, p, cqb + q2l), *mt = Mtab(v2, p, cqb + q2l);
    const int cfs = (int)(v2.span[cqb + q2l] - kfa);
    double J[3][3];
    #pragma unroll
    for (int c = 0; c < 3; ++c)
        #pragma unroll
        for (int m = 0; m < 3; ++m) J[c][m] = 0.0;
    const double *X = Xsm + (tm * 3) * 3 * KFM;
    #pragma unroll
    for (int r = 0; r <= p; ++r) {
        const double nv = nt[2 * r], mv = r < p ? mt[r] : 0.0;
        #pragma unroll
        for (int c = 0; c < 3; ++c) {
            J[c][0] = fma(nv, X[(0 * 3 + c) * KFM + cfs + r], J[c][0]);
            J[c][1] = fma(nv, X[(1 * 3 + c) * KFM + cfs + r], J[c][1]);
            if (r < p) J[c][2] = fma(mv, X[(2 * 3 + c) * KFM + cfs + 1 + r], J[c][2]);
        }
    }
    double adj[3][3];
    adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double det = J[0][0] * adj[0][0] + J[0][1] * adj[1][0] + J[0][2] * adj[2][0];
    if (!(det > 0.0) && !(det < 0.0)) atomicOr(&a.flags->det_zero, 1);
    else if (det > 0.0) { if (!a.flags->det_pos) atomicOr(&a.flags->det_pos, 1); }
    else { if (!a.flags->det_neg) atomicOr(&a.flags->det_neg, 1); }
    const double ad = fabs(det), inv = 1.0 / ad;
    int comp = 0;
    #pragma unroll
    for (int l = 0; l < 3; ++l)
        #pragma unroll
        for (int m = l; m < 3; ++m) {
            double sv = 0.0;
            #pragma unroll
            for (int k = 0; k < 3; ++k) sv = fma(adj[l][k], adj[m][k], sv);
            a.coefz[(int64_t)comp * a.zcs + (q0 * v1.nq + q1p) * a.zld + q2l] = sv * inv;
            ++comp;
        }
    if (a.need_m) a.coef[a.c0off + q0 + a.cld1 * (q1p + v1.nq * q2l)] = ad;  // standard layout, component 0
}

}  // namespace

wq_status launch_coef(wq_plan_s *P, const double *ctrl, cudaStream_t s) {
    CoefArgs a;
    a.dnet = nullptr;
    for (int l = 0; l < 3; ++l) a.v[l] = P->dir[l];
    a.d = P->d;
    a.p = P->p;
    a.ctrl = ctrl;
    a.coef = P->coef;
    a.cq_b = P->cq_b;
    a.nq_loc_d = P->cq_e - P->cq_b;
    a.cld1 = P->cld1;
    a.c0off = P->c0off;
    a.cstride = P->cstride;
    a.ncomp_s = P->ncomp_s;
    a.ncomp = P->ncomp;
    a.need_s = P->need_stiff;
    a.need_m = P->need_mass;
    a.flags = P->flags;
    a.zlayout = P->zlayout;
    a.coefz = P->coefz;
    a.zld = P->zld;
    a.zcs = P->zcs;
    const int K1M = TQ1 + P->p + 1, K2M = TQ2 + P->p + 1;
    if (P->d == 3 && P->zlayout) {
        const int64_t ntot = P->dir[0].n * P->dir[1].n * P->dir[2].n;
        if (P->dnet_bytes < sizeof(double) * 9 * (size_t)ntot) {
            if (P->dnet) cudaFree(P->dnet);
            P->dnet_bytes = sizeof(double) * 9 * (size_t)ntot;
            if (cudaMalloc((void **)&P->dnet, P->dnet_bytes) != cudaSuccess) {
                P->dnet = nullptr;
                P->dnet_bytes = 0;
                wq_set_error("derivative control-net allocation failed");
                return WQ_ENOMEM;
            }
        }
        k_dnet<<<(unsigned)((ntot + 255) / 256), 256, 0, s>>>(ctrl, P->dnet, P->dir[0], P->dir[1], P->dir[2], P->p, ntot);
        wq_count_launches(1);
        a.dnet = P->dnet;
        const int tqm = getenv("WQ_COEF_TQM") ? atoi(getenv("WQ_COEF_TQM")) : 16;  // tile height (tuning experiments)
        auto run = [&](auto TT, auto PPc) {
            constexpr int TQM = decltype(TT)::value, PP = decltype(PPc)::value;
            const size_t na = (size_t)9 * (TQM + P->p + 1) * (TQF + P->p + 1), nx = (size_t)TQM * 9 * (TQF + P->p + 1);
            const size_t sm = (na > nx ? na : nx) * sizeof(double);
            cudaFuncSetAttribute(k_coefz<TQM, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
            dim3 g((unsigned)((a.nq_loc_d + TQF - 1) / TQF), (unsigned)((P->dir[0].nq + TQM - 1) / TQM), (unsigned)P->dir[1].nq);
            k_coefz<TQM, PP><<<g, TQF * TQM, sm, s>>>(a);
        };
        auto run_p = [&](auto TT) {
            switch (P->p) {
            case 2: run(TT, std::integral_constant<int, 2>{}); break;
            case 3: run(TT, std::integral_constant<int, 3>{}); break;
            case 4: run(TT, std::integral_constant<int, 4>{}); break;
            case 5: run(TT, std::integral_constant<int, 5>{}); break;
            case 6: run(TT, std::integral_constant<int, 6>{}); break;
            default: run(TT, std::integral_constant<int, 0>{}); break;
            }
        };
        if (tqm == 4) run_p(std::integral_constant<int, 4>{});
        else if (tqm == 16) run_p(std::integral_constant<int, 16>{});
        else run_p(std::integral_constant<int, 8>{});
    } else if (P->d == 3) {
        size_t sm = (size_t)(9 * K2M * K1M + TQ2 * 9 * K1M) * sizeof(double);
        static bool set = false;
        if (!set) { cudaFuncSetAttribute(k_coef<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024); set = true; }
        dim3 g((unsigned)a.nq_loc_d, (unsigned)((P->dir[0].nq + TQ1 - 1) / TQ1),
               (unsigned)((P->dir[1].nq + TQ2 - 1) / TQ2));
        k_coef<3><<<g, NTC, sm, s>>>(a);
    } else if (P->d == 2) {
        size_t sm = (size_t)(TQ2 * 9 * K1M) * sizeof(double);
        dim3 g((unsigned)((P->dir[0].nq + TQ1 - 1) / TQ1), (unsigned)((a.nq_loc_d + TQ2 - 1) / TQ2), 1);
        k_coef<2><<<g, NTC, sm, s>>>(a);
    } else {
        dim3 g((unsigned)((a.nq_loc_d + TQ1 - 1) / TQ1), 1, 1);
        k_coef<1><<<g, NTC, 0, s>>>(a);
    }
    wq_count_launches(1);
    return wq_cuda_status(cudaGetLastError(), "coefficient kernel");
}
