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
#include <algorithm>
#include "wq_internal.cuh"

namespace {

constexpr int TQ1 = 32;  // q_1 points per CTA
constexpr int TQ2 = 8;   // q_2 points per CTA (D >= 2); threads = TQ1 * TQ2, one per point in stage C
constexpr int NTC = TQ1 * TQ2;

struct CoefArgs {
    DirView v[3];
    int d, p;
    const double *ctrl;   // [N_DOF][d]
    const double *kappa;  // [N_DOF] diffusion coefficient net or null (= 1), reading R17
    const double *gamma;  // [N_DOF] reaction coefficient net or null (= 1)
    double *coef;         // [ncomp][cs] (d = 3: z layout, d <= 2: standard; wq_internal.cuh CoefView)
    int64_t cs;
    int64_t cq_b;         // first q_d of the sub-grid
    int64_t nq_loc_d;     // q_d extent of the sub-grid
    int ncomp_s, comp_mass;
    int need_s, need_m;
    Flags *flags;
    const double *dnet;   // d = 3: derivative control nets (+ coefficient nets) [k][NE] (k_dnet)
    int64_t k3b;          // first control plane held in dnet
    int64_t zld;          // d = 3: z-layout row length
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

// d <= 2 (standard layout): the control net read directly; CTA = TQ1 x TQ2 points (d = 2) or TQ1
// points (d = 1).  The coefficient nets kappa, gamma are evaluated with the plain basis values.
template <int D>
__global__ void __launch_bounds__(NTC) k_coef(CoefArgs a) {
    static_assert(D == 1 || D == 2, "d <= 2");
    extern __shared__ __align__(16) double sm[];
    const int p = a.p;
    const DirView &v1 = a.v[0], &v2 = a.v[1];
    const int64_t q1a = (int64_t)blockIdx.x * TQ1;
    const int64_t q2a = D >= 2 ? (int64_t)blockIdx.y * TQ2 : 0;
    const int64_t q1off = D == 1 ? a.cq_b : 0;  // D == 1: direction 1 is the slab direction
    const int64_t nq1 = D == 1 ? a.nq_loc_d : v1.nq;
    const int64_t nq2 = D == 2 ? a.nq_loc_d : 1;
    const int64_t q2off = D == 2 ? a.cq_b : 0;  // D == 2: direction 2 is the slab direction
    const int64_t q1e = q1a + TQ1 < nq1 ? q1a + TQ1 : nq1;
    const int64_t q2e = q2a + TQ2 < nq2 ? q2a + TQ2 : nq2;
    const int nt1 = (int)(q1e - q1a), nt2 = (int)(q2e - q2a);
    const int64_t k1a = v1.span[q1off + q1a];
    const int64_t n1 = v1.n;
    const int K1M = TQ1 + p + 1;
    // smem (D == 2): X[TQ2][5 rows: 0,1 = N2.Q^1 (2 comps), 2,3 = M2.Q^2, 4 = N2.kappa, 5 = N2.gamma][K1M]
    double *Xsm = sm;
    const int tid = threadIdx.x;
    const double *P = a.ctrl;
    if (D == 2) {
        const int K1 = (int)(v1.span[q1e - 1] + p + 1 - k1a);
        for (int t = tid; t < nt2 * K1; t += blockDim.x) {
            const int t2 = t / K1, c1 = t % K1;
            const int64_t q2 = q2off + q2a + t2;
            const double *n2t = Ntab(v2, p, q2), *m2t = Mtab(v2, p, q2);
            const int64_t e2 = v2.span[q2];
            const int64_t k1 = k1a + c1;
            const double s1 = k1 >= 1 ? dscale(v1, p, k1) : 0.0;
            double X1[2] = {0, 0}, X2[2] = {0, 0}, prev[2] = {0, 0}, Xk = 0.0, Xg = 0.0;
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
                if (a.kappa && k1 < n1) Xk = fma(n2t[2 * r], __ldg(a.kappa + k), Xk);
                if (a.gamma && k1 < n1) Xg = fma(n2t[2 * r], __ldg(a.gamma + k), Xg);
            }
            double *X = Xsm + t2 * 6 * K1M + c1;
            X[0 * K1M] = X1[0]; X[1 * K1M] = X1[1]; X[2 * K1M] = X2[0]; X[3 * K1M] = X2[1];
            X[4 * K1M] = Xk; X[5 * K1M] = Xg;
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
    double J[2][2] = {{0, 0}, {0, 0}}, kap = a.kappa ? 0.0 : 1.0, gam = a.gamma ? 0.0 : 1.0;
    if (D == 1) {
        for (int r = 0; r < p; ++r) {
            const int64_t k = e1 + 1 + r;
            J[0][0] = fma(m1t[r], (__ldg(P + k) - __ldg(P + k - 1)) * dscale(v1, p, k), J[0][0]);
        }
        for (int r = 0; r <= p; ++r) {
            if (a.kappa) kap = fma(n1t[2 * r], __ldg(a.kappa + e1 + r), kap);
            if (a.gamma) gam = fma(n1t[2 * r], __ldg(a.gamma + e1 + r), gam);
        }
    } else {
        const double *X = Xsm + t2 * 6 * K1M;
        for (int r = 0; r <= p; ++r) {
            const double nv = n1t[2 * r], mv = r < p ? m1t[r] : 0.0;
            #pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (r < p) J[c][0] = fma(mv, X[c * K1M + c1s + 1 + r], J[c][0]);
                J[c][1] = fma(nv, X[(2 + c) * K1M + c1s + r], J[c][1]);
            }
            if (a.kappa) kap = fma(nv, X[4 * K1M + c1s + r], kap);
            if (a.gamma) gam = fma(nv, X[5 * K1M + c1s + r], gam);
        }
    }
    double det, adj[2][2];
    if (D == 1) {
        det = J[0][0];
        adj[0][0] = 1.0;
    } else {
        det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        adj[0][0] = J[1][1]; adj[0][1] = -J[0][1];
        adj[1][0] = -J[1][0]; adj[1][1] = J[0][0];
    }
    if (!(det > 0.0) && !(det < 0.0)) atomicOr(&a.flags->det_zero, 1);
    else if (det > 0.0) { if (!a.flags->det_pos) atomicOr(&a.flags->det_pos, 1); }
    else { if (!a.flags->det_neg) atomicOr(&a.flags->det_neg, 1); }
    const double ad = fabs(det);
    const double inv = kap / ad;
    const int64_t pt = q1 + (D == 2 ? v1.nq * (q2a + t2) : 0);
    if (a.need_s) {
        int comp = 0;
        #pragma unroll
        for (int l = 0; l < D; ++l)
            #pragma unroll
            for (int m = l; m < D; ++m) {
                double sv = 0.0;
                #pragma unroll
                for (int k = 0; k < D; ++k) sv = fma(adj[l][k], adj[m][k], sv);
                a.coef[(int64_t)comp * a.cs + pt] = sv * inv;
                ++comp;
            }
    }
    if (a.need_m) a.coef[(int64_t)a.comp_mass * a.cs + pt] = gam * ad;
}

// derivative control nets (d = 3): Q^m_k = (P_k - P_{k - e_m}) p / (xi_{k_m + p} - xi_{k_m}) for k_m >= 1,
// else 0, then the coefficient nets: [k][NE], NE = 9 + NNU, entries (m, c) = 3 m + c, 9 = kappa,
// 9 or 10 = gamma; one thread per control point of the planes k_3 in [k3b, k3b + ntot / (n0 n1)).
template <int NNU>
__global__ void __launch_bounds__(256) k_dnet(const double *__restrict__ P, const double *__restrict__ kap,
                                              const double *__restrict__ gam, double *__restrict__ Q, DirView v0,
                                              DirView v1, DirView v2, int p, int64_t k3b, int64_t ntot) {
    constexpr int NE = 9 + NNU;
    // the CTA's 256 consecutive control points are written as one contiguous run of 256 NE doubles:
    // staged in shared memory, then stored with consecutive threads on consecutive words
    __shared__ double st[256 * NE];
    const int64_t kb = (int64_t)blockIdx.x * 256;
    const int64_t kl = kb + threadIdx.x;
    if (kl < ntot) {
        const int64_t n0 = v0.n, n1 = v1.n;
        const int64_t k0 = kl % n0, k1 = (kl / n0) % n1, k2 = k3b + kl / (n0 * n1);
        const int64_t k = k0 + n0 * (k1 + n1 * k2);
        const double s0 = k0 >= 1 ? dscale(v0, p, k0) : 0.0;
        const double s1 = k1 >= 1 ? dscale(v1, p, k1) : 0.0;
        const double s2 = k2 >= 1 ? dscale(v2, p, k2) : 0.0;
        double *q = st + threadIdx.x * NE;
        #pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double cur = P[k * 3 + c];
            q[0 + c] = k0 >= 1 ? (cur - P[(k - 1) * 3 + c]) * s0 : 0.0;
            q[3 + c] = k1 >= 1 ? (cur - P[(k - n0) * 3 + c]) * s1 : 0.0;
            q[6 + c] = k2 >= 1 ? (cur - P[(k - n0 * n1) * 3 + c]) * s2 : 0.0;
        }
        int e = 9;
        if (NNU > 0 && kap) q[e++] = kap[k];
        if (NNU > 0 && gam) q[e++] = gam[k];
    }
    __syncthreads();
    const int64_t nv = (ntot - kb < 256 ? ntot - kb : 256) * NE;
    double *out = Q + kb * NE;
    for (int x = threadIdx.x; x < nv; x += 256) out[x] = st[x];
}
// Tiled form (p <= 6): CTA = TQF points q_3 x TQM points q_1 of one q_2 plane, the three
// contractions of the tile in one kernel:
//   stage A contracts k_2 (plane):   A0 = N2 . Q^1, A1 = M2 . Q^2, A2 = N2 . Q^3, Ak = N2 . kappa, ...
//   stage B contracts k_1:           X0 = M1 . A0,  X1 = N1 . A1,  X2 = N1 . A2,  Xk = N1 . Ak
//   stage C contracts k_3 per point: J[:,0] = N3 . X0, J[:,1] = N3 . X1, J[:,2] = M3 . X2,
//                                    kappa = N3 . Xk, gamma likewise
constexpr int TQF = 32;
// PP > 0: the degree as a compile-time constant (p <= 6), so that the r loops unroll and each thread
// issues all of its derivative-net loads of stage A before the first FMA (the kernel is bound by
// their L2 latency); PP = 0: any degree.  NNU: number of coefficient nets (0..2).
template <int TQM, int PP, int NNU, int MINB>
__global__ void __launch_bounds__(TQF * TQM, MINB) k_coefz(CoefArgs a) {
    constexpr int NE = 9 + NNU;
    extern __shared__ __align__(16) double sm[];
    static_assert(PP > 0, "compile-time degree");
    const int p = PP;
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
    // k windows of the tile: 32 (16) consecutive points lie in at most 17 (9) spans (two points per
    // interior span, reading R1), so KF <= TQF/2 + 1 + p and KM <= TQM/2 + 1 + p
    constexpr int KFM = TQF / 2 + 2 + PP, KMM = TQM / 2 + 2 + PP;
    if (KF > KFM || KM > KMM) __trap();  // point-layout invariant
    constexpr int NEP = (NE + 1) & ~1;     // X row: the NE entries padded to whole double2 pairs
    constexpr int BS = wq_bstride(PP), BSP = BS + 1;  // table rows, padded to an odd stride in smem
    // A row (one k_3): the tile's k_1 window x NE entries, padded to an odd length so that the lanes
    // of stage B (consecutive k_3) hit distinct banks
    constexpr int RL = (KMM * NE) | 1;
    double *Asm = sm;                                   // [KFM][RL]: entry (k_1 - kma) * NE + e
    double *Xsm = Asm + ((KFM * RL + 1) & ~1);          // [TQM][KFM][NEP]
    double *T2s = Xsm + TQM * KFM * NEP;                // [TQF][BSP] basis rows of the tile's q_3 points
    double *T0s = T2s + TQF * BSP;                      // [TQM][BSP] basis rows of the tile's q_1 points
    const int tid = threadIdx.x;
    const int64_t n0 = v0.n, n1 = v1.n;
    {
        const double *b2 = v2.B + (cqb + qfa) * BS, *b0 = v0.B + qma * BS;
        for (int x = tid; x < ntf * BS; x += TQF * TQM) T2s[(x / BS) * BSP + x % BS] = b2[x];
        for (int x = tid; x < ntm * BS; x += TQF * TQM) T0s[(x / BS) * BSP + x % BS] = b0[x];
    }
    {
        // stage A: contract k_2 with the plane's basis.  Thread = one fixed column e = (k_1 - kma)*NE +
        // entry of the tile and a row group g, looping over the rows k_3 = g, g + G, ...: for fixed
        // (k_2, k_3) the net entries of the tile's k_1 range are one contiguous run, so consecutive
        // threads load consecutive doubles (coalesced); the column's weights sit in registers and the
        // loop only advances two pointers (derivative in direction 2 (entries 3..5) with M2, all others
        // with N2; the M2 column's weight 0 is paired with the valid row span, so every lane loads)
        const double *nt = Ntab(v1, p, q1p), *mt = Mtab(v1, p, q1p);
        const int64_t e1 = v1.span[q1p];
        // fixed thread -> (row group, column) map for the largest window (compile-time divisions)
        constexpr int KEM = KMM * NE, G = TQF * TQM / KEM;
        static_assert(G >= 1, "one row group");
        const int g = tid / KEM, e = tid - g * KEM;
        if (g < G && e < KM * NE) {
            const int cm = e / NE, vc = e - cm * NE;
            const bool dv = vc >= 3 && vc < 6;
            double w[PP + 1];
            #pragma unroll
            for (int r = 0; r <= PP; ++r) w[r] = dv ? (r >= 1 ? mt[r - 1] : 0.0) : nt[2 * r];
            const int64_t rs = n0 * NE, ps = n0 * n1 * NE * G;
            const double *Qe = a.dnet + (kma + n0 * (e1 + n1 * (kfa - a.k3b + g))) * NE + e;
            double *As = Asm + g * RL + e;  // consecutive lanes, consecutive words
            #pragma unroll 2
            for (int cf = g; cf < KF; cf += G, Qe += ps, As += G * RL) {
                double acc = 0.0;
                #pragma unroll
                for (int r = 0; r <= PP; ++r) acc = fma(w[r], __ldg(Qe + r * rs), acc);
                *As = acc;
            }
        }
    }
    __syncthreads();
    // stage B: contract k_1 for each q_1 point of the tile (items (q_1, k_3), k_3 fastest)
    for (int t = tid; t < ntm * KF; t += TQF * TQM) {
        const int tm = t / KF, cf = t - tm * KF;
        const double *nt = T0s + tm * BSP, *mt = nt + 2 * (PP + 1);
        const int cms = (int)(v0.span[qma + tm] - kma);
        double X[NEP];
        #pragma unroll
        for (int vc = 0; vc < NEP; ++vc) X[vc] = 0.0;
        #pragma unroll
        for (int r = 0; r <= PP; ++r) {
            const double nv = nt[2 * r], mv = r < PP ? mt[r] : 0.0;
            #pragma unroll
            for (int vc = 0; vc < NE; ++vc) {
                if (vc < 3) {  // derivative in direction 1: M1
                    if (r < PP) X[vc] = fma(mv, Asm[cf * RL + (cms + 1 + r) * NE + vc], X[vc]);
                } else {
                    X[vc] = fma(nv, Asm[cf * RL + (cms + r) * NE + vc], X[vc]);
                }
            }
        }
        double2 *xr = (double2 *)(Xsm + (tm * KFM + cf) * NEP);
        #pragma unroll
        for (int h = 0; h < NEP / 2; ++h) xr[h] = make_double2(X[2 * h], X[2 * h + 1]);
    }
    __syncthreads();
    // stage C: one thread per point (q_3 fastest)
    const int tf = tid % TQF, tm = tid / TQF;
    if (tf >= ntf || tm >= ntm) return;
    const int64_t q2l = qfa + tf, q0 = qma + tm;
    const double *nt = T2s + tf * BSP, *mt = nt + 2 * (PP + 1);
    const int cfs = (int)(v2.span[cqb + q2l] - kfa);
    double J[3][3], nu[2] = {0.0, 0.0};
    #pragma unroll
    for (int c = 0; c < 3; ++c)
        #pragma unroll
        for (int m = 0; m < 3; ++m) J[c][m] = 0.0;
    // rows r' = 0..p of the point's k_3 window, each read once as NEP/2 double2 (rows at an 80/96-B
    // stride: the 4 distinct rows of a quarter-warp fall on disjoint banks): entries 0..5 and the
    // coefficient nets with N3 (row r'), entries 6..8 with M3 (functions span+1.., row r' >= 1)
    const double2 *X = (const double2 *)(Xsm + (tm * KFM + cfs) * NEP);
    #pragma unroll
    for (int r = 0; r <= PP; ++r) {
        double x[NEP];
        #pragma unroll
        for (int h = 0; h < NEP / 2; ++h) {
            const double2 v = X[r * (NEP / 2) + h];
            x[2 * h] = v.x;
            x[2 * h + 1] = v.y;
        }
        const double nv = nt[2 * r];
        #pragma unroll
        for (int c = 0; c < 3; ++c) {
            J[c][0] = fma(nv, x[0 * 3 + c], J[c][0]);
            J[c][1] = fma(nv, x[1 * 3 + c], J[c][1]);
        }
        if (r >= 1) {
            const double mv = mt[r - 1];
            #pragma unroll
            for (int c = 0; c < 3; ++c) J[c][2] = fma(mv, x[2 * 3 + c], J[c][2]);
        }
        #pragma unroll
        for (int u = 0; u < NNU; ++u) nu[u] = fma(nv, x[9 + u], nu[u]);
    }
    // coefficient values: kappa then gamma among the NNU nets
    const double kap = a.kappa ? nu[0] : 1.0;
    const double gam = a.gamma ? nu[a.kappa ? 1 : 0] : 1.0;
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
    const double ad = fabs(det), inv = kap / ad;
    const int64_t pt = (q0 * v1.nq + q1p) * a.zld + q2l;
    if (a.need_s) {
        int comp = 0;
        #pragma unroll
        for (int l = 0; l < 3; ++l)
            #pragma unroll
            for (int m = l; m < 3; ++m) {
                double sv = 0.0;
                #pragma unroll
                for (int k = 0; k < 3; ++k) sv = fma(adj[l][k], adj[m][k], sv);
                a.coef[(int64_t)comp * a.cs + pt] = sv * inv;
                ++comp;
            }
    }
    if (a.need_m) a.coef[(int64_t)a.comp_mass * a.cs + pt] = gam * ad;
}

// Streaming form of the d = 3 sum factorisation (3 passes over the whole sub-grid, each a 1D
// contraction with coalesced access; the degree is a compile-time constant PP):
//   k_dnet  derivative control nets Q^m (+ coefficient nets), [k][NE]
//   k_cz12  X2[k_3][q_1][q_0][e] = sum_{k_1} T1_e(q_1, k_1) sum_{k_0} T0_e(q_0, k_0) Q[k_3][k_1][k_0][e]
//           (thread = column (q_0, e) of one control plane k_3, marching along q_1 with the p+1 rows
//           k_1 of the current span in a sliding register window)
//   k_cz3   J_e(q) = sum_{k_3} T2_e(q_2, k_3) X2[k_3][q_1][q_0][e] per point, then det J, adj J,
//           c and C; CTA = 32 points q_2 (the contiguous axis of the z layout) x 8 points q_0 of
//           one q_1 row, the X2 rows of the tile's k_3 window staged in shared memory.
// T_e is the degree p-1 table M (functions span+1..span+p) in the entry's derivative direction
// and the degree p table N (functions span..span+p) elsewhere.
template <int PP, int NNU>
__global__ void __launch_bounds__(256) k_cz12(CoefArgs a, double *__restrict__ X2, int64_t n2l) {
    constexpr int NE = 9 + NNU, p = PP;
    const DirView &v0 = a.v[0], &v1 = a.v[1];
    const int64_t nq0 = v0.nq, nq1 = v1.nq, n0 = v0.n, n1 = v1.n;
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k2l = blockIdx.y;
    if (col >= nq0 * NE) return;
    const int q0 = (int)(col / NE), e = (int)(col % NE);
    const bool m0 = e < 3, m1 = e >= 3 && e < 6;  // derivative in direction 0 / 1
    // direction-0 table of this column (registers): N values or M values
    double t0[PP + 1];
    const int64_t s0 = v0.span[q0];
    {
        const double *nt = Ntab(v0, p, q0), *mt = Mtab(v0, p, q0);
        #pragma unroll
        for (int r = 0; r <= PP; ++r) t0[r] = m0 ? (r < PP ? mt[r] : 0.0) : nt[2 * r];
    }
    const int64_t kb0 = s0 + (m0 ? 1 : 0);  // first k_0 of the contraction
    const double *Qp = a.dnet + (k2l * n1 * n0) * NE + e;
    auto x1row = [&](int64_t k1) {  // sum_{k_0} T0 Q[k_3][k_1][k_0][e]
        double s = 0.0;
        const double *q = Qp + (k1 * n0 + kb0) * NE;
        #pragma unroll
        for (int r = 0; r <= PP; ++r)
            if (!m0 || r < PP) s = fma(t0[r], __ldg(q + r * NE), s);
        return s;
    };
    double win[PP + 1];
    int64_t cur = v1.span[0];
    #pragma unroll
    for (int r = 0; r <= PP; ++r) win[r] = x1row(cur + r);
    double *out = X2 + (k2l * nq1 * nq0 + q0) * NE + e;
    for (int64_t q1 = 0; q1 < nq1; ++q1) {
        const int64_t s1 = v1.span[q1];
        while (cur < s1) {  // slide the window by one control row
            #pragma unroll
            for (int r = 0; r < PP; ++r) win[r] = win[r + 1];
            ++cur;
            win[PP] = x1row(cur + PP);
        }
        const double *nt = Ntab(v1, p, q1), *mt = Mtab(v1, p, q1);
        double s = 0.0;
        #pragma unroll
        for (int r = 0; r <= PP; ++r) {
            if (m1) { if (r < PP) s = fma(mt[r], win[r + 1], s); }
            else s = fma(nt[2 * r], win[r], s);
        }
        out[q1 * nq0 * NE] = s;
    }
}

constexpr int CZ_T2 = 32, CZ_T0 = 8;
// shared row stride of k_cz3 (doubles): CZ_T0 * NE + 1, so that the lanes' different rows k_3 fall on
// different banks
__host__ __device__ constexpr int cz_rs(int ne) { return CZ_T0 * ne + 1; }

template <int PP, int NNU>
__global__ void __launch_bounds__(CZ_T2 * CZ_T0) k_cz3(CoefArgs a, const double *__restrict__ X2) {
    constexpr int NE = 9 + NNU, p = PP;
    extern __shared__ __align__(16) double sm[];
    const DirView &v0 = a.v[0], &v1 = a.v[1], &v2 = a.v[2];
    const int64_t nq0 = v0.nq, nq1 = v1.nq, nql = a.nq_loc_d;
    const int64_t q2a = (int64_t)blockIdx.x * CZ_T2, q0a = (int64_t)blockIdx.y * CZ_T0, q1 = blockIdx.z;
    const int64_t q2e = q2a + CZ_T2 < nql ? q2a + CZ_T2 : nql, q0e = q0a + CZ_T0 < nq0 ? q0a + CZ_T0 : nq0;
    const int64_t cqb = a.cq_b;
    const int64_t kfa = v2.span[cqb + q2a], kfe = v2.span[cqb + q2e - 1] + p + 1;
    const int KF = (int)(kfe - kfa), n0t = (int)(q0e - q0a);
    const int tid = threadIdx.x;
    // stage the rows k_3 in [kfa, kfe) of X2 for this q_1 and the tile's q_0 (contiguous (q_0, e) runs)
    const int rowlen = n0t * NE;
    for (int x = tid; x < KF * rowlen; x += blockDim.x) {
        const int kr = x / rowlen, j = x % rowlen;
        sm[kr * cz_rs(NE) + j] = __ldg(X2 + (((kfa - a.k3b + kr) * nq1 + q1) * nq0 + q0a) * NE + j);
    }
    __syncthreads();
    const int t2 = tid % CZ_T2, t0 = tid / CZ_T2;
    const int64_t q2l = q2a + t2, q0 = q0a + t0;
    if (q2l >= q2e || q0 >= q0e) return;
    const double *nt = Ntab(v2, p, cqb + q2l), *mt = Mtab(v2, p, cqb + q2l);
    const int ks = (int)(v2.span[cqb + q2l] - kfa);
    double J[3][3], nu[2] = {0.0, 0.0};
    #pragma unroll
    for (int c = 0; c < 3; ++c)
        #pragma unroll
        for (int m = 0; m < 3; ++m) J[c][m] = 0.0;
    const double *S = sm + t0 * NE;
    #pragma unroll
    for (int r = 0; r <= PP; ++r) {
        const double nv = nt[2 * r], mv = r < PP ? mt[r] : 0.0;
        const double *Sr = S + (ks + r) * cz_rs(NE), *Sm = Sr + cz_rs(NE);  // M: functions span+1..
        #pragma unroll
        for (int c = 0; c < 3; ++c) {
            J[c][0] = fma(nv, Sr[0 * 3 + c], J[c][0]);
            J[c][1] = fma(nv, Sr[1 * 3 + c], J[c][1]);
            if (r < PP) J[c][2] = fma(mv, Sm[2 * 3 + c], J[c][2]);
        }
        #pragma unroll
        for (int u = 0; u < NNU; ++u) nu[u] = fma(nv, Sr[9 + u], nu[u]);
    }
    const double kap = a.kappa ? nu[0] : 1.0;
    const double gam = a.gamma ? nu[a.kappa ? 1 : 0] : 1.0;
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
    const double ad = fabs(det), inv = kap / ad;
    const int64_t pt = (q0 * nq1 + q1) * a.zld + q2l;
    if (a.need_s) {
        int comp = 0;
        #pragma unroll
        for (int l = 0; l < 3; ++l)
            #pragma unroll
            for (int m = l; m < 3; ++m) {
                double sv = 0.0;
                #pragma unroll
                for (int k = 0; k < 3; ++k) sv = fma(adj[l][k], adj[m][k], sv);
                a.coef[(int64_t)comp * a.cs + pt] = sv * inv;
                ++comp;
            }
    }
    if (a.need_m) a.coef[(int64_t)a.comp_mass * a.cs + pt] = gam * ad;
}

// z layout [comp][q_1][q_2][q_3 - cq_b] -> standard layout [comp][q_3 - cq_b][q_2][q_1] (row-tile kernel):
// 32 x 32 tiles of (q_1, q_3) for one (comp, q_2), transposed through shared memory
__global__ void __launch_bounds__(256) k_z2std(const double *__restrict__ z, double *__restrict__ st, int64_t nq0,
                                               int64_t nq1, int64_t nql, int64_t zld, int64_t zcs, int64_t scs) {
    __shared__ double tile[32][33];
    const int64_t q3a = (int64_t)blockIdx.x * 32, q0a = (int64_t)blockIdx.y * 32;
    const int64_t q1 = blockIdx.z % nq1, comp = blockIdx.z / nq1;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    for (int r = ty; r < 32; r += 8) {  // read rows q_0, contiguous along q_3
        const int64_t q0 = q0a + r, q3 = q3a + tx;
        tile[r][tx] = (q0 < nq0 && q3 < nql) ? z[comp * zcs + (q0 * nq1 + q1) * zld + q3] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // write rows q_3, contiguous along q_0
        const int64_t q3 = q3a + r, q0 = q0a + tx;
        if (q0 < nq0 && q3 < nql) st[comp * scs + (q3 * nq1 + q1) * nq0 + q0] = tile[tx][r];
    }
}

}  // namespace

static wq_status finish_coef(wq_plan_s *P, cudaStream_t s) {
    if (P->d == 3 && P->coef_std) {
        const int64_t nql = P->cq_e - P->cq_b, nq0 = P->dir[0].nq, nq1 = P->dir[1].nq;
        dim3 g((unsigned)((nql + 31) / 32), (unsigned)((nq0 + 31) / 32), (unsigned)(nq1 * P->ncomp));
        k_z2std<<<g, 256, 0, s>>>(P->coef, P->coef_std, nq0, nq1, nql, P->zld, P->zcs, P->coef_points);
        wq_count_launches(1);
    }
    return wq_cuda_status(cudaGetLastError(), "coefficient kernel");
}

wq_status launch_coef(wq_plan_s *P, const double *ctrl, const double *kappa, const double *gamma, cudaStream_t s) {
    CoefArgs a;
    a.dnet = nullptr;
    for (int l = 0; l < 3; ++l) a.v[l] = P->dir[l];
    a.d = P->d;
    a.p = P->p;
    a.ctrl = ctrl;
    a.kappa = kappa;
    a.gamma = gamma;
    a.coef = P->coef;
    a.cs = P->zcs;
    a.cq_b = P->cq_b;
    a.nq_loc_d = P->cq_e - P->cq_b;
    a.ncomp_s = P->ncomp_s;
    a.comp_mass = P->comp_mass;
    a.need_s = P->need_stiff;
    a.need_m = P->need_mass;
    a.flags = P->flags;
    a.zld = P->zld;
    a.k3b = 0;
    const int nnu = (kappa ? 1 : 0) + (gamma ? 1 : 0);
    if (P->d == 3) {
        // control planes seen by the slab's points: spans of cq_b .. cq_e - 1 plus p, and one below
        // for the derivative differences (the derivative nets are formed on the slab + halo only)
        const DirView &v2 = P->dir[2];
        const int p = P->p;
        int64_t spb = 0, spe = 0;
        {
            // span of a grid point from the integer point layout (reading R1): boundary span 0 holds
            // points 0..p+1, knot e sits at p + 2e, midpoint of span e at p + 2e + 1
            auto span_of = [&](int64_t g) -> int64_t {
                const int64_t E = v2.E, nq = v2.nq;
                if (g <= p + 1) return 0;
                if (E >= 2 && g >= p + 2 * (E - 1) + 1) return E - 1;
                if (g >= nq - 1) return E - 1;
                const int64_t t = g - p;
                return (t & 1) == 0 ? (t / 2 < E ? t / 2 : E - 1) : (t - 1) / 2;
            };
            spb = span_of(P->cq_b);
            spe = span_of(P->cq_e - 1);
        }
        const int64_t k3b = spb >= 1 ? spb - 1 : 0;       // control index of span s: s .. s + p
        const int64_t k3e = std::min<int64_t>(spe + p + 1, v2.n);
        P->k3b = k3b;
        P->k3e = k3e;
        a.k3b = k3b;
        const int64_t ntot = P->dir[0].n * P->dir[1].n * (k3e - k3b);
        const size_t need = sizeof(double) * (9 + nnu) * (size_t)ntot;
        if (P->dnet_bytes < need) {
            if (P->dnet) cudaFree(P->dnet);
            P->dnet_bytes = need;
            if (cudaMalloc((void **)&P->dnet, P->dnet_bytes) != cudaSuccess) {
                P->dnet = nullptr;
                P->dnet_bytes = 0;
                wq_set_error("derivative control-net allocation failed");
                return WQ_ENOMEM;
            }
        }
        const unsigned gd = (unsigned)((ntot + 255) / 256);
        if (nnu == 0) k_dnet<0><<<gd, 256, 0, s>>>(ctrl, kappa, gamma, P->dnet, P->dir[0], P->dir[1], P->dir[2], P->p, k3b, ntot);
        else if (nnu == 1) k_dnet<1><<<gd, 256, 0, s>>>(ctrl, kappa, gamma, P->dnet, P->dir[0], P->dir[1], P->dir[2], P->p, k3b, ntot);
        else k_dnet<2><<<gd, 256, 0, s>>>(ctrl, kappa, gamma, P->dnet, P->dir[0], P->dir[1], P->dir[2], P->p, k3b, ntot);
        wq_count_launches(1);
        a.dnet = P->dnet;
        // measured at C4 (tools/time_step.py): the tiled kernel for p <= 4, the streaming passes above
        const bool tiled = P->p >= 2 && P->p <= 4 && !getenv("WQ_COEF_STREAM");
        if (tiled) {
            constexpr int TQM = 16;
            auto runt = [&](auto PPc, auto NUc) {
                constexpr int PP = decltype(PPc)::value, NNU = decltype(NUc)::value;
                const size_t ne = 9 + NNU;
                const size_t kfm = TQF / 2 + 2 + PP, kmm = TQM / 2 + 2 + PP, bsp = wq_bstride(PP) + 1;
                const size_t na = (kfm * ((kmm * ne) | 1) + 1) & ~(size_t)1, nx = (size_t)TQM * ((ne + 1) & ~(size_t)1) * kfm;
                const size_t sm = (na + nx + (TQF + TQM) * bsp) * sizeof(double);
                dim3 g((unsigned)((a.nq_loc_d + TQF - 1) / TQF), (unsigned)((P->dir[0].nq + TQM - 1) / TQM), (unsigned)P->dir[1].nq);
                if (getenv("WQ_COEFZ_MINB2")) {
                    wq_smem_attr((const void *)k_coefz<TQM, PP, NNU, 2>, sm);
                    k_coefz<TQM, PP, NNU, 2><<<g, TQF * TQM, sm, s>>>(a);
                } else {
                    wq_smem_attr((const void *)k_coefz<TQM, PP, NNU, 3>, sm);
                    k_coefz<TQM, PP, NNU, 3><<<g, TQF * TQM, sm, s>>>(a);
                }
            };
            auto runt_p = [&](auto NUc) {
                switch (P->p) {
                case 2: runt(std::integral_constant<int, 2>{}, NUc); break;
                case 3: runt(std::integral_constant<int, 3>{}, NUc); break;
                default: runt(std::integral_constant<int, 4>{}, NUc); break;
                }
            };
            if (nnu == 0) runt_p(std::integral_constant<int, 0>{});
            else if (nnu == 1) runt_p(std::integral_constant<int, 1>{});
            else runt_p(std::integral_constant<int, 2>{});
            wq_count_launches(1);
            return finish_coef(P, s);
        }
        // X2 workspace: the slab's control planes x nq_1 x nq_0 x NE
        const int64_t n2l = k3e - k3b;
        const int ne = 9 + nnu;
        const size_t xb = sizeof(double) * (size_t)n2l * P->dir[1].nq * P->dir[0].nq * ne;
        if (P->x2_bytes < xb) {
            if (P->x2) cudaFree(P->x2);
            P->x2_bytes = xb;
            if (cudaMalloc((void **)&P->x2, xb) != cudaSuccess) {
                P->x2 = nullptr;
                P->x2_bytes = 0;
                wq_set_error("coefficient workspace allocation failed");
                return WQ_ENOMEM;
            }
        }
        auto run = [&](auto PPc, auto NUc) {
            constexpr int PP = decltype(PPc)::value, NNU = decltype(NUc)::value;
            dim3 g1((unsigned)((P->dir[0].nq * (9 + NNU) + 255) / 256), (unsigned)n2l);
            k_cz12<PP, NNU><<<g1, 256, 0, s>>>(a, P->x2, n2l);
            const int kfmax = CZ_T2 + PP + 1;
            const size_t sm = sizeof(double) * (size_t)kfmax * cz_rs(9 + NNU);
            dim3 g3((unsigned)((a.nq_loc_d + CZ_T2 - 1) / CZ_T2), (unsigned)((P->dir[0].nq + CZ_T0 - 1) / CZ_T0),
                    (unsigned)P->dir[1].nq);
            wq_smem_attr((const void *)k_cz3<PP, NNU>, sm);
            k_cz3<PP, NNU><<<g3, CZ_T2 * CZ_T0, sm, s>>>(a, P->x2);
            wq_count_launches(1);
        };
        auto run_p = [&](auto NUc) {
            switch (P->p) {
            case 1: run(std::integral_constant<int, 1>{}, NUc); break;
            case 2: run(std::integral_constant<int, 2>{}, NUc); break;
            case 3: run(std::integral_constant<int, 3>{}, NUc); break;
            case 4: run(std::integral_constant<int, 4>{}, NUc); break;
            case 5: run(std::integral_constant<int, 5>{}, NUc); break;
            case 6: run(std::integral_constant<int, 6>{}, NUc); break;
            case 7: run(std::integral_constant<int, 7>{}, NUc); break;
            case 8: run(std::integral_constant<int, 8>{}, NUc); break;
            case 9: run(std::integral_constant<int, 9>{}, NUc); break;
            default: run(std::integral_constant<int, 10>{}, NUc); break;
            }
        };
        if (nnu == 0) run_p(std::integral_constant<int, 0>{});
        else if (nnu == 1) run_p(std::integral_constant<int, 1>{});
        else run_p(std::integral_constant<int, 2>{});
    } else if (P->d == 2) {
        size_t sm = (size_t)(TQ2 * 6 * (TQ1 + P->p + 1)) * sizeof(double);
        dim3 g((unsigned)((P->dir[0].nq + TQ1 - 1) / TQ1), (unsigned)((a.nq_loc_d + TQ2 - 1) / TQ2), 1);
        k_coef<2><<<g, NTC, sm, s>>>(a);
    } else {
        dim3 g((unsigned)((a.nq_loc_d + TQ1 - 1) / TQ1), 1, 1);
        k_coef<1><<<g, NTC, 0, s>>>(a);
    }
    wq_count_launches(1);
    return finish_coef(P, s);
}
