// wq_assemble_sf2.cu -- step 7 for d <= 2 (WQ_KERNEL_SF2): the row loop of
// Alg. 3 with the sum factorisation of Eq. sumfactorization
// (P:837), one warp per row.  For a 2D row i = (i_1, i_2):
//   stage 1 (contract q_1):  Y_{lm}(t_1, c_2) = sum_{c_1} A_1^{f_1}(t_1, c_1) C_{lm}(q_1, q_2)
//   stage 2 (contract q_2):  s_ij = sum_{lm} sum_{c_2} A_2^{f_2}(t_2, c_2) Y_{lm}(t_1, c_2)
// with A_k^f(t, c) = w^f_{k,i_k,q} D^{b(f)} B_{j_k}(x_q) (family f = a + 2b,
// (a,b) = (delta_kl, delta_km), reading R3; mass: the single term f = 0 and c).
// O(#I_1 #Q_1 #Q_2 + #I_1 #I_2 #Q_2) per row, i.e. O(p) per entry instead of
// the O(p^d) of the direct kernel.
//   k_sf2l (d = 2): CTA = one i_1 and a chunk of RC consecutive rows i_2.  The
//     rows share A_1 and, over the chunk's whole point range in q_2, stage 1
//     (Y does not depend on i_2): it is done once per CTA, then stage 2 per
//     row batch with that row's A_2 (stage 1 amortised over the chunk, as the
//     line kernels of d = 3 amortise their first two contractions).
//   k_sf2 (d = 1, and d = 2 when the chunk tables do not fit): one warp per
//     row, both stages per row; d = 1 is the same code with a trivial
//     direction 2 (#Q_2 = #I_2 = 1, A_2 = 1).
#include <cstdlib>
#include "wq_rows.cuh"

namespace {

struct Sf2Args {
    RowGeo g;
    DirView v[2];
    int d, p, matrix;
    CoefView cv;
    int64_t cq_b;
    int comp_mass;
    double *val;
    int32_t *col;
    int64_t row_lo, rows;
    int64_t val_base;
    int km, qm;              // table strides: max #I (2p+1), max #Q over the directions
    int wstride;             // doubles of shared memory per warp
};

__global__ void __launch_bounds__(256) k_sf2(Sf2Args a) {
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r = a.row_lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (r >= a.row_lo + a.rows) return;
    const int p = a.p, D = a.d, KM = a.km, QM = a.qm;
    const int nf = a.matrix == 0 ? 1 : 4;
    const int nterm = a.matrix == 0 ? 1 : D * D;
    double *A1 = sm + (size_t)warp * a.wstride;  // [f][t][c]
    double *A2 = A1 + nf * KM * QM;              // [f][t][c]
    double *Y = A2 + nf * KM * QM;               // [term][t_1][c_2]
    int64_t ii[3];
    a.g.row(r, ii[0], ii[1], ii[2]);
    int ni[2] = {1, 1}, nq[2] = {1, 1};
    int64_t jl[2] = {0, 0}, ql[2] = {0, 0};
    for (int l = 0; l < D; ++l) {
        ni[l] = a.v[l].jlen[ii[l]];
        nq[l] = a.v[l].qlen[ii[l]];
        jl[l] = a.v[l].jlo[ii[l]];
        ql[l] = a.v[l].qlo[ii[l]];
    }
    // univariate factors of both directions (direction 2 trivial when d = 1)
    for (int l = 0; l < 2; ++l) {
        double *A = l == 0 ? A1 : A2;
        const int n = nf * ni[l] * nq[l];
        for (int x = lane; x < n; x += 32) {
            const int f = x / (ni[l] * nq[l]), t = (x / nq[l]) % ni[l], c = x % nq[l];
            double w;
            if (l >= D) {
                w = f == 0 ? 1.0 : 0.0;
            } else {
                const DirView &v = a.v[l];
                const int64_t q = ql[l] + c, j = jl[l] + t;
                const int loc = (int)(j - v.span[q]);
                const int b = f >> 1;
                const double B = (loc >= 0 && loc <= p) ? v.B[q * wq_bstride(p) + 2 * loc + b] : 0.0;
                w = v.W[(ii[l] * v.maxq + c) * 4 + f] * B;
            }
            A[(f * KM + t) * QM + c] = w;
        }
    }
    __syncwarp();
    // coefficient point (q_1, q_2): the slab direction is counted from cq_b
    const int64_t o1 = D == 1 ? a.cq_b : 0, o2 = D == 2 ? a.cq_b : 0;
    // stage 1
    const int n1 = nterm * ni[0] * nq[1];
    for (int x = lane; x < n1; x += 32) {
        const int term = x / (ni[0] * nq[1]), t1 = (x / nq[1]) % ni[0], c2 = x % nq[1];
        const int lt = term / D, mt = term % D;
        const int f1 = a.matrix == 0 ? 0 : (lt == 0) + 2 * (mt == 0);
        const int comp = a.matrix == 0 ? a.comp_mass : (D == 1 ? 0 : lt + mt);  // C_00, C_01, C_11
        const double *Cc = a.cv.ptr(comp, ql[0] - o1, ql[1] + c2 - o2, 0);
        const double *Ar = A1 + (f1 * KM + t1) * QM;
        double s = 0.0;
        for (int c1 = 0; c1 < nq[0]; ++c1) s = fma(Ar[c1], __ldg(Cc + c1 * a.cv.s1), s);
        Y[(term * KM + t1) * QM + c2] = s;
    }
    __syncwarp();
    // stage 2 and the row's CSR segment (column (t_1, t_2) at t_1 + #I_1 t_2)
    const int64_t off = a.g.offset(ii[0], ii[1], ii[2]) - a.val_base;
    const int cnt = ni[0] * ni[1];
    for (int x = lane; x < cnt; x += 32) {
        const int t1 = x % ni[0], t2 = x / ni[0];
        double s = 0.0;
        for (int term = 0; term < nterm; ++term) {
            const int lt = term / D, mt = term % D;
            const int f2 = a.matrix == 0 || D == 1 ? 0 : (lt == 1) + 2 * (mt == 1);
            const double *Ar = A2 + (f2 * KM + t2) * QM;
            const double *Yr = Y + (term * KM + t1) * QM;
            for (int c2 = 0; c2 < nq[1]; ++c2) s = fma(Ar[c2], Yr[c2], s);
        }
        a.val[off + x] = s;
        if (a.col) a.col[off + x] = (int32_t)((jl[0] + t1) + a.g.n[0] * (jl[1] + t2));
    }
}


struct Sf2lArgs {
    RowGeo g;
    DirView v[2];
    int p, matrix;
    CoefView cv;
    int64_t cq_b;
    int comp_mass;
    double *val;
    int32_t *col;
    int64_t val_base;
    int64_t i2b, i2e;        // rows i_2 of this launch (global)
    int rc, rb;              // rows i_2 per CTA, stage-2 warps
    int km, qm, qrm;         // strides: max #I, max #Q (odd), max points of a chunk in q_2 (odd)
};

// sum_{c < N} a[c] b[c] with N a compile-time bound (rows padded with zeros beyond their #Q)
template <int N>
__device__ __forceinline__ double dotn(const double *x, const double *y) {
    double s0 = 0.0, s1 = 0.0;
    #pragma unroll
    for (int c = 0; c + 1 < N; c += 2) {
        s0 = fma(x[c], y[c], s0);
        s1 = fma(x[c + 1], y[c + 1], s1);
    }
    if (N & 1) s0 = fma(x[N - 1], y[N - 1], s0);
    return s0 + s1;
}


// Stage 2 of one row for lane (g, t_1): acc[k] += sum_{c < N} A2[f][g + G k][c] y[c] with the lane's
// Y row y (registers) reused across its KT/G trial rows t_2; A2 rows are read as 16-B pairs
// (the same address for the lanes of a group: broadcasts)
template <int N, int G, int NT2, int QA>
__device__ __forceinline__ void sf2_rows(const double *__restrict__ A2f, const double *__restrict__ Yr, int g,
                                         double (&acc)[NT2]) {
    double y[N];
    #pragma unroll
    for (int c = 0; c < N; ++c) y[c] = Yr[c];
    #pragma unroll
    for (int k = 0; k < NT2; ++k) {
        const double2 *ar = (const double2 *)(A2f + (g + G * k) * QA);
        double s0 = 0.0, s1 = 0.0;
        #pragma unroll
        for (int c = 0; c + 1 < N; c += 2) {
            const double2 v = ar[c / 2];
            s0 = fma(v.x, y[c], s0);
            s1 = fma(v.y, y[c + 1], s1);
        }
        if (N & 1) s0 = fma(A2f[(g + G * k) * QA + N - 1], y[N - 1], s0);
        acc[k] += s0 + s1;
    }
}

// Shared-memory layout (doubles), strides compile-time from the degree: QS = (3p+1)|1 point slots
// per row (#Q_i <= 3p+1 when n_EL >= p+2), zero padded beyond the row's #Q:
//   A1 [f][t_1][QS], Cs [u][r][QS] (r < QR, the chunk's points in q_2), Y [term][t_1][QY]
//   (QY = (QR + QS) | 1, zero beyond the chunk), A2 [row of batch][f][t_2][QS], per-row scalars.
template <int P, bool MASS>
__global__ void __launch_bounds__(256) k_sf2l(Sf2lArgs a) {
    extern __shared__ __align__(16) double sm[];
    constexpr int KM = 2 * P + 1, QX = 3 * P + 1, QS = QX | 1, BS = wq_bstride(P);
    constexpr int NF = MASS ? 1 : 4, NT = NF, NCU = MASS ? 1 : 3;
    // stage-2 lane map (g, t_1): G groups of KM lanes, each group NT2 trial rows t_2 = g + G k
    // (rows KM .. KT-1 of A2 are zero); A2 rows padded to an even length QA (16-B pairs)
    constexpr int G = 32 / KM, NT2 = (KM + G - 1) / G, KT = G * NT2, QA = QS + 1;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int QR = a.qrm, QY = (QR + QS) | 1;  // odd: the lanes of stage 2 (consecutive t_1) hit distinct banks
    const DirView &v0 = a.v[0], &v1 = a.v[1];
    const int64_t i1 = blockIdx.y;
    const int64_t i2a = a.i2b + (int64_t)blockIdx.x * a.rc;
    const int64_t i2e = i2a + a.rc < a.i2e ? i2a + a.rc : a.i2e;
    const int ni1 = v0.jlen[i1], nq1 = v0.qlen[i1];
    const int64_t jl1 = v0.jlo[i1], ql1 = v0.qlo[i1];
    const int64_t q2a = v1.qlo[i2a];
    const int nr2 = (int)(v1.qlo[i2e - 1] + v1.qlen[i2e - 1] - q2a);  // points of the chunk in q_2
    double *A1 = sm;
    double *Cs = A1 + NF * KM * QS;
    double *Y = Cs + NCU * QR * QS;
    // per stage-2 warp: [f][t_2 < KT][QA], 16-B aligned
    double *A2 = sm + ((NF * KM * QS + NCU * QR * QS + NT * KM * QY + 1) & ~1);
    // the chunk's coefficient values, zero padded beyond #Q_1: asynchronous 8-B copies (cp.async),
    // in flight while the A1 table is built
    #pragma unroll
    for (int u = 0; u < NCU; ++u)
        for (int x = tid; x < QR * QS; x += nth) {
            const int r = x / QS, c = x - r * QS;
            double *dst = Cs + u * QR * QS + x;
            if (r < nr2 && c < nq1)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                             "l"(a.cv.ptr(MASS ? a.comp_mass : u, ql1 + c, q2a + r - a.cq_b, 0))
                             : "memory");
            else
                *dst = 0.0;
        }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // A1: thread = point slot c of direction 1
    for (int c = tid; c < QS; c += nth) {
        double w[4] = {0.0, 0.0, 0.0, 0.0}, bv[2 * (P + 1)];
        int sp = 0;
        if (c < nq1) {
            const int64_t q = ql1 + c;
            sp = v0.span[q];
            #pragma unroll
            for (int f = 0; f < NF; ++f) w[f] = v0.W[(i1 * v0.maxq + c) * 4 + f];
            #pragma unroll
            for (int k = 0; k < 2 * (P + 1); ++k) bv[k] = v0.B[q * BS + k];
        }
        #pragma unroll
        for (int t = 0; t < KM; ++t) {
            const int loc = (int)(jl1 + t - sp);
            #pragma unroll
            for (int f = 0; f < NF; ++f) {
                double x = 0.0;
                #pragma unroll
                for (int k = 0; k <= P; ++k)
                    if (loc == k) x = bv[2 * k + (f >> 1)];
                A1[(f * KM + t) * QS + c] = c < nq1 && t < ni1 ? w[f] * x : 0.0;
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // stage 1: item (term, t_1, r); term (l, m) = (term >> 1, term & 1): family of direction 1
    // (l == 0) + 2 (m == 0), component C_{l+m} (C_01 = C_10)
    for (int x = tid; x < KM * QY; x += nth) {
        const int t1 = x / QY, r = x - t1 * QY;
        #pragma unroll
        for (int term = 0; term < NT; ++term) {
            const int lt = term >> 1, mt = term & 1;
            const int f1 = MASS ? 0 : (lt == 0) + 2 * (mt == 0);
            const int u = MASS ? 0 : lt + mt;
            double s = 0.0;
            if (r < nr2) s = nq1 == 2 * P + 1 ? dotn<2 * P + 1>(A1 + (f1 * KM + t1) * QS, Cs + (u * QR + r) * QS)
                                              : dotn<QX>(A1 + (f1 * KM + t1) * QS, Cs + (u * QR + r) * QS);
            Y[(term * KM + t1) * QY + r] = s;
        }
    }
    __syncthreads();
    // stage 2: warp w < a.rb takes the rows i2a + w, i2a + w + rb, ...: its own A2 (no CTA barrier)
    const int warp = tid >> 5, lane = tid & 31;
    if (warp >= a.rb) return;
    double *A2w = A2 + warp * (NF * KT * QA);
    for (int64_t i2 = i2a + warp; i2 < i2e; i2 += a.rb) {
        const int ni2 = v1.jlen[i2], nq2 = v1.qlen[i2];
        const int64_t jl2 = v1.jlo[i2], ql2 = v1.qlo[i2];
        const int r0 = (int)(ql2 - q2a);
        // A2 column of point slot c = lane: zeros, then the p+1 nonzero functions t_2 = span - jlo + k
        if (lane < QS) {
            #pragma unroll
            for (int f = 0; f < NF; ++f)
                #pragma unroll
                for (int t = 0; t < KT; ++t) A2w[(f * KT + t) * QA + lane] = 0.0;
            if (lane < nq2) {
                const int64_t q = ql2 + lane;
                const int t0 = (int)(v1.span[q] - jl2);
                double w[4];
                #pragma unroll
                for (int f = 0; f < NF; ++f) w[f] = v1.W[(i2 * v1.maxq + lane) * 4 + f];
                #pragma unroll
                for (int k = 0; k <= P; ++k) {
                    const int t = t0 + k;
                    if (t >= 0 && t < ni2) {
                        const double b0 = v1.B[q * BS + 2 * k], b1 = v1.B[q * BS + 2 * k + 1];
                        #pragma unroll
                        for (int f = 0; f < NF; ++f) A2w[(f * KT + t) * QA + lane] = w[f] * ((f >> 1) ? b1 : b0);
                    }
                }
            }
        }
        __syncwarp();
        const int64_t off = a.g.offset(i1, i2, 0) - a.val_base;
        if constexpr (P <= 8) {
            // lane (g, t_1) forms the entries (t_1, g + G k): its Y row stays in registers across them
            const int g = lane / KM, t1 = lane - g * KM;
            if (g < G) {
                double acc[NT2];
                #pragma unroll
                for (int k = 0; k < NT2; ++k) acc[k] = 0.0;
                #pragma unroll
                for (int term = 0; term < NT; ++term) {
                    const int lt = term >> 1, mt = term & 1;
                    const int f2 = MASS ? 0 : (lt == 1) + 2 * (mt == 1);
                    const double *A2f = A2w + f2 * KT * QA, *Yr = Y + (term * KM + t1) * QY + r0;
                    if (nq2 == 2 * P + 1) sf2_rows<2 * P + 1, G, NT2, QA>(A2f, Yr, g, acc);
                    else sf2_rows<QX, G, NT2, QA>(A2f, Yr, g, acc);
                }
                if (t1 < ni1) {
                    #pragma unroll
                    for (int k = 0; k < NT2; ++k) {
                        const int t2 = g + G * k;
                        if (t2 < ni2) {
                            const int64_t o = off + t1 + ni1 * t2;
                            a.val[o] = acc[k];
                            if (a.col) a.col[o] = (int32_t)((jl1 + t1) + a.g.n[0] * (jl2 + t2));
                        }
                    }
                }
            }
        } else {
            // p >= 9: one entry per lane and pass (the register-blocked form spills here: measured
            // 2D 1000^2 p = 10 mass 7.6 ms against 13.2)
            for (int e = lane; e < KM * KM; e += 32) {
                const int t2 = e / KM, t1 = e - t2 * KM;
                if (t1 >= ni1 || t2 >= ni2) continue;
                double s = 0.0;
                #pragma unroll
                for (int term = 0; term < NT; ++term) {
                    const int lt = term >> 1, mt = term & 1;
                    const int f2 = MASS ? 0 : (lt == 1) + 2 * (mt == 1);
                    const double *Ar = A2w + (f2 * KT + t2) * QA, *Yr = Y + (term * KM + t1) * QY + r0;
                    s += nq2 == 2 * P + 1 ? dotn<2 * P + 1>(Ar, Yr) : dotn<QX>(Ar, Yr);
                }
                const int64_t o = off + t1 + ni1 * t2;
                a.val[o] = s;
                if (a.col) a.col[o] = (int32_t)((jl1 + t1) + a.g.n[0] * (jl2 + t2));
            }
        }
        __syncwarp();
    }
}

}  // namespace

// doubles of shared memory per warp; 0 when d > 2
static int64_t sf2_wstride(const wq_plan_s *P, int matrix, int &km, int &qm) {
    km = 2 * P->p + 1;
    qm = 1;
    for (int l = 0; l < P->d; ++l) qm = P->dir[l].maxq > qm ? P->dir[l].maxq : qm;
    const int nf = matrix == 0 ? 1 : 4, nterm = matrix == 0 ? 1 : P->d * P->d;
    return P->d > 2 ? 0 : ((int64_t)(2 * nf + nterm) * km * qm + 1) / 2 * 2;
}

// d = 2 chunked-line kernel: rows i_2 per CTA (rc), stage-2 batch (rb) and strides; false if it does
// not fit in shared memory
static bool sf2l_config(const wq_plan_s *P, int matrix, Sf2lArgs &a, size_t &smem) {
    if (P->d != 2 || P->p < 1 || P->p > 10) return false;
    const int p = P->p, KM = 2 * p + 1, QS = (3 * p + 1) | 1;
    // compile-time point slots: #Q_i <= 3p+1 (not so when one support holds both boundary spans)
    if (P->dir[0].maxq > 3 * p + 1 || P->dir[1].maxq > 3 * p + 1) return false;
    const bool stiff = matrix != 0;
    const int nf = stiff ? 4 : 1, nterm = stiff ? 4 : 1, ncu = stiff ? 3 : 1;
    const int64_t E1 = P->dir[1].E;
    // rc rows i_2 per CTA and rb stage-2 warps (each with its own A2): 8 warps and the largest
    // rc >= 8 that leave 3 CTAs per SM, else 2, else 1 (fewer warps before fewer rows)
    const int G = 32 / KM, KT = G * ((KM + G - 1) / G);
    const size_t a2 = (size_t)nf * KT * (QS + 1);
    int64_t qrs[4];  // rc = 32, 16, 8, 4: max points in q_2 of a chunk, odd
    for (int k = 0; k < 4; ++k) {
        const int rc = 32 >> k;
        int64_t qr = 1;
        // any chunk start (launches over plane sub-ranges start anywhere in the slab)
        for (int64_t ia = P->slab_b; ia < P->slab_e; ++ia) {
            const int64_t ie = ia + rc < P->slab_e ? ia + rc : P->slab_e;
            const int64_t w = wq_host_qhi(ie - 1, E1, p) - wq_host_qlo(ia, E1, p) + 1;
            qr = w > qr ? w : qr;
        }
        qrs[k] = qr | 1;
    }
    for (size_t budget : {(size_t)72 * 1024, (size_t)110 * 1024, (size_t)200 * 1024})
        for (int rb = 8; rb >= 1; rb >>= 1)
            for (int k = 0; k < 4; ++k) {
                const int rc = 32 >> k;
                if (budget < 200 * 1024 && (rc < 8 || rb < 8)) break;
                const int64_t qr = qrs[k];
                const size_t n = (((size_t)nf * KM * QS + (size_t)ncu * qr * QS + (size_t)nterm * KM * ((qr + QS) | 1) + 1) &
                                  ~(size_t)1) + (size_t)rb * a2;
                const size_t bytes = n * sizeof(double);
                if (bytes <= budget) {
                    a.rc = rc;
                    a.rb = rb;
                    a.km = KM;
                    a.qm = QS;
                    a.qrm = (int)qr;
                    smem = bytes;
                    return true;
                }
            }
    return false;
}

template <int PP>
static wq_status launch_sf2l_p(const Sf2lArgs &a, size_t sm, int matrix, dim3 g, cudaStream_t s) {
    const void *fn = matrix == 0 ? (const void *)k_sf2l<PP, true> : (const void *)k_sf2l<PP, false>;
    cudaError_t ce = wq_smem_attr(fn, sm);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "sf2 kernel attribute");
    if (matrix == 0) k_sf2l<PP, true><<<g, 256, sm, s>>>(a);
    else k_sf2l<PP, false><<<g, 256, sm, s>>>(a);
    return WQ_OK;
}

bool sf2_supported(const wq_plan_s *P, int matrix) {
    Sf2lArgs l;
    size_t sl;
    if (sf2l_config(P, matrix, l, sl)) return true;
    int km, qm;
    const int64_t w = sf2_wstride(P, matrix, km, qm);
    return w > 0 && w * (int64_t)sizeof(double) <= 200 * 1024;
}

static wq_status launch_sf2l(wq_plan_s *P, Sf2lArgs &a, size_t sm, int matrix, double *val, int32_t *col,
                             int64_t plane_lo, int64_t plane_hi, int64_t val_base, cudaStream_t s) {
    a.g.init(P);
    a.i2b = P->slab_b + plane_lo;
    a.i2e = P->slab_b + plane_hi;
    for (int l = 0; l < 2; ++l) a.v[l] = P->dir[l];
    a.p = P->p;
    a.matrix = matrix;
    a.cv = P->cview;
    a.cq_b = P->cq_b;
    a.comp_mass = P->comp_mass;
    a.val = val;
    a.col = col;
    a.val_base = val_base;
    const int64_t nchunk = (plane_hi - plane_lo + a.rc - 1) / a.rc;
    if (nchunk > 0) {
        const dim3 g((unsigned)nchunk, (unsigned)P->dir[0].n);
        wq_status st = WQ_OK;
        switch (P->p) {
        case 1: st = launch_sf2l_p<1>(a, sm, matrix, g, s); break;
        case 2: st = launch_sf2l_p<2>(a, sm, matrix, g, s); break;
        case 3: st = launch_sf2l_p<3>(a, sm, matrix, g, s); break;
        case 4: st = launch_sf2l_p<4>(a, sm, matrix, g, s); break;
        case 5: st = launch_sf2l_p<5>(a, sm, matrix, g, s); break;
        case 6: st = launch_sf2l_p<6>(a, sm, matrix, g, s); break;
        case 7: st = launch_sf2l_p<7>(a, sm, matrix, g, s); break;
        case 8: st = launch_sf2l_p<8>(a, sm, matrix, g, s); break;
        case 9: st = launch_sf2l_p<9>(a, sm, matrix, g, s); break;
        case 10: st = launch_sf2l_p<10>(a, sm, matrix, g, s); break;
        }
        if (st) return st;
        wq_count_launches(1);
    }
    return wq_cuda_status(cudaGetLastError(), "sf2 (d = 2 line) assembly kernel");
}
wq_status launch_assemble_sf2(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                              int64_t plane_hi, int64_t val_base, cudaStream_t s) {
    {
        Sf2lArgs l;
        size_t sl;
        if (!getenv("WQ_SF2_ROWS") && sf2l_config(P, matrix, l, sl))
            return launch_sf2l(P, l, sl, matrix, val, col, plane_lo, plane_hi, val_base, s);
    }
    Sf2Args a;
    const int64_t ws = sf2_wstride(P, matrix, a.km, a.qm);
    int64_t rpp = 1;
    for (int l = 0; l < P->d - 1; ++l) rpp *= P->dir[l].n;
    a.g.init(P);
    for (int l = 0; l < 2; ++l) a.v[l] = P->dir[l];
    a.d = P->d;
    a.p = P->p;
    a.matrix = matrix;
    a.cv = P->cview;
    a.cq_b = P->cq_b;
    a.comp_mass = P->comp_mass;
    a.val = val;
    a.col = col;
    a.row_lo = plane_lo * rpp;
    a.rows = (plane_hi - plane_lo) * rpp;
    a.val_base = val_base;
    a.wstride = (int)ws;
    // warps (rows) per CTA: up to 8 within 200 KB of shared memory
    int wpc = 8;
    while (wpc > 1 && (int64_t)wpc * ws * (int64_t)sizeof(double) > 200 * 1024) wpc >>= 1;
    const size_t sm = (size_t)wpc * ws * sizeof(double);
    cudaError_t ce = wq_smem_attr((const void *)k_sf2, sm);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "sf2 kernel attribute");
    if (a.rows > 0) {
        k_sf2<<<(unsigned)((a.rows + wpc - 1) / wpc), 32 * wpc, sm, s>>>(a);
        wq_count_launches(1);
    }
    return wq_cuda_status(cudaGetLastError(), "sf2 assembly kernel");
}
