// wq_assemble_sf2.cu -- step 7 for d <= 2 (WQ_KERNEL_SF2): the row loop of
// Alg. 3 with the sum factorisation of Eq. sumfactorization
// (P:837), one warp per row.  For a 2D row i = (i_1, i_2):
//   stage 1 (contract q_1):  Y_{lm}(t_1, c_2) = sum_{c_1} A_1^{f_1}(t_1, c_1) C_{lm}(q_1, q_2)
//   stage 2 (contract q_2):  s_ij = sum_{lm} sum_{c_2} A_2^{f_2}(t_2, c_2) Y_{lm}(t_1, c_2)
// with A_k^f(t, c) = w^f_{k,i_k,q} D^{b(f)} B_{j_k}(x_q) (family f = a + 2b,
// (a,b) = (delta_kl, delta_km), reading R3; mass: the single term f = 0 and c).
// O(#I_1 #Q_1 #Q_2 + #I_1 #I_2 #Q_2) per row, i.e. O(p) per entry instead of
// the O(p^d) of the direct kernel.  d = 1 is the same code with a trivial
// direction 2 (#Q_2 = #I_2 = 1, A_2 = 1).
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

}  // namespace

// doubles of shared memory per warp; 0 when d > 2
static int64_t sf2_wstride(const wq_plan_s *P, int matrix, int &km, int &qm) {
    km = 2 * P->p + 1;
    qm = 1;
    for (int l = 0; l < P->d; ++l) qm = P->dir[l].maxq > qm ? P->dir[l].maxq : qm;
    const int nf = matrix == 0 ? 1 : 4, nterm = matrix == 0 ? 1 : P->d * P->d;
    return P->d > 2 ? 0 : ((int64_t)(2 * nf + nterm) * km * qm + 1) / 2 * 2;
}

bool sf2_supported(const wq_plan_s *P, int matrix) {
    int km, qm;
    const int64_t w = sf2_wstride(P, matrix, km, qm);
    return w > 0 && w * (int64_t)sizeof(double) <= 200 * 1024;
}

wq_status launch_assemble_sf2(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                              int64_t plane_hi, int64_t val_base, cudaStream_t s) {
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
