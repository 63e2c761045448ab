// wq_assemble_direct.cu -- step 7, direct kernel (WQ_KERNEL_DIRECT): every
// entry of row i is the nested WQ sum of Eq. massquadrature /
// its stiffness analogue (reading R3) over q in Q_i, evaluated
// directly (no sum factorisation).  O(#Q^d) per entry: used for d < 3, for
// small problems, and as an in-library cross-check of the tile kernel.
// One CTA per row; the row's univariate factors A^f_k[t][c] = w^f_{k,i_k,q} *
// D^{b(f)} B_{j_k}(x_q) are staged in shared memory.
#include "wq_rows.cuh"

namespace {

struct DirectArgs {
    RowGeo g;
    DirView v[3];
    int d, p, matrix;
    CoefView cv;             // coefficient field (any layout)
    int64_t cq_b;
    int comp_mass, ncomp_s;
    double *val;
    int32_t *col;
    int64_t row_lo;
    int64_t val_base;        // subtracted from row offsets (chunked launches)
    int qmax;                // max_i #Q_i over the directions
};

__device__ __forceinline__ int comp_index(int D, int l, int m) {
    if (l > m) { int t = l; l = m; m = t; }
    return l * D - l * (l - 1) / 2 + (m - l);
}

__global__ void __launch_bounds__(128) k_direct(DirectArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int p = a.p, P1 = p + 1, D = a.d;
    const int KM = 2 * p + 1, QM = a.qmax;
    const int64_t r = a.row_lo + blockIdx.x;
    int64_t ii[3];
    a.g.row(r, ii[0], ii[1], ii[2]);
    int ni[3] = {1, 1, 1}, nq[3] = {1, 1, 1};
    int64_t jl[3] = {0, 0, 0}, ql[3] = {0, 0, 0};
    for (int l = 0; l < D; ++l) {
        ni[l] = a.v[l].jlen[ii[l]];
        nq[l] = a.v[l].qlen[ii[l]];
        jl[l] = a.v[l].jlo[ii[l]];
        ql[l] = a.v[l].qlo[ii[l]];
    }
    const int nf = a.matrix == 0 ? 1 : 4;
    // A[l][f][t][c]
    double *A = sm;
    const int tid = threadIdx.x;
    for (int l = 0; l < 3; ++l)
        for (int x = tid; x < nf * KM * QM; x += blockDim.x) {
            int f = x / (KM * QM), t = (x / QM) % KM, c = x % QM;
            double val = 0.0;
            if (l >= D) {
                val = (t == 0 && c == 0 && f == 0) ? 1.0 : 0.0;
            } else if (t < ni[l] && c < nq[l]) {
                const DirView &v = a.v[l];
                int64_t q = ql[l] + c, j = jl[l] + t;
                int loc = (int)(j - v.span[q]);
                int b = f >> 1;
                double B = (loc >= 0 && loc <= p) ? v.B[q * wq_bstride(p) + 2 * loc + b] : 0.0;
                val = v.W[(ii[l] * v.maxq + c) * 4 + f] * B;
            }
            A[((l * nf + f) * KM + t) * QM + c] = val;
        }
    __syncthreads();
    const int64_t cnt = (int64_t)ni[0] * ni[1] * ni[2];
    const int64_t off = a.g.offset(ii[0], ii[1], ii[2]) - a.val_base;
    const int nterm = a.matrix == 0 ? 1 : D * D;
    for (int64_t t = tid; t < cnt; t += blockDim.x) {
        int t1 = (int)(t % ni[0]), t2 = (int)((t / ni[0]) % ni[1]), t3 = (int)(t / ((int64_t)ni[0] * ni[1]));
        double s = 0.0;
        for (int term = 0; term < nterm; ++term) {
            int lt = term / D, mt = term % D;
            int f[3];
            int comp;
            for (int k = 0; k < 3; ++k) f[k] = a.matrix == 0 || k >= D ? 0 : ((k == lt) + 2 * (k == mt));
            comp = a.matrix == 0 ? a.comp_mass : comp_index(D, lt, mt);
            const double *A1 = A + ((0 * nf + f[0]) * KM + t1) * QM;
            const double *A2 = A + ((1 * nf + f[1]) * KM + t2) * QM;
            const double *A3 = A + ((2 * nf + f[2]) * KM + t3) * QM;
            for (int c3 = 0; c3 < nq[2]; ++c3) {
                double s2 = 0.0;
                for (int c2 = 0; c2 < nq[1]; ++c2) {
                    double s1 = 0.0;
                    // local coordinate along the slab direction d (the view counts it from cq_b)
                    const double *Cc = D == 3 ? a.cv.ptr(comp, ql[0], ql[1] + c2, ql[2] + c3 - a.cq_b)
                                     : D == 2 ? a.cv.ptr(comp, ql[0], ql[1] + c2 - a.cq_b, 0)
                                              : a.cv.ptr(comp, ql[0] - a.cq_b, 0, 0);
                    for (int c1 = 0; c1 < nq[0]; ++c1) s1 = fma(A1[c1], __ldg(Cc + c1 * a.cv.s1), s1);
                    s2 = fma(A2[c2], s1, s2);
                }
                s = fma(A3[c3], s2, s);
            }
        }
        a.val[off + t] = s;
        if (a.col) {
            int64_t j = (jl[0] + t1) + a.g.n[0] * ((jl[1] + t2) + a.g.n[1] * (jl[2] + t3));
            a.col[off + t] = (int32_t)j;
        }
    }
}

}  // namespace

wq_status launch_assemble_direct(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                                 int64_t plane_hi, int64_t val_base, cudaStream_t s) {
    int64_t rpp = 1;
    for (int l = 0; l < P->d - 1; ++l) rpp *= P->dir[l].n;
    const int64_t row_lo = plane_lo * rpp, row_hi = plane_hi * rpp;
    DirectArgs a;
    a.g.init(P);
    for (int l = 0; l < 3; ++l) a.v[l] = P->dir[l];
    a.d = P->d;
    a.p = P->p;
    a.matrix = matrix;
    a.cv = P->cview;
    a.cq_b = P->cq_b;
    a.ncomp_s = P->ncomp_s;
    a.comp_mass = P->comp_mass;
    a.val = val;
    a.col = col;
    a.row_lo = row_lo;
    a.val_base = val_base;
    int p = P->p;
    int qmax = 1;
    for (int l = 0; l < P->d; ++l) qmax = P->dir[l].maxq > qmax ? P->dir[l].maxq : qmax;
    a.qmax = qmax;
    int KM = 2 * p + 1, QM = qmax;
    int nf = matrix == 0 ? 1 : 4;
    size_t sm = (size_t)3 * nf * KM * QM * sizeof(double);
    wq_smem_attr((const void *)k_direct, sm);
    int64_t rows = row_hi - row_lo;
    if (rows > 0) {
        k_direct<<<(unsigned)rows, 128, sm, s>>>(a);
        wq_count_launches(1);
    }
    return wq_cuda_status(cudaGetLastError(), "direct assembly kernel");
}
