// wq_pattern.cu -- step 6: bit-exact CSR pattern.
//   row_ptr(i) = base + offset(i)   (closed form, wq_rows.cuh)
//   columns of row i: j = (jlo_1+t_1) + n_1((jlo_2+t_2) + n_2(jlo_3+t_3)),
//   t = t_1 + #I_1 (t_2 + #I_2 t_3), t_1 fastest -> ascending.
// One CTA per line of constant (i_2, i_3); the line's column segment is
// contiguous, so stores are fully coalesced (HBM-write bound, 4 B/nnz).
#include "wq_rows.cuh"

namespace {

__global__ void k_rowptr(RowGeo g, int64_t base, int64_t *rp, int64_t r_lo, int64_t r_hi, int64_t n_rows) {
    for (int64_t r = r_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= r_hi; r += (int64_t)gridDim.x * blockDim.x) {
        int64_t off;
        if (r == n_rows) {
            // one past the last row: offset of the first row of the next slab plane
            int64_t i1, i2, i3;
            g.row(r - 1, i1, i2, i3);
            off = g.offset(i1, i2, i3) + g.ni(0, i1) * g.ni(1, i2) * g.ni(2, i3);
        } else {
            int64_t i1, i2, i3;
            g.row(r, i1, i2, i3);
            off = g.offset(i1, i2, i3);
        }
        rp[r - r_lo] = base + off;
    }
}

__global__ void __launch_bounds__(256) k_cols(RowGeo g, int32_t *col, int64_t line_lo, int64_t col_base) {
    const int64_t k = line_lo + blockIdx.x;
    int64_t i1b, i2, i3;
    g.line(k, i1b, i2, i3);
    const int64_t n1 = g.n[0], n2 = g.n[1];
    const int64_t ni2 = g.ni(1, i2), ni3 = g.ni(2, i3);
    const int64_t jl2 = g.d > 1 ? g.jlo[1][i2] : 0, jl3 = g.d > 2 ? g.jlo[2][i3] : 0;
    const int64_t i1e = i1b + g.line_len;
    int64_t off = g.offset(i1b, i2, i3) - col_base;
    for (int64_t i1 = i1b; i1 < i1e; ++i1) {
        const int64_t ni1 = g.jlen[0][i1], jl1 = g.jlo[0][i1];
        const int64_t cnt = ni1 * ni2 * ni3;
        for (int64_t t = threadIdx.x; t < cnt; t += blockDim.x) {
            int64_t t1 = t % ni1, u = t / ni1, t2 = u % ni2, t3 = u / ni2;
            col[off + t] = (int32_t)((jl1 + t1) + n1 * ((jl2 + t2) + n2 * (jl3 + t3)));
        }
        off += cnt;
    }
}

}  // namespace

// rows [row_lo, row_hi] of row_ptr (row_hi may equal n_rows_local), and if
// col != NULL the columns of ALL owned rows.
wq_status launch_pattern(wq_plan_s *P, int64_t base, int64_t *rp, int32_t *col, int64_t row_lo, int64_t row_hi,
                         cudaStream_t s) {
    RowGeo g;
    g.init(P);
    if (rp) {
        int64_t cnt = row_hi - row_lo + 1;
        unsigned blocks = (unsigned)((cnt + 255) / 256);
        if (blocks > 148 * 16) blocks = 148 * 16;
        k_rowptr<<<blocks, 256, 0, s>>>(g, base, rp, row_lo, row_hi, P->n_rows_local);
        wq_count_launches(1);
    }
    if (col && g.n_lines > 0) {
        k_cols<<<(unsigned)g.n_lines, 256, 0, s>>>(g, col, 0, 0);
        wq_count_launches(1);
    }
    return wq_cuda_status(cudaGetLastError(), "pattern kernels");
}
