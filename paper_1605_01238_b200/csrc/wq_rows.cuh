// wq_rows.cuh -- row bookkeeping shared by the pattern and row-block kernels:
// local row <-> multi-index, closed-form CSR offsets (the column
// set of row i is prod_l I_{l,i_l}, so nnz(i) = prod_l #I_{l,i_l} and the
// row offsets factor through the 1D prefix sums P_l(i) = sum_{i'<i} #I_{l,i'}).
#pragma once
#include "wq_internal.cuh"

struct RowGeo {
    int d, p;
    int64_t n[3];
    int64_t L[3];            // sum_i #I_{l,i}
    const int64_t *pref[3];  // [n_l + 1]
    const int32_t *jlo[3], *jlen[3];
    int64_t slab_b, slab_e;  // planes of i_d
    int64_t n_lines;         // lines of constant (i_2, i_3)
    int64_t line_len;        // rows per line (i_1 range)

    __host__ void init(const wq_plan_s *P) {
        d = P->d;
        p = P->p;
        for (int l = 0; l < 3; ++l) {
            n[l] = P->dir[l].n;
            L[l] = P->L[l];
            pref[l] = P->dir[l].pref;
            jlo[l] = P->dir[l].jlo;
            jlen[l] = P->dir[l].jlen;
        }
        slab_b = P->slab_b;
        slab_e = P->slab_e;
        if (d == 1) { n_lines = 1; line_len = slab_e - slab_b; }
        else if (d == 2) { n_lines = slab_e - slab_b; line_len = n[0]; }
        else { n_lines = n[1] * (slab_e - slab_b); line_len = n[0]; }
    }
    // line k -> (i1 start, i2, i3) in global indices
    __device__ __forceinline__ void line(int64_t k, int64_t &i1b, int64_t &i2, int64_t &i3) const {
        if (d == 1) { i1b = slab_b; i2 = 0; i3 = 0; }
        else if (d == 2) { i1b = 0; i2 = slab_b + k; i3 = 0; }
        else { i1b = 0; i2 = k % n[1]; i3 = slab_b + k / n[1]; }
    }
    __device__ __forceinline__ int64_t ni(int l, int64_t i) const { return l < d ? (int64_t)jlen[l][i] : 1; }
    // offset of row (i1, i2, i3) relative to the first owned row
    __device__ __forceinline__ int64_t offset(int64_t i1, int64_t i2, int64_t i3) const {
        if (d == 1) return pref[0][i1] - pref[0][slab_b];
        if (d == 2) return (pref[1][i2] - pref[1][slab_b]) * L[0] + ni(1, i2) * pref[0][i1];
        int64_t n3 = ni(2, i3);
        return (pref[2][i3] - pref[2][slab_b]) * L[1] * L[0] + n3 * pref[1][i2] * L[0] + n3 * ni(1, i2) * pref[0][i1];
    }
    // local row r -> global multi-index
    __device__ __forceinline__ void row(int64_t r, int64_t &i1, int64_t &i2, int64_t &i3) const {
        if (d == 1) { i1 = slab_b + r; i2 = 0; i3 = 0; }
        else if (d == 2) { i1 = r % n[0]; i2 = slab_b + r / n[0]; i3 = 0; }
        else { i1 = r % n[0]; int64_t t = r / n[0]; i2 = t % n[1]; i3 = slab_b + t / n[1]; }
    }
};
