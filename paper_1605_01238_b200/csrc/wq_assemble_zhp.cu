// wq_assemble_zhp.cu -- host dispatch of the ZHP line kernel (wq_zhp.cuh) to the per-degree
// translation units wq_zhp_deg<p>.cu.
#include "wq_zhp.cuh"

bool zhp_supported(const wq_plan_s *P, int matrix) {
    if (P->d != 3 || P->p < 1 || P->p > 10 || !P->zh_dev) return false;
    if (matrix == WQ_MASS ? !P->need_mass : !P->need_stiff) return false;
    for (int l = 0; l < 3; ++l)
        if (P->dir[l].maxq > 3 * P->p + 1 || P->dir[l].n < 2) return false;  // a support holding both boundary spans
    switch (P->p) {
    case 1: return zhp_supported_deg_1(P, matrix);
    case 2: return zhp_supported_deg_2(P, matrix);
    case 3: return zhp_supported_deg_3(P, matrix);
    case 4: return zhp_supported_deg_4(P, matrix);
    case 5: return zhp_supported_deg_5(P, matrix);
    case 6: return zhp_supported_deg_6(P, matrix);
    case 7: return zhp_supported_deg_7(P, matrix);
    case 8: return zhp_supported_deg_8(P, matrix);
    case 9: return zhp_supported_deg_9(P, matrix);
    case 10: return zhp_supported_deg_10(P, matrix);
    }
    return false;
}

wq_status launch_assemble_zhp(wq_plan_s *P, int matrix, int64_t pl_lo, int64_t pl_hi, double *val, int32_t *col,
                              int64_t val_base, cudaStream_t s, int classes) {
    switch (P->p) {
    case 1: return zhp_launch_deg_1(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 2: return zhp_launch_deg_2(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 3: return zhp_launch_deg_3(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 4: return zhp_launch_deg_4(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 5: return zhp_launch_deg_5(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 6: return zhp_launch_deg_6(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 7: return zhp_launch_deg_7(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 8: return zhp_launch_deg_8(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 9: return zhp_launch_deg_9(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    case 10: return zhp_launch_deg_10(P, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);
    }
    wq_set_error("ZHP kernel: unsupported degree");
    return WQ_EINVAL;
}
