// wq_zline_deg5.cu -- instantiations of the z-line kernel for degree 5 (one translation unit
// per degree, so that the library build compiles the degrees in parallel).
#include "wq_zline.cuh"

wq_status zline_launch_deg_5(wq_plan_s *P, bool bnd, bool pu, bool cu, const int32_t *lines, int64_t n_lines,
                              int64_t pl_lo, int64_t pl_hi, double *val, int32_t *col, int64_t val_base,
                              const void *uni, cudaStream_t s) {
    const ZUni &un = *(const ZUni *)uni;
    (void)pu;
    if (bnd)
        return cu ? launch_zline_p<5, true, false, true>(P, lines, n_lines, pl_lo, pl_hi, val, col, val_base, un, s)
                  : launch_zline_p<5, true, false, false>(P, lines, n_lines, pl_lo, pl_hi, val, col, val_base, un, s);
    return cu ? launch_zline_p<5, false, false, true>(P, lines, n_lines, pl_lo, pl_hi, val, col, val_base, un, s)
              : launch_zline_p<5, false, false, false>(P, lines, n_lines, pl_lo, pl_hi, val, col, val_base, un, s);
}
