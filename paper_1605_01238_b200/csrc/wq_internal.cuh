// wq_internal.cuh -- plan layout and helpers shared by the libwq kernels.
// Product code (sm_100a).  Shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include "../../include/wq.h"

#define WQ_PMAX WQ_MAX_DEGREE          // compile-time bound on p
#define WQ_KMAX (2 * WQ_PMAX + 1)      // max #I_i
#define WQ_BROWS 3                     // rows of the per-point basis table
// doubles per point of the basis table, even so (value, derivative) pairs are 16-B aligned
__host__ __device__ constexpr int wq_bstride(int p) { return (WQ_BROWS * (p + 1) + 1) & ~1; }

// Device view of one parametric direction.  For l >= d the direction is a
// dummy of extent 1 (n = nq = 1, one point, weight 1, B = 1, B' = 0).
struct DirView {
    int64_t n;        // DOFs
    int64_t E;        // knot spans
    int64_t nq;       // grid points (Remark 1)
    int64_t nk;       // knots
    int32_t maxq;     // max #Q_i
    const double *knots;  // [nk]
    double *pts;          // [nq]
    int32_t *span;        // [nq] first nonzero function at the point (span index e)
    int32_t *qlo, *qlen;  // [n] Q_i = [qlo, qlo+qlen)
    int32_t *jlo, *jlen;  // [n] I_i = [jlo, jlo+jlen)
    int64_t *pref;        // [n+1] prefix sums of jlen
    double *B;            // [nq][wq_bstride(p)]: (value, first derivative) pairs of functions
                          // span..span+p, then degree p-1 values of span+1..span+p (last slot 0)
    double *W;            // [n][maxq][4] weights, family f = a + 2b fastest
};

struct Flags {   // device-side latched errors
    int weights_bad;   // first failing (dir,row,family) + 1, packed
    int det_pos;
    int det_neg;
    int det_zero;
};

struct wq_plan_s {
    int d, p, device;
    int need_mass, need_stiff;
    int64_t slab_b, slab_e;        // planes of i_d
    int64_t n_dof_total, nnz_total, row_begin, n_rows_local, nnz_local;
    int64_t L[3];                  // sum_i #I_{l,i}
    DirView dir[3];
    int dir_src[3];                // direction whose rules tables dir[l] shares (identical knots), or l
    // coefficient sub-grid: q_d in [cq_b, cq_e)
    int64_t cq_b, cq_e, coef_points;
    int64_t c0off;                 // d = 3: point q_1 is stored at column q_1 + 1 (c0off = 1), so that
                                   // the 2-point boxes [1 + 2k, 2 + 2k] of the row kernels start 16-B
                                   // aligned for TMA; else 0
    int64_t cld1;                  // leading dimension along q_1 (d = 3: nq_1 + 1 rounded up to even)
    int64_t cstride;               // doubles per component = cld1 * (points / nq_1)
    int ncomp_s, ncomp;            // stiffness components, total components
    int ncomp_std;                 // components held in coef (standard layout)
    double *coef;                  // [ncomp][cstride], point (q1, q2, q3) at q1 + c0off + cld1 * (q2 + nq2 * (q3 - cq_b))
    // Gauss-Legendre rule on [-1,1] in double-double: [p+1] (hi, lo) pairs
    double *gl;                    // [2*(p+1)] t, [2*(p+1)] w
    Flags *flags;                  // device
    void *arena;                   // one allocation for all small tables
    size_t arena_bytes;
    double *ctrl_dev;              // device control-net staging (wq_form_host)
    double *dnet;                  // z layout: derivative control nets [N_DOF][3][3] (k_dnet)
    size_t dnet_bytes;
    size_t ctrl_bytes;
    // form_host staging
    double *stage_val; int32_t *stage_col; int64_t *stage_rp; size_t stage_bytes;
    int64_t workspace_bytes;
    // d = 3 row lines (i2 + n2 * (i3 - slab_b)) split by the line kernel's applicability:
    // interior in directions 2 and 3 (#Q = 2p+1, no boundary span) first, then the rest.
    // Both sorted; device copy in lines_dev (interior at 0, boundary at n_lines_int).
    std::vector<int32_t> lines_int, lines_bnd;
    int32_t *lines_dev;
    // z-line kernel (d = 3 stiffness): the stiffness components live in the z layout
    // [comp][q_1][q_2][q_3 - cq_b] (q_3 fastest, row length zld even, zero padded) instead of coef;
    // coef then holds only the mass component.  Lines (i1 + n1 * i2) interior in directions 1 and 2
    // first, then the rest (device copy zlines_dev).
    int zlayout;
    double *coefz;
    int64_t zld, zcs;              // row length along q_3, doubles per component
    int comp_mass;                 // component index of c in coef
    std::vector<int32_t> zlines_uni, zlines_int, zlines_bnd;
    int32_t *zlines_dev;
    // uniform-mesh interior rules for the z-line kernel (fetched once per plan at the first
    // assembly): 0 not checked yet, 1 usable (zuni_buf holds them), -1 not uniform
    int32_t *zbounds_dev;          // cost-balanced chunks of the boundary lines for zbounds_n CTAs
    int64_t zbounds_n;
    int zuni_state;
    double zuni_buf[3 * 13 * 4 + 3 * 2 * 7 * 2];
};

// host helpers
int64_t wq_host_qlo(int64_t i, int64_t E, int p);  // first grid point of Q_i (Remark 1, reading R1)
void wq_count_launches(int n);  // adds n to the process-wide launch counter
void wq_set_error(const std::string &msg);
wq_status wq_cuda_status(cudaError_t e, const char *what);

// 1D counts (host and device)
__host__ __device__ inline int64_t wq_jlo(int64_t i, int p) { return i - p > 0 ? i - p : 0; }
__host__ __device__ inline int64_t wq_jhi(int64_t i, int p, int64_t n) { return i + p < n - 1 ? i + p : n - 1; }
__host__ __device__ inline int64_t wq_ni(int64_t i, int p, int64_t n) { return wq_jhi(i, p, n) - wq_jlo(i, p) + 1; }

// kernel launchers (defined in the .cu files)
wq_status launch_rules(wq_plan_s *P, cudaStream_t s);
wq_status launch_coef(wq_plan_s *P, const double *ctrl, cudaStream_t s);
wq_status launch_pattern(wq_plan_s *P, int64_t base, int64_t *rp, int32_t *col, int64_t row_lo,
                         int64_t row_hi, cudaStream_t s);
// value kernels over the slab planes [plane_lo, plane_hi) (relative to the
// plan's first plane); entries are written at (row offset - val_base).
wq_status launch_assemble_direct(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                                 int64_t plane_hi, int64_t val_base, cudaStream_t s);
wq_status launch_assemble_tile(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                               int64_t plane_hi, int64_t val_base, cudaStream_t s);
bool tile_supported(const wq_plan_s *P, int matrix);
wq_status launch_assemble_ws(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                             int64_t plane_hi, int64_t val_base, cudaStream_t s);
bool ws_supported(const wq_plan_s *P, int matrix);
// line kernel over a list of lines; bnd = lines touching a boundary span in direction 2 or 3
wq_status launch_assemble_line(wq_plan_s *P, int matrix, bool bnd, const int32_t *lines, int64_t n_lines,
                               double *val, int32_t *col, int64_t val_base, cudaStream_t s);
bool line_supported(const wq_plan_s *P, int matrix, bool bnd);
// z-line kernel (stiffness, d = 3, coefficients in the z layout) over a list of lines (i1 + n1 * i2)
// and the planes [pl_lo, pl_hi) of the slab
bool zline_supported_p(int d, int p, const int64_t *n, const int32_t *maxq, int64_t n2l, int64_t nq2l);
// cls: 0 lines with i1, i2 in [2p, n-1-2p] (uniform rules possible), 1 other lines interior in
// directions 1 and 2, 2 lines touching a boundary span
wq_status launch_assemble_zline(wq_plan_s *P, int cls, const int32_t *lines, int64_t n_lines, int64_t pl_lo,
                                int64_t pl_hi, double *val, int32_t *col, int64_t val_base, cudaStream_t s);
// tile kernel over an explicit list of lines of the plan's slab
wq_status launch_assemble_tile_list(wq_plan_s *P, int matrix, const int32_t *lines, int64_t n_lines, double *val,
                                    int32_t *col, int64_t val_base, cudaStream_t s);

