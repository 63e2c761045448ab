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

// Coefficient field view: component k at grid point (q1, q2, q3) is
//   base[k * cs + q1 * s1 + q2 * s2 + (q_d - cq_b) * s_d]
// with the slab direction d counted from the plan's first point cq_b.
//   d = 3 (z layout): [comp][q_1][q_2][q_3 - cq_b], q_3 fastest, rows of zld (even) doubles,
//       so a task box of 2 consecutive q_3 x #Q_1 x #Q_2 points is one 4D TMA tile;
//   d = 2: [comp][q_2 - cq_b][q_1];  d = 1: [comp][q_1 - cq_b].
// Components: the d(d+1)/2 stiffness components C_lm (upper triangle, row major) first when the
// plan needs the stiffness matrix, then c (mass) when it needs the mass matrix.
struct CoefView {
    const double *base;
    int64_t cs, s1, s2, s3;
    __device__ __forceinline__ const double *ptr(int comp, int64_t q1, int64_t q2, int64_t q3l) const {
        return base + comp * cs + q1 * s1 + q2 * s2 + q3l * s3;
    }
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
    int ncomp_s, ncomp;            // stiffness components, total components
    int comp_mass;                 // component index of c
    double *coef;                  // [ncomp][cs] (layout: CoefView above)
    int64_t zld, zcs;              // d = 3: row length along q_3 (even), doubles per component
    int64_t nld1;                  // d <= 2: leading dimension (nq_1)
    CoefView cview;                // device view of coef
    double *coef_std;              // d = 3: copy of the field in the standard layout [comp][q_3][q_2][q_1]
    CoefView cview_std;            // (q_1 contiguous, coalesced fibre loads of the row-tile kernel), made
                                   // by launch_coef when AUTO runs the row-tile kernel for a matrix
    int has_coef;                  // a coefficient field has been built (create or wq_build_coef)
    // Gauss-Legendre rule on [-1,1] in double-double: [p+1] (hi, lo) pairs
    double *gl;                    // [2*(p+1)] t, [2*(p+1)] w
    Flags *flags;                  // device
    void *arena;                   // one allocation for all small tables
    size_t arena_bytes;
    double *ctrl_dev;              // device copies of the control net and coefficient nets (create,
    double *kappa_dev, *gamma_dev; // wq_form_host staging); kappa/gamma null = 1
    size_t ctrl_bytes;
    double *x2;                    // d = 3: coefficient-field workspace (k_cz12 -> k_cz3)
    size_t x2_bytes;
    double *dnet;                  // d = 3: derivative control nets (+ coefficient nets) of the slab's
    size_t dnet_bytes;             // control planes k_3 in [k3b, k3e): [k][NE] (k_dnet)
    int64_t k3b, k3e;
    // form_host staging
    double *stage_val; size_t stage_bytes;
    int64_t workspace_bytes;
    // z-line kernel (d = 3 stiffness, 2 <= p <= 6): lines (i1 + n1 * i2) with uniform rules
    // possible, other lines interior in directions 1 and 2, lines touching a boundary span (device
    // copy zlines_dev; zbounds_dev: cost-balanced CTA chunks of the boundary lines)
    int zline_ok;
    std::vector<int32_t> zlines_uni, zlines_int, zlines_bnd;
    int32_t *zlines_dev;
    int32_t *zbounds_dev;
    int64_t zbounds_n;
    // uniform-mesh interior rules (reading R16), fetched and verified once at plan creation:
    // 1 usable (zuni_buf holds them), -1 not uniform
    int zuni_state;
    double zuni_buf[3 * 21 * 4 + 3 * 2 * 11 * 2];
    // z-line: the interior and boundary launches run on two forked streams beside the uniform one
    // (event fork / join on the caller's stream; created on first use)
    cudaStream_t zfork[2] = {nullptr, nullptr};
    cudaEvent_t zev[3] = {nullptr, nullptr, nullptr};
    int kernel_auto[2];            // wq_kernel AUTO runs for [mass, stiffness]
    // z-line (ZHP) kernel lines (i1 + n1 * i2): interior in directions 1 and 2 first (#Q = 2p+1),
    // then the rest; device copy zh_dev
    std::vector<int32_t> zh_int, zh_bnd;
    int32_t *zh_dev;
};

// host helpers
int64_t wq_host_qlo(int64_t i, int64_t E, int p);  // first grid point of Q_i (Remark 1, reading R1)
int64_t wq_host_qhi(int64_t i, int64_t E, int p);  // last grid point of Q_i
void wq_count_launches(int n);  // adds n to the process-wide launch counter
// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the current device, set once per
// (function, device) pair
cudaError_t wq_smem_attr(const void *func, size_t bytes);
void wq_set_error(const std::string &msg);
wq_status wq_cuda_status(cudaError_t e, const char *what);

// 1D counts (host and device)
__host__ __device__ inline int64_t wq_jlo(int64_t i, int p) { return i - p > 0 ? i - p : 0; }
__host__ __device__ inline int64_t wq_jhi(int64_t i, int p, int64_t n) { return i + p < n - 1 ? i + p : n - 1; }
__host__ __device__ inline int64_t wq_ni(int64_t i, int p, int64_t n) { return wq_jhi(i, p, n) - wq_jlo(i, p) + 1; }

// kernel launchers (defined in the .cu files)
wq_status launch_rules(wq_plan_s *P, cudaStream_t s);
wq_status launch_pattern(wq_plan_s *P, int64_t base, int64_t *rp, int32_t *col, int64_t row_lo,
                         int64_t row_hi, cudaStream_t s);
// value kernels over the slab planes [plane_lo, plane_hi) (relative to the
// plan's first plane); entries are written at (row offset - val_base).
wq_status launch_assemble_direct(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                                 int64_t plane_hi, int64_t val_base, cudaStream_t s);
wq_status launch_assemble_tile(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                               int64_t plane_hi, int64_t val_base, cudaStream_t s);
bool tile_supported(const wq_plan_s *P, int matrix);
// d <= 2: sum-factorised rows, one warp per row
wq_status launch_assemble_sf2(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                              int64_t plane_hi, int64_t val_base, cudaStream_t s);
bool sf2_supported(const wq_plan_s *P, int matrix);
// z-line kernel (stiffness, d = 3, coefficients in the z layout) over a list of lines (i1 + n1 * i2)
// and the planes [pl_lo, pl_hi) of the slab
bool zline_supported_p(int d, int p, const int64_t *n, const int32_t *maxq, int64_t n2l, int64_t nq2l);
// cls: 0 lines with i1, i2 in [2p, n-1-2p] (uniform rules possible), 1 other lines interior in
// directions 1 and 2, 2 lines touching a boundary span
wq_status launch_assemble_zline(wq_plan_s *P, int cls, const int32_t *lines, int64_t n_lines, int64_t pl_lo,
                                int64_t pl_hi, double *val, int32_t *col, int64_t val_base, cudaStream_t s);
// z-line uniform tables + row-type check (reading R16), once per plan after the rules are built
// (synchronous device -> host copies; called from wq_plan_create only)
wq_status zline_prepare(wq_plan_s *P);
// high-degree / mass line kernel (d = 3, any p)
bool zhp_supported(const wq_plan_s *P, int matrix);
wq_status launch_assemble_zhp(wq_plan_s *P, int matrix, int64_t pl_lo, int64_t pl_hi, double *val, int32_t *col,
                              int64_t val_base, cudaStream_t s, int classes = 3);
// standard element-loop Gauss quadrature (SGQ), scatter-added into the CSR values
wq_status launch_assemble_sgq(wq_plan_s *P, int matrix, const double *ctrl, const double *kappa, const double *gamma,
                              double *val, int32_t *col, cudaStream_t s);
wq_status launch_coef(wq_plan_s *P, const double *ctrl, const double *kappa, const double *gamma, cudaStream_t s);
