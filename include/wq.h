/*
 * wq.h -- C-ABI of libwq: B200-native (sm_100a) weighted-quadrature (WQ)
 * formation of the isogeometric Galerkin mass and stiffness matrices,
 * Calabro, Sangalli, Tani, "Fast formation of isogeometric Galerkin matrices
 * by weighted quadrature", arXiv:1605.01238.  "P:<n>" cites a line of the
 * paper text; DESIGN.md lists the readings R1..R15 referred to.
 *
 * Problem statement: a single-patch d-variate
 * (d = 1,2,3) tensor-product spline space of degree p and maximal regularity
 * C^{p-1} on open knot vectors Xi_l, and an isoparametric geometry map
 * F(zeta) = sum_i C_i B_i(zeta).  The library forms the N_DOF x N_DOF matrices
 *   M~ (mass,      Eq. mass2 P:505-507 evaluated by Eq. massquadrature)
 *   S~ (stiffness, Eq. stiff P:518-524 with Eq. coef_stiff P:527-529 evaluated
 *       by the stiffness analogue of Eq. massquadrature, reading R3)
 * by the row loop of Alg. 3 and writes them as CSR.
 *
 * Conventions (all calls):
 *  - Indices are 0-based.  Multi-indices are linearised with i_1 fastest
 *    (P:487-491); columns of a row are ascending.
 *  - row_ptr is int64 (nnz exceeds 2^31 at the BASELINE sizes); columns are
 *    int32 global indices (N_DOF < 2^31 is checked at plan creation).
 *  - Device pointers are CUDA global-memory pointers on the plan's device;
 *    host pointers are ordinary (preferably pinned) host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Stream-ordered calls never synchronise.
 *  - Errors: every call returns a wq_status; wq_last_error() gives a
 *    thread-local human-readable detail of the last failure.  Input
 *    validation happens in wq_plan_create; numerical failures detected on
 *    the device (singular weight system, folded geometry) are reported by
 *    wq_check.  WQ_ECUDA reports a CUDA launch/runtime error.
 *  - Ownership: the caller owns every buffer it passes; the plan copies the
 *    knot vectors and owns its device workspaces until wq_plan_destroy.
 *  - Threads: one plan must not be used by two host threads at once;
 *    distinct plans are independent.
 */
#ifndef WQ_H
#define WQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    WQ_OK = 0,
    WQ_EINVAL = 1,     /* bad argument: d, p, sizes, slab, null pointer        */
    WQ_EKNOTS = 2,     /* knot vector not open / repeated interior knot /
                          non-monotone / p < 1                     */
    WQ_ESINGULAR = 3,  /* a WQ exactness system (Eq. exact) has no
                          solution to 1e-13 backward-relative residual, or
                          #Q_i < #I_i (Eq. numb_nodes)               */
    WQ_EGEOMETRY = 4,  /* det J = 0 or changes sign on the point grid (R7)     */
    WQ_ENOMEM = 5,     /* device allocation failed                             */
    WQ_ECUDA = 6,      /* CUDA error (launch / runtime)                        */
    WQ_ERANGE = 7      /* index range: N_DOF >= 2^31, dir out of range         */
} wq_status;

typedef enum { WQ_MASS = 0, WQ_STIFFNESS = 1 } wq_matrix;

/* Row-block kernel selection for wq_assemble (all give results within the
 * parity tolerance of the oracle).                     */
typedef enum {
    WQ_KERNEL_AUTO = 0,   /* fastest available for (d, p)                     */
    WQ_KERNEL_DIRECT = 1, /* per-entry direct nested sum (Eq. massquadrature) */
    WQ_KERNEL_TILE = 2,   /* sum-factorised row-tile kernel (Eq. sumfactorization
                             P:837, rows of a tile share the d..2 stages)      */
    WQ_KERNEL_WS = 3,     /* same arithmetic as TILE, warp-specialised
                             persistent pipeline (TMA coefficient stream,
                             stage-3/2 producer warps, stage-1 consumer warps) */
    WQ_KERNEL_LINE = 4,   /* lines interior in directions 2, 3 by the
                             warp-specialised line kernel (independent producer
                             warps, 2-point TMA tasks), the others by TILE    */
    WQ_KERNEL_ZLINE = 5   /* stiffness, d = 3, p <= 4: lines along direction 3
                             (rows share the direction-1/2 mode products, the
                             direction-3 product per row) with direct coalesced
                             stores; needs the z coefficient layout (default
                             for such plans, see wq_plan_desc.coef_layout)    */
} wq_kernel;

typedef struct wq_plan_s *wq_plan;

typedef struct {
    int d;                        /* 1..3                                      */
    int p;                        /* degree, 1..WQ_MAX_DEGREE                  */
    const int64_t *n_knots;       /* [d] host; n_knots[l] = n_dof[l] + p + 1    */
    const double *const *knots;   /* [d] host FP64 knot vectors Xi_l*/
    int64_t slab_begin;           /* rows owned by this plan: planes           */
    int64_t slab_end;             /*   [slab_begin, slab_end) of the slowest
                                     index i_d; (0, -1) = all planes            */
    int need_mass;                /* allocate for WQ_MASS                       */
    int need_stiffness;           /* allocate for WQ_STIFFNESS                  */
    int device;                   /* CUDA device ordinal                        */
    int coef_layout;              /* 0: the library's choice (the stiffness
                                     components in the z layout when
                                     WQ_KERNEL_ZLINE applies; then the TILE /
                                     WS / LINE / DIRECT kernels are unavailable
                                     for WQ_STIFFNESS); 1: standard layout for
                                     every component (all kernels but ZLINE)  */
} wq_plan_desc;

#define WQ_MAX_DEGREE 10

typedef struct {
    int64_t n_dof_total;          /* N_DOF = prod_l n_dof[l]                    */
    int64_t nnz_total;            /* nnz of the whole matrix = prod_l ((2p+1)n_l - p(p+1)) */
    int64_t row_begin;            /* first global row owned by this plan        */
    int64_t n_rows_local;         /* rows owned                                 */
    int64_t nnz_local;            /* nnz of the owned rows                      */
    int64_t n_dof[3];             /* per direction (1 for l >= d)               */
    int64_t n_qp[3];              /* grid points per direction (Remark 1)       */
    int32_t max_q[3];             /* max_i #Q_{l,i}                             */
    int64_t coef_points;          /* points of the coefficient sub-grid held    */
    int64_t workspace_bytes;      /* device bytes owned by the plan             */
} wq_plan_info_t;

/* Validate the description (WQ_EKNOTS / WQ_EINVAL / WQ_ERANGE), copy the knot
 * vectors to the device, allocate the plan's device workspaces.  Launches no
 * kernels.  Synchronous.  *out is NULL on failure.                          */
wq_status wq_plan_create(const wq_plan_desc *desc, wq_plan *out);
wq_status wq_plan_destroy(wq_plan plan);
wq_status wq_plan_info(wq_plan plan, wq_plan_info_t *info);

/* Step 1-4 of the hot path (Alg. 1 lines 3-8, Alg. 2): point grid
 * and index ranges (Remark 1, reading R1), basis tables B^(0), B^(1),
 * exact integrals I^(a,b) (Eq. integrals) by (p+1)-point Gauss in
 * double-double, and the four min-norm weight families W^(a,b) (Alg. 2,
 * reading R4/R5) in double-double, rounded once to FP64.  Stream-ordered.
 * A failing exactness residual is latched and reported by wq_check.        */
wq_status wq_build_rules(wq_plan plan, void *stream);

/* Step 5 (Alg. 1 lines 12/15): the geometry coefficient field on
 * the plan's tensor sub-grid by sum-factorised evaluation of J = dF/dzeta:
 * c = |det J| (mass) and C = |det J| J^{-1} J^{-T} (stiffness, symmetric).
 * d_ctrl: device FP64 [N_DOF][d], row = linear control index (i_1 fastest).
 * Requires wq_build_rules on the same stream first.  A vanishing or
 * sign-changing det J is latched and reported by wq_check.                  */
wq_status wq_build_coef(wq_plan plan, const double *d_ctrl, void *stream);

/* Step 6: CSR pattern of the owned rows (bit-exact closed form).
 * d_row_ptr: device int64 [n_rows_local + 1], row_ptr[0] = nnz_base;
 * d_col: device int32 [nnz_local] or NULL (row_ptr only).
 * nnz_base = number of nonzeros in all rows before row_begin (multi-GPU).   */
wq_status wq_pattern(wq_plan plan, int64_t nnz_base, int64_t *d_row_ptr, int32_t *d_col, void *stream);

/* Step 7: values of the owned rows of M~ or S~ in CSR order.
 * d_val: device FP64 [nnz_local]; d_col_or_null: if non-NULL the column
 * indices are written in the same pass (fused pattern).
 * Requires wq_build_rules and wq_build_coef on the same stream first.       */
wq_status wq_assemble(wq_plan plan, wq_matrix matrix, double *d_val, int32_t *d_col_or_null, void *stream);
wq_status wq_assemble_ex(wq_plan plan, wq_matrix matrix, wq_kernel kernel, double *d_val,
                         int32_t *d_col_or_null, void *stream);

/* Synchronise `stream` and report latched device-side failures:
 * WQ_ESINGULAR (weights), WQ_EGEOMETRY (det J), or WQ_ECUDA.                */
wq_status wq_check(wq_plan plan, void *stream);

/* End to end with HOST buffers (the call a CPU-side user makes): copies
 * h_ctrl [N_DOF][d] to the device, runs steps 1-7 for `matrix`, and copies
 * the owned CSR block back to h_row_ptr [n_rows_local+1], h_col [nnz_local],
 * h_val [nnz_local] (pinned host memory recommended).  The value kernel is
 * run in row chunks whose device->host copies overlap the next chunk.
 * Synchronous; includes wq_check.                                           */
wq_status wq_form_host(wq_plan plan, wq_matrix matrix, const double *h_ctrl, int64_t nnz_base,
                       int64_t *h_row_ptr, int32_t *h_col, double *h_val, void *stream);

/* Test/inspection exports (synchronous device->host copies):
 * points [n_qp[dir]], qlo/qlen [n_dof[dir]] (Q_i = [qlo, qlo+qlen)),
 * w [n_dof[dir]][4][max_q[dir]] in family order (0,0),(1,0),(0,1),(1,1),
 * (a,b) = (test, trial) derivative order (reading R3), zero padded;
 * basis [n_qp[dir]][3][p+1]: values and derivatives of functions span..span+p
 * and degree p-1 values of functions span+1..span+p (last slot 0),
 * span [n_qp[dir]] (first nonzero function).  Any pointer may
 * be NULL.                                                                   */
wq_status wq_export_rules(wq_plan plan, int dir, double *h_points, int32_t *h_qlo, int32_t *h_qlen,
                          double *h_w, double *h_basis, int32_t *h_span);
/* Coefficient sub-grid [ncomp][q_d][...][q_1] (ncomp = d(d+1)/2 stiffness
 * components C_00, C_01, .. upper triangle row-major, then c if mass) and
 * its first q_d plane; h_out may be NULL to query the size.                  */
wq_status wq_export_coef(wq_plan plan, double *h_out, int64_t *n_values, int32_t *ncomp, int64_t *q_d_begin);

const char *wq_status_string(wq_status s);
const char *wq_last_error(void);
/* Library build identification, e.g. "libwq sm_100a <date>".                */
const char *wq_version(void);
/* Number of CUDA kernels this library has launched in this process (all
 * plans, all threads); used by benchmarks to report gpu_launches.            */
uint64_t wq_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* WQ_H */
