/*
 * wq.h -- C-ABI of libwq: B200-native (sm_100a) weighted-quadrature (WQ)
 * formation of the isogeometric Galerkin mass and stiffness matrices,
 * Calabro, Sangalli, Tani, "Fast formation of isogeometric Galerkin matrices
 * by weighted quadrature", arXiv:1605.01238.  "P:<n>" cites a line of the
 * paper text; DESIGN.md lists the readings R1..R17 referred to.
 *
 * Problem statement: a single-patch d-variate
 * (d = 1,2,3) tensor-product spline space of degree p and maximal regularity
 * C^{p-1} on open knot vectors Xi_l, and an isoparametric geometry map
 * F(zeta) = sum_i C_i B_i(zeta) (control points C_i).  The library
 * forms the N_DOF x N_DOF matrices
 *   M~ (mass,      Eq. mass2 P:505-507 evaluated by Eq. massquadrature)
 *   S~ (stiffness, Eq. stiff P:518-524 with Eq. coef_stiff P:527-529 evaluated
 *       by the stiffness analogue of Eq. massquadrature, reading R3)
 * by the row loop of Alg. 3 and writes them as CSR.  Optional
 * scalar PDE coefficients ("Non-constant coefficients could be included
 * as well", "c incorporates the coefficient of the equation") are
 * folded into c and C (reading R17): for -div(kappa grad u) + gamma u,
 *   c = gamma |det J|,   C = kappa |det J| J^{-1} J^{-T}.
 * The SGQ entry point forms the same matrices by the standard element loop
 * with (p+1)^d Gauss points per element, the paper's comparison
 * method.
 *
 * Conventions (all calls):
 *  - Indices are 0-based.  Multi-indices are linearised with i_1 fastest
 *    (P:487-491); columns of a row are ascending.
 *  - row_ptr is int64 (nnz exceeds 2^31 at the BASELINE sizes); columns are
 *    int32 global indices (N_DOF < 2^31 is checked at plan creation).
 *  - Device pointers are CUDA global-memory pointers on the plan's device;
 *    host pointers are ordinary (preferably pinned) host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  The stream-ordered calls (wq_build_rules, wq_build_coef,
 *    wq_pattern, wq_assemble, wq_assemble_sgq) never synchronise the host and
 *    may be captured into a CUDA graph.
 *  - Errors: every call returns a wq_status; wq_last_error() gives a
 *    thread-local human-readable detail of the last failure.  All validation
 *    happens in wq_plan_create (WQ_EINVAL, WQ_EKNOTS, WQ_ERANGE, WQ_ESINGULAR,
 *    WQ_EGEOMETRY, WQ_ENOMEM); after a successful create only WQ_ECUDA (and
 *    WQ_EINVAL for bad arguments of a later call) can occur.  A control net
 *    passed later to the stream-ordered wq_build_coef is checked on the
 *    device; its geometry verdict is reported by wq_check.
 *  - Ownership: the caller owns every buffer it passes; the plan copies the
 *    knot vectors, control net and coefficient nets, and owns its device
 *    workspaces until wq_plan_destroy.
 *  - Threads: one plan must not be used by two host threads at once;
 *    distinct plans are independent (also on distinct devices).
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

/* Points of the two boundary knot spans (Remark 1, reading R1).
 * WQ_BPTS_INTERIOR: p+1 equispaced points strictly inside the span (the
 * default; every exactness system is solvable).  WQ_BPTS_ENDPOINTS: p+1
 * equispaced points including the span's two knots (SPEC's reading); it
 * leaves #Q_i = p-1+2i < #I_i = p+1+i for rows 0 and 1, which violates Eq.
 * numb_nodes, so wq_plan_create rejects it with WQ_ESINGULAR and
 * names the first such row.  It exists to make that reading testable.        */
typedef enum { WQ_BPTS_INTERIOR = 0, WQ_BPTS_ENDPOINTS = 1 } wq_bpts;

/* Row-block kernel selection for wq_assemble_ex (all give results within the
 * parity tolerance of the oracle); every kernel reads
 * the plan's coefficient field whatever its layout.                          */
typedef enum {
    WQ_KERNEL_AUTO = 0,   /* the library's choice for (d, p, matrix): see
                             wq_plan_info_t.kernel                            */
    WQ_KERNEL_DIRECT = 1, /* per-entry direct nested sum (Eq. massquadrature),
                             a reference kernel                               */
    WQ_KERNEL_TILE = 2,   /* sum-factorised row-tile kernel (Eq.
                             sumfactorization P:837): lines of rows along
                             direction 1 share the direction-3/2 stages        */
    WQ_KERNEL_ZLINE = 3,  /* d = 3, 2 <= p <= 6, stiffness, n_EL >= p+2 in
                             every direction (the 2p+3 row staircase types it
                             compiles in; else WQ_EINVAL): lines along
                             direction 3 (rows share the direction-1/2 mode
                             products, the direction-3 product per row),
                             warp-specialised TMA pipeline, direct coalesced
                             stores                                           */
    WQ_KERNEL_ZHP = 4,    /* d = 3, any p, mass and stiffness: lines along
                             direction 3 in t_1 column chunks, CTA-wide
                             phases (the high-degree / mass kernel)           */
    WQ_KERNEL_SF2 = 5     /* d <= 2, any p, mass and stiffness: one warp per
                             row, the two contractions of Eq.
                             sumfactorization in shared memory
                             (Alg. 3); WQ_EINVAL when d = 3 or
                             the row tables exceed 200 KB of shared memory  */
} wq_kernel;

typedef struct wq_plan_s *wq_plan;

typedef struct {
    int d;                        /* 1..3                                      */
    int p;                        /* degree, 1..WQ_MAX_DEGREE                  */
    const int64_t *n_knots;       /* [d] host; n_knots[l] = n_dof[l] + p + 1    */
    const double *const *knots;   /* [d] host FP64 knot vectors Xi_l:
                                     open (p+1 equal end knots), interior knots
                                     simple and strictly increasing            */
    const double *ctrl;           /* host FP64 [N_DOF][d] control points C_i of
                                     the geometry map, row = linear
                                     index (i_1 fastest); NULL: no geometry yet
                                     (call wq_build_coef before assembling)    */
    const double *kappa;          /* host FP64 [N_DOF] spline coefficients of the
                                     diffusion coefficient kappa(zeta) (same
                                     space as the geometry), or NULL (kappa = 1) */
    const double *gamma;          /* host FP64 [N_DOF] reaction coefficient
                                     gamma(zeta) folded into c, or NULL (= 1)   */
    int64_t slab_begin;           /* rows owned by this plan: planes           */
    int64_t slab_end;             /*   [slab_begin, slab_end) of the slowest
                                     index i_d; (0, -1) = all planes            */
    int need_mass;                /* allocate for WQ_MASS                       */
    int need_stiffness;           /* allocate for WQ_STIFFNESS                  */
    int bpts;                     /* wq_bpts (0 = WQ_BPTS_INTERIOR)             */
    int device;                   /* CUDA device ordinal                        */
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
    int32_t max_q[3];             /* max_i #Q_{l,i}: 3p+1 when n_EL >= p+2      */
    int64_t coef_points;          /* points of the coefficient sub-grid held    */
    int64_t workspace_bytes;      /* device bytes owned by the plan             */
    int32_t kernel[2];            /* wq_kernel that WQ_KERNEL_AUTO runs for
                                     [WQ_MASS], [WQ_STIFFNESS] (0: not allocated) */
    int32_t uniform_rules;        /* 1 if the uniform-mesh interior rules (R16)
                                     are in use, else 0                          */
} wq_plan_info_t;

/* Validate the description, copy the knots (and control / coefficient nets)
 * to the device, allocate the plan's workspaces, and run steps 1-5 of the hot
 * path synchronously on an internal stream: the point grid and rules
 * (wq_build_rules) and, if desc->ctrl is given, the coefficient field
 * (wq_build_coef).  Returns
 *   WQ_EINVAL / WQ_EKNOTS / WQ_ERANGE  for invalid sizes, knots or slab,
 *   WQ_ESINGULAR  if an exactness system has no solution (#Q_i < #I_i, or
 *                 a residual above 1e-13 backward-relative; R4/R5),
 *   WQ_EGEOMETRY  if det J vanishes or changes sign on the grid (R7),
 *   WQ_ENOMEM / WQ_ECUDA.
 * *out is NULL on failure.                                                  */
wq_status wq_plan_create(const wq_plan_desc *desc, wq_plan *out);
wq_status wq_plan_destroy(wq_plan plan);
wq_status wq_plan_info(wq_plan plan, wq_plan_info_t *info);

/* Steps 1-4 (Alg. 1 lines 3-8, Alg. 2), stream-ordered re-run of
 * what wq_plan_create computed: point grid and index ranges (Remark 1,
 * reading R1), basis tables B^(0), B^(1), exact integrals I^(a,b) (Eq.
 * integrals) by (p+1)-point Gauss in double-double, and the four min-norm
 * weight families W^(a,b) (Alg. 2, readings R4/R5) in double-double, rounded
 * once to FP64.  The rules are a pure function of the knots: the result is
 * bit-identical to the one validated at create.                             */
wq_status wq_build_rules(wq_plan plan, void *stream);

/* Step 5 (Alg. 1 lines 12/15): the coefficient field on the plan's
 * tensor sub-grid by sum-factorised evaluation of J = dF/dzeta:
 * c = gamma |det J| (mass) and C = kappa |det J| J^{-1} J^{-T} (stiffness).
 * d_ctrl: device FP64 [N_DOF][d] (new geometry), row = linear control index;
 * d_kappa, d_gamma: device FP64 [N_DOF] coefficient nets or NULL (= 1).
 * A vanishing or sign-changing det J is latched on the device and reported
 * by wq_check.                                                              */
wq_status wq_build_coef(wq_plan plan, const double *d_ctrl, const double *d_kappa, const double *d_gamma,
                        void *stream);

/* Step 6: CSR pattern of the owned rows (bit-exact closed form).
 * d_row_ptr: device int64 [n_rows_local + 1], row_ptr[0] = nnz_base;
 * d_col: device int32 [nnz_local] or NULL (row_ptr only).
 * nnz_base = number of nonzeros in all rows before row_begin (multi-GPU).   */
wq_status wq_pattern(wq_plan plan, int64_t nnz_base, int64_t *d_row_ptr, int32_t *d_col, void *stream);

/* Step 7: values of the owned rows of M~ or S~ in CSR order.
 * d_val: device FP64 [nnz_local]; d_col_or_null: if non-NULL the column
 * indices are written in the same pass (fused pattern).  Needs a coefficient
 * field (desc->ctrl at create, or wq_build_coef earlier on the stream).
 * WQ_EINVAL if the plan was created without the matrix or has no geometry.  */
wq_status wq_assemble(wq_plan plan, wq_matrix matrix, double *d_val, int32_t *d_col_or_null, void *stream);
wq_status wq_assemble_ex(wq_plan plan, wq_matrix matrix, wq_kernel kernel, double *d_val,
                         int32_t *d_col_or_null, void *stream);

/* The standard method the paper compares against (Sect. 5.2):
 * element loop with (p+1)^d Gauss-Legendre points per element, local
 * (p+1)^d x (p+1)^d matrices scatter-added into the same CSR layout
 * (d_val is overwritten; d_col_or_null as in wq_assemble).  d_ctrl: device
 * FP64 [N_DOF][d]; d_kappa / d_gamma: device [N_DOF] or NULL (= 1).  The
 * geometry and coefficients are evaluated at the Gauss points themselves.   */
wq_status wq_assemble_sgq(wq_plan plan, wq_matrix matrix, const double *d_ctrl, const double *d_kappa,
                          const double *d_gamma, double *d_val, int32_t *d_col_or_null, void *stream);

/* Synchronise `stream` and report device-side verdicts of the last
 * stream-ordered wq_build_coef: WQ_EGEOMETRY (det J), or WQ_ECUDA.          */
wq_status wq_check(wq_plan plan, void *stream);

/* End to end with HOST buffers (the call a CPU-side user makes): copies
 * h_ctrl [N_DOF][d] (and h_kappa / h_gamma [N_DOF] or NULL) to the device,
 * runs steps 1-7 for `matrix`, and copies the owned CSR block back to
 * h_row_ptr [n_rows_local+1], h_col [nnz_local], h_val [nnz_local] (pinned
 * host memory recommended).  The value kernel is run in row chunks whose
 * device->host copies overlap the next chunk.  Synchronous; includes
 * wq_check.                                                                 */
wq_status wq_form_host(wq_plan plan, wq_matrix matrix, const double *h_ctrl, const double *h_kappa,
                       const double *h_gamma, int64_t nnz_base, int64_t *h_row_ptr, int32_t *h_col, double *h_val,
                       void *stream);

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
