#pragma once
// wq_zline.cuh -- step 7 for the stiffness matrix in 3D: the z-line
// kernel (WQ_KERNEL_ZLINE), warp-specialised persistent kernel, compile-time P.
//
// Arithmetic (Eq. sumfactorization P:837 / Alg. 3; stiffness
// reading R8, families R3).  A LINE is the set of rows i = (i0, i1, i2) with
// (i0, i1) fixed and i2 running over the plan's slab; its rows share the first
// two mode products, the third one is done per row:
//   stage A (contract c0):
//     Y_{m,a2}(pt; c1, t0) = sum_c0 B0^{[m==0]}_{t0}(c0) H_{m,a2}(c0, c1)
//     H_{m,1} = w0^(0,b0) w1^(0,b1) C_2m
//     H_{m,0} = w0^(1,b0) w1^(0,b1) C_0m + w0^(0,b0) w1^(1,b1) C_1m,   b_k = [m==k]
//   stage B (contract c1):
//     G[b2][a2](pt; t0, t1) = sum_{m: [m==2]=b2} sum_c1 B1^{[m==1]}_{t1}(c1) Y_{m,a2}(pt; c1, t0)
//   stage C (contract c2, per row i2):
//     S(i; t0, t1, t2) = sum_c2 B2_{t2}(c2) U0(c2) + B2'_{t2}(c2) U1(c2),
//     U0 = w2^(0,0) G[0][0] + w2^(1,0) G[0][1],  U1 = w2^(0,1) G[1][0] + w2^(1,1) G[1][1].
// Direction 2 is the slowest index of a row's CSR segment (columns ascend with
// j0 fastest), so a lane that owns one column pair (t0, t1) writes S for every
// t2 with plain coalesced stores straight from registers: no staging buffer,
// no barrier among the consumers.
//
// Roles inside one persistent CTA per SM (roles fixed by SM sub-partition):
//   producer warps (warp % 4 in {0, 1}): task = 2 consecutive points q2 of a
//     line.  Lane 0 TMA-loads the task's coefficient box (2 points x #Q0 x #Q1
//     x 6 components) from the z-layout field [comp][q0][q1][q2]; stage A with
//     lanes = (m, c1), Y over the consumed box (separate buffer for boundary
//     lines), stage B with lanes = (m, t0); G of the two points and their
//     direction-2 basis pairs go to a ring of NTS task slots (mbarriers
//     gfull / gempty).
//   consumer warps (warp % 4 in {2, 3}): batches of NR consecutive rows,
//     batches round-robin over the consumer warps; each lane owns CPL columns
//     (t0, t1); per-row weights w2 come in by one bulk copy per batch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <cmath>
#include <algorithm>
#include <vector>
#include "wq_rows.cuh"
#include "wq_dev.cuh"

using namespace wqdev;

// debug builds (-DWQ_ZL_PROF): per-warp wait accounting buffer (defined in wq_assemble_zline.cu)
extern unsigned long long *g_zprof;

// one translation unit per degree (wq_zline_deg<p>.cu) instantiates the kernels of that degree
#define WQ_ZLINE_DEG_DECL(PP) \
    wq_status zline_launch_deg_##PP(wq_plan_s *P, bool bnd, bool pu, bool cu, const int32_t *lines, int64_t n_lines, \
                                    int64_t pl_lo, int64_t pl_hi, double *val, int32_t *col, int64_t val_base, \
                                    const void *uni, cudaStream_t s);
WQ_ZLINE_DEG_DECL(2) WQ_ZLINE_DEG_DECL(3) WQ_ZLINE_DEG_DECL(4) WQ_ZLINE_DEG_DECL(5) WQ_ZLINE_DEG_DECL(6)

namespace {

struct ZPar {
    // rows per consumer batch, producer / consumer warps per SM sub-partition (sub-partitions 0, 1
    // produce, 2, 3 consume), task slots, box buffers per producer, t_1 columns per chunk, consumer
    // batches as one stream over the CTA's items (1) or restarting at warp 0 on every item (0)
    int nr, rwp, rwc, nts, nb, t0c, rot;
};
// p >= 5: the columns (t_1, t_2) of a line are done in chunks of t0c values of t_1 (one launch per
// chunk; stage A/B work splits without redundancy, only the coefficient boxes are re-read), which
// keeps the G ring (4 t0c (2p+1) doubles per point) and the registers within the SM
__host__ __device__ constexpr ZPar z_par(int p, bool bnd) {
    switch (p) {
    case 2: return bnd ? ZPar{2, 3, 3, 32, 1, 5, 1} : ZPar{4, 3, 3, 32, 2, 5, 1};
    case 3: return bnd ? ZPar{1, 3, 3, 16, 1, 7} : ZPar{1, 3, 3, 32, 2, 7};
    case 4: return bnd ? ZPar{1, 2, 2, 16, 1, 9} : ZPar{1, 2, 2, 16, 2, 9};
    case 5: return bnd ? ZPar{1, 1, 2, 16, 1, 6} : ZPar{1, 2, 2, 16, 1, 6};
    case 6: return bnd ? ZPar{1, 1, 2, 16, 1, 7} : ZPar{1, 2, 2, 16, 1, 7};
    default: return {0, 0, 0, 0, 0, 0, 0};
    }
}

template <int P, bool BND>
struct ZCfg {
    static constexpr ZPar W = z_par(P, BND);
    static constexpr bool ENABLED = W.nr > 0;
    static constexpr int K = 2 * P + 1;   // #I of an interior row = #Q of an interior row
    static constexpr int QI = 2 * P + 1;
    static constexpr int QB = 3 * P + 1;  // max #Q of a row
    static constexpr int NP = P + 1;
    static constexpr int T0C = ENABLED ? W.t0c : K;   // t_1 values per column chunk
    static constexpr int NCH = (K + T0C - 1) / T0C;   // chunks (launches per line class)
    static constexpr int COLS = T0C * K;              // columns (t0 local, t1) of a chunk, t0 fastest
    static constexpr int CPL = (COLS + 31) / 32;  // columns (t0, t1) per consumer lane
    static constexpr int NR = ENABLED ? W.nr : 1;
    static constexpr int RWP = ENABLED ? W.rwp : 1, RWC = ENABLED ? W.rwc : 1;
    static constexpr int NWC = 2 * RWC, NWP = 2 * RWP;
    static constexpr int NT = 128 * (RWP > RWC ? RWP : RWC);
    static constexpr int NTS = ENABLED ? W.nts : 2;
    static constexpr int NB = ENABLED ? W.nb : 1;
    static constexpr bool ROT = W.rot != 0;
    // boundary lines: three staircase groups instead of 2P+3 row types (ZTy::group; the full set of
    // unrolled staircases overflows the instruction cache: 40 % no-instruction stalls at p = 4)
    // ZMA: direction 0 (stage A) - only without column chunks (the shift moves slots across chunks);
    // ZMB: direction 1 (stage B)
    static constexpr bool ZMA = BND && NCH == 1 && P >= 3;
    static constexpr bool ZMB = BND && P >= 3;
    // points per producer task: 4 at p = 2 (interior boxes), the two point pairs on the two half-warps
    // (15 stage-A fibres and 15 stage-B lanes per pair), else 2
    static constexpr int PTS = P == 2 && !BND ? 4 : 2;
    static constexpr int RING = PTS * NTS;
    static constexpr int QX = BND ? QB : QI;         // box / table extent in directions 0, 1
    static constexpr int NF = 3 * QX;                // stage-A fibres (m, c1)
    static constexpr int NPASS = (NF + 31) / 32;
    static constexpr int NPP = (NP + 1) & ~1;        // table row length (r pairs)
    // Y blocks (m*2 + a2) of QX*K*2 doubles, 128-B aligned block stride plus a per-block shift that
    // spreads the stage-B lanes (g, t0) over distinct bank groups
    static constexpr int YB = (QX * T0C * 2 + 4 + 15) / 16 * 16;
    __host__ __device__ static constexpr int yoff(int bi) { return bi * YB + (bi == 1 || bi == 3 ? 2 : (bi >= 4 ? 4 : 0)); }
    static constexpr int YTOT = 6 * YB;
    // Y in its own buffer (the box is then only read through the generic proxy and its next TMA load
    // needs no proxy fence, and it can be issued right after stage A: C4 p = 4 5.52 -> 5.45 ms), except
    // for the 4-point tasks of p = 2, where Y goes over the consumed box
    static constexpr bool YSEP = BND || NPASS > 1 || P >= 3;
    static constexpr int BOXD = YSEP ? (6 * QX * QX * PTS + 15) / 16 * 16
                                     : ((6 * QX * QX * PTS > YTOT * (PTS / 2) ? 6 * QX * QX * PTS : YTOT * (PTS / 2)) + 15) / 16 * 16;
    static constexpr int YD = YSEP ? YTOT : 0;
    static constexpr int TABD = (4 * QX * NPP + 8 * QX + QX + 1) & ~1;  // T0, T1, W0, W1, offsets (ints); 16-B multiple
    static constexpr int W2D = NR * QB * 4;                  // doubles per consumer weight buffer
    __host__ __device__ static constexpr size_t al(size_t x) { return (x + 127) & ~(size_t)127; }
    static constexpr size_t O_BAR = 0;
    static constexpr size_t O_BOX = al(8 * (NB * NWP + 2 * NTS + 2 * NWC));
    static constexpr size_t O_TAB = al(O_BOX + (size_t)NWP * (NB * BOXD + YD) * 8);
    static constexpr size_t O_G = al(O_TAB + (size_t)NWP * TABD * 8);
    static constexpr size_t O_B2 = al(O_G + (size_t)RING * 2 * COLS * 16);
    static constexpr size_t O_W2 = al(O_B2 + (size_t)RING * NP * 16);
    static constexpr size_t SMEM = al(O_W2 + (size_t)NWC * 2 * W2D * 8);
    // direction-2 tables of the slab follow at SMEM: pref [n2l+1] int64 (relative to the slab), then
    // qlo (local point), qlen, jlo, jlen [n2l] int32, span [nq2l] int32
    __host__ __device__ static constexpr size_t d2_bytes(int64_t n2l, int64_t nq2l) {
        return al(8 * (size_t)(n2l + 1) + 16 * (size_t)n2l + 4 * (size_t)nq2l);
    }
    static constexpr bool FITS = ENABLED && 3 * T0C <= 32 && NT <= 1024 &&
                                 SMEM + d2_bytes(64, 2 * 64 + 2 * P + 1) <= 227 * 1024;
};

// Row types of one direction (n >= 2p+3 rows, n_EL >= p+2): 0 interior (p+1 <= i <= n-p-2), 1..p+1
// left boundary row i = t-1, p+2..2p+2 right boundary row i = n-1-(t-p-2).  Each type has a fixed
// #Q and staircase offset of its point c (first nonzero function - jlo), from the point grid of
// Remark 1 (reading R1):
//   interior      [0, 1,1, 2,2, .., p,p]                      #Q = 2p+1
//   left i        [0]*(p+1) + [1,1, .., i,i]                   #Q = p+1+2i
//   right i'      [0] + [1,1, .., i'-1,i'-1] + [i'] + [i']*(p+1)  #Q = p+1+2i'
// (verified against the device tables of every row by z_check_types before the first launch)
template <int P>
struct ZTy {
    static constexpr int NTY = 2 * P + 3;
    __host__ __device__ static constexpr int nq(int t) {
        return t == 0 ? 2 * P + 1 : (t <= P + 1 ? P + 1 + 2 * (t - 1) : P + 1 + 2 * (t - P - 2));
    }
    __host__ __device__ static constexpr int off(int t, int c) {
        if (t == 0) return (c + 1) / 2;
        if (t <= P + 1) return c <= P ? 0 : (c - P + 1) / 2;
        const int ip = t - P - 2;
        if (ip == 0 || c == 0) return 0;
        return c >= 2 * ip - 1 ? ip : (c + 1) / 2;
    }
    __host__ __device__ static int type(int64_t i, int64_t n) {
        if (i <= P) return (int)i + 1;
        if (i >= n - 1 - P) return (int)(n - 1 - i) + P + 2;
        return 0;
    }
    // Staircase groups (boundary-line kernel): every left type is a prefix of the longest left type
    // P+1 (the extra points get zero weights), and right type i' equals the longest right type 2P+2
    // on points shifted by 2 sh, sh = P - i', with every offset raised by sh:
    //   off(2P+2, c + 2 sh) = off(t, c) + sh.
    // So three staircases (interior, left P+1, right 2P+2) serve all 2P+3 types: the box and tables
    // start 2 sh points earlier (zero weights there) and the results are written sh slots lower.
    __host__ __device__ static constexpr int group(int t) { return t == 0 ? 0 : (t <= P + 1 ? P + 1 : 2 * P + 2); }
    __host__ __device__ static constexpr int shift(int t) { return t <= P + 1 ? 0 : 2 * P + 2 - t; }
};
// f(integral_constant<t>) for the runtime row type t in [0, 2P+2]
template <int P, int T = 0, class F>
__device__ __forceinline__ void zdispatch(int t, F &&f) {
    if constexpr (T < ZTy<P>::NTY) {
        if (t == T) f(std::integral_constant<int, T>{});
        else zdispatch<P, T + 1>(t, f);
    }
}

struct ZArgs {
    DirView v[3];
    int64_t L0, L1;        // sum_i #I_{0,i}, sum_i #I_{1,i}
    int64_t slab_b;        // first owned plane of i2 (CSR offsets are relative to it)
    int64_t i2b, n2l;      // rows of this launch: planes [i2b, i2b + n2l) of the slab
    int64_t cq_b;          // first q2 of the coefficient sub-grid
    int64_t qoff;          // even local q2 (relative to cq_b) of this launch's first task point
    const int32_t *lines;  // line = i0 + n0 * i1
    int64_t n_items;
    const int32_t *bounds;  // boundary lines: [gridDim.x + 1] cost-balanced contiguous chunks, or null
    double *val;
    int32_t *col;
    int64_t val_base;
    unsigned long long *prof;  // debug builds (-DWQ_ZL_PROF): per (block, warp) [total, wait1, wait2] cycles
    int dbg;                   // debug builds: ablation mask (WQ_ZL_DBG): 1 no consumer stores, 2 no consumer
                               // fast-path arithmetic, 4 no producer stage A/B arithmetic
};

// debug builds: per-warp wait accounting (tools/prof_zline.py); compiled out of the product build
#ifdef WQ_ZL_MIXED
#define ZMIXED 1
#else
#define ZMIXED 0
#endif
#ifdef WQ_ZL_PROF
#define ZPROF 1
#define ZDBG(bit) (a.dbg & (bit))
#else
#define ZPROF 0
#define ZDBG(bit) false
#endif
__device__ __forceinline__ void zwait(uint64_t *b, unsigned par, unsigned long long &acc) {
    if (ZPROF) {
        const long long t0 = clock64();
        mbar_wait(b, par);
        acc += clock64() - t0;
    } else {
        mbar_wait(b, par);
    }
}

// Interior rules of a uniform mesh (translation invariant: every interior row i has the same
// weights w(c) on its points c = 0..2p, and the basis values at its points depend only on whether
// the point is a span midpoint (c even) or a knot (c odd), Remark 1).  Verified against the
// device-computed rules of every interior row before use (z_fetch_uniform).
#define WQ_ZPMAX 6
struct __align__(16) ZUni {
    double w[3][2 * WQ_ZPMAX + 1][4];  // [dir][c][f], f = a + 2b
    double b[3][2][WQ_ZPMAX + 1][2];   // [dir][c & 1][r][value, derivative] of functions span..span+p
};

struct ZItem {
    int i0, i1, ql0, ql1, jl0, jl1, nq0, nq1, ni0, ni1;
};

__device__ __forceinline__ ZItem z_item(const ZArgs &a, int64_t it) {
    ZItem I;
    const int line = a.lines[it];
    const int n0 = (int)a.v[0].n;
    I.i0 = line % n0;
    I.i1 = line / n0;
    I.ql0 = a.v[0].qlo[I.i0];
    I.jl0 = a.v[0].jlo[I.i0];
    I.nq0 = a.v[0].qlen[I.i0];
    I.ni0 = a.v[0].jlen[I.i0];
    I.ql1 = a.v[1].qlo[I.i1];
    I.jl1 = a.v[1].jlo[I.i1];
    I.nq1 = a.v[1].qlen[I.i1];
    I.ni1 = a.v[1].jlen[I.i1];
    return I;
}

// PU: the line's producer tables from the uniform rules (lines with i0, i1 in [2p, n-1-2p]);
// CU: rows i2 in [2p, n2-1-2p] take the uniform rules in the consumer
template <int P, bool BND, bool PU, bool CU, int CH>
__global__ void __launch_bounds__(ZCfg<P, BND>::NT, 1)
    k_zline(const __grid_constant__ CUtensorMap tm, ZArgs a, const __grid_constant__ ZUni u) {
    using CF = ZCfg<P, BND>;
    constexpr int QX = CF::QX;
    constexpr int K = CF::K, QI = CF::QI, NP = CF::NP, COLS = CF::COLS, CPL = CF::CPL;
    constexpr int NR = CF::NR, NWC = CF::NWC, NWP = CF::NWP, NTS = CF::NTS, RING = CF::RING, NB = CF::NB;
    constexpr int NF = CF::NF, BOXD = CF::BOXD, NPP = CF::NPP;
    constexpr int T0C = CF::T0C, T0A = CH * T0C, T0N = K - T0A < T0C ? K - T0A : T0C;  // this chunk's t_1 range
    constexpr bool YSEP = CF::YSEP;
    constexpr int BS = wq_bstride(P);
    extern __shared__ __align__(128) unsigned char smb[];
    uint64_t *pfull = (uint64_t *)(smb + CF::O_BAR);  // [NWP][NB]
    uint64_t *gfull = pfull + NB * NWP;                // [NTS]
    uint64_t *gempty = gfull + NTS;                    // [NTS]
    uint64_t *wfull = gempty + NTS;                    // [NWC][2]
    double *Boxes = (double *)(smb + CF::O_BOX);
    double *Tabs = (double *)(smb + CF::O_TAB);
    double2 *Gs = (double2 *)(smb + CF::O_G);  // [RING][b2][COLS] (a2 = 0, 1) pairs
    double2 *B2r = (double2 *)(smb + CF::O_B2);  // [RING][NP] (value, derivative) of direction 2
    double *W2all = (double *)(smb + CF::O_W2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const DirView &v2 = a.v[2];
    const int n2l = (int)a.n2l;
    const int i2b = (int)a.i2b;
    const int cqb = (int)(a.cq_b + a.qoff);  // local point 0 of this launch (even offset in the z field)
    // direction-2 tables of the slab (shared by every line)
    int64_t *pref2 = (int64_t *)(smb + CF::SMEM);
    int *qlo2 = (int *)(pref2 + n2l + 1), *qlen2 = qlo2 + n2l, *jlo2 = qlen2 + n2l, *jlen2 = jlo2 + n2l;
    int *span2 = jlen2 + n2l;
    const int q_end = v2.qlo[i2b + n2l - 1] + v2.qlen[i2b + n2l - 1] - cqb;  // local end of the last row's Q
    const int nq2l = q_end;
    for (int x = tid; x < n2l; x += blockDim.x) {
        qlo2[x] = v2.qlo[i2b + x] - cqb; qlen2[x] = v2.qlen[i2b + x]; jlo2[x] = v2.jlo[i2b + x]; jlen2[x] = v2.jlen[i2b + x];
    }
    for (int x = tid; x <= n2l; x += blockDim.x) pref2[x] = v2.pref[i2b + x] - v2.pref[a.slab_b];
    for (int x = tid; x < nq2l; x += blockDim.x) span2[x] = v2.span[cqb + x];
    // tasks: local points (2 tau, 2 tau + 1); the slab's first point is local 0
    constexpr int PTS = CF::PTS;
    static_assert(PTS == 2 || (3 * QX <= 16 && 3 * CF::T0C <= 16 && !CF::YSEP), "4-point tasks");
    const int NTASK = (q_end + PTS - 1) / PTS;
    // items of this CTA: round-robin (neighbouring lines run concurrently and share their coefficient
    // boxes in L2), or a contiguous chunk (boundary lines, sorted by row type: one code path per CTA)
    // boundary lines: chunks of ZCH consecutive lines (same row types, sorted on the host) dealt
    // round-robin, which keeps the per-CTA work balanced
    // (with a.bounds: the host's cost-balanced per-CTA item ranges)
    constexpr int64_t ZCH = BND ? 4 : 1;
    const int64_t G = gridDim.x, c_ = blockIdx.x;
    int64_t my_items, ib = 0;
    if (a.bounds) {
        ib = a.bounds[c_];
        my_items = a.bounds[c_ + 1] - ib;
    } else {
        const int64_t R = a.n_items / (G * ZCH), rem = a.n_items - R * G * ZCH;
        const int64_t ex = rem - c_ * ZCH;
        my_items = R * ZCH + (ex < 0 ? 0 : (ex > ZCH ? ZCH : ex));
    }
    auto item_of = [&](int64_t k) { return a.bounds ? ib + k : ((k / ZCH) * G + c_) * ZCH + k % ZCH; };
    const int64_t n_tasks = my_items * NTASK;

    if (tid == 0) {
        for (int s = 0; s < NB * NWP; ++s) mbar_init(&pfull[s], 1);
        for (int s = 0; s < NTS; ++s) { mbar_init(&gfull[s], 32); mbar_init(&gempty[s], NWC); }
        for (int s = 0; s < 2 * NWC; ++s) mbar_init(&wfull[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int smsp = warp & 3, wrow = warp >> 2;
    const long long t_start = clock64();
    unsigned long long wt1 = 0, wt2 = 0;
    auto prof_out = [&]() {
        if (ZPROF && a.prof && lane == 0) {
            unsigned long long *o = a.prof + ((size_t)blockIdx.x * (blockDim.x / 32) + warp) * 3;
            o[0] = clock64() - t_start; o[1] = wt1; o[2] = wt2;
        }
    };
    // roles: WQ_ZL_MIXED: warps 0..NWP-1 producers (one per SM sub-partition and row), the rest
    // consumers; else by sub-partition (warp % 4 in {0, 1} producers)
    const bool is_prod = ZMIXED ? warp < NWP : smsp < 2;
    if (!ZMIXED && (is_prod ? wrow >= CF::RWP : wrow >= CF::RWC)) return;  // idle warp (RWP != RWC)
    if (is_prod) {
        // ============================================================ producer warp
        const int wp = ZMIXED ? warp : wrow * 2 + smsp;
        double *wbase = Boxes + wp * (NB * BOXD + CF::YD);
        double *Ybuf = wbase + NB * BOXD;  // YSEP only
        if constexpr (CF::ZMB) {
            // group staircases read Y rows beyond the row's points (times zero tables): keep them finite
            for (int x = lane; x < CF::YD; x += 32) Ybuf[x] = 0.0;
            __syncwarp();
        }
        double *tab = Tabs + wp * CF::TABD;
        // line tables: T0[sel][c0][NPP], T1[sel][c1][NPP] (sel 0: derivative, 1: value; r padded to
        // NPP so that (r, r+1) pairs load as one 16-B word), W0t / W1t [c][f] (f = a + 2b)
        double *T0 = tab, *T1 = T0 + 2 * QX * NPP;
        double *W0t = T1 + 2 * QX * NPP, *W1t = W0t + 4 * QX;
        constexpr unsigned BOX_BYTES = 6 * QX * QX * PTS * 8;
        // PTS = 4: half-warp hp works on point pair hp of the task, sub-lane sl
        const int hp = PTS == 4 ? lane >> 4 : 0, sl = PTS == 4 ? lane & 15 : lane;
        // task T = k * NTASK + tau of this warp (T = wp, wp + NWP, ...): item k, point pair tau; the
        // issue stream (TMA of the coefficient boxes) runs NB tasks ahead of the compute stream
        int64_t ik = -1, is_k = wp / NTASK, is_T = wp;
        int is_tau = wp % NTASK;
        int iq0 = 0, iq1 = 0;
        auto issue = [&](int b) {  // lane 0: TMA of the next task of the issue stream into buffer b
            if (is_T >= n_tasks) return;
            if (is_k != ik) {
                const ZItem I = z_item(a, item_of(is_k));
                ik = is_k; iq0 = I.ql0; iq1 = I.ql1;
                if (CF::ZMA) iq0 -= 2 * ZTy<P>::shift(ZTy<P>::type(I.i0, a.v[0].n));
                if (CF::ZMB) iq1 -= 2 * ZTy<P>::shift(ZTy<P>::type(I.i1, a.v[1].n));
            }
            if (ZDBG(8)) {
                mbar_arrive(&pfull[wp * NB + b]);  // debug ablation: no box load
            } else {
                mbar_arrive_tx(&pfull[wp * NB + b], BOX_BYTES);
                tma_load_4d(wbase + b * BOXD, &tm, &pfull[wp * NB + b], (int)a.qoff + PTS * is_tau, iq1, iq0, 0);
            }
            is_T += NWP;
            is_tau += NWP;
            while (is_tau >= NTASK) { is_tau -= NTASK; ++is_k; }
        };
        if (lane == 0) {
            issue(0);
            if (NB == 2) issue(1);
        }
        int64_t k = wp / NTASK;
        int tau = wp % NTASK;
        int64_t cur_item = -1;
        // stage B lanes (g, t0): g = 0, 1 -> b2 = 0, a2 = g (chains m = 0 and m = 1 summed in the lane);
        // g = 2 -> b2 = 1 (chain m = 2, both a2).  Input blocks x = 0, 1 of Y and their tables:
        const int fg = sl / T0C, fc = sl % T0C;
        const bool fl = sl < 3 * T0C && fc < T0N;
        const int ybx0 = fg == 0 ? 0 : (fg == 1 ? 1 : 4), ybx1 = fg == 0 ? 2 : (fg == 1 ? 3 : 5);  // Y blocks m*2+a2
        const int tsel1 = fg == 2 ? 1 : 0;  // table of block x = 1: B1' for m = 1, B1 for m = 2
        // PU: this lane's selections of the uniform tables (stage A: family b0 = [m == 0], weights of
        // its c1; stage B: table of block x = 1)
        double b0s[2][NP], w0s[QI][2], b1x[2][NP], w1u0 = 0.0, w1u1 = 0.0;
        if constexpr (PU) {
            const int m = sl / QX < 3 ? sl / QX : 2, c1 = sl % QX;
            #pragma unroll
            for (int par = 0; par < 2; ++par)
                #pragma unroll
                for (int r = 0; r <= P; ++r) {
                    b0s[par][r] = u.b[0][par][r][m == 0 ? 1 : 0];
                    b1x[par][r] = u.b[1][par][r][tsel1 ? 0 : 1];
                }
            #pragma unroll
            for (int c = 0; c < QI; ++c) {
                w0s[c][0] = u.w[0][c][m == 0 ? 2 : 0];
                w0s[c][1] = u.w[0][c][m == 0 ? 3 : 1];
            }
            w1u0 = u.w[1][c1][m == 1 ? 2 : 0];
            w1u1 = u.w[1][c1][m == 1 ? 3 : 1];
        }

        int cq0 = QI, cq1 = QI, ty0 = 0, ty1 = 0, sh0 = 0, sh1 = 0;
        // boundary lines with column chunks (p >= 5, no direction-0 staircase groups): stage A loops
        // over the offset groups of the line's row type (first plane of offset o = og0[o]) instead of
        // one fully unrolled staircase per row type (2p+3 of them: 12.8 K instructions at p = 6)
        constexpr bool OGA = BND && !CF::ZMA && P >= 5;
        int og0[OGA ? NP + 1 : 1];
        #pragma unroll
        for (int o = 0; o < (OGA ? NP + 1 : 1); ++o) og0[o] = 0;
        int use = 0;
        for (int64_t T = wp; T < n_tasks; T += NWP, ++use) {
            const int b = NB == 2 ? (use & 1) : 0;
            if (use > 0) {
                tau += NWP;
                while (tau >= NTASK) { tau -= NTASK; ++k; }
            }
            if (!PU && k != cur_item) {
                cur_item = k;
                const ZItem I = z_item(a, item_of(k));
                const DirView &v0 = a.v[0], &v1 = a.v[1];
                __syncwarp();
                if (BND) {
                    cq0 = I.nq0; cq1 = I.nq1;
                    ty0 = ZTy<P>::type(I.i0, v0.n);
                    ty1 = ZTy<P>::type(I.i1, v1.n);
                    if (CF::ZMA) {
                        sh0 = ZTy<P>::shift(ty0);
                        ty0 = ZTy<P>::group(ty0);
                        cq0 += 2 * sh0;
                    }
                    if (CF::ZMB) {
                        sh1 = ZTy<P>::shift(ty1);
                        ty1 = ZTy<P>::group(ty1);
                        cq1 += 2 * sh1;
                    }
                }
                if constexpr (OGA) {
                    #pragma unroll
                    for (int o = 0; o <= P; ++o) {
                        int c = 0;
                        while (c < cq0 && ZTy<P>::off(ty0, c) < o) ++c;
                        og0[o] = c;
                    }
                    og0[P + 1] = cq0;
                }
                // tables over the box's points c (the row's points start at c = 2 sh)
                const int64_t tq0 = I.ql0 - 2 * sh0, tq1 = I.ql1 - 2 * sh1;
                for (int x = lane; x < QX * NPP; x += 32) {
                    const int c = x / NPP, r = x % NPP;
                    const double2 b0 = c < cq0 && r < NP ? __ldg((const double2 *)(v0.B + (tq0 + c) * BS) + r) : make_double2(0.0, 0.0);
                    const double2 b1 = c < cq1 && r < NP ? __ldg((const double2 *)(v1.B + (tq1 + c) * BS) + r) : make_double2(0.0, 0.0);
                    T0[x] = b0.y; T0[QX * NPP + x] = b0.x; T1[x] = b1.y; T1[QX * NPP + x] = b1.x;
                }
                for (int x = lane; x < 4 * QX; x += 32) {
                    W0t[x] = x / 4 >= 2 * sh0 && x / 4 < cq0 ? __ldg(v0.W + (int64_t)I.i0 * v0.maxq * 4 + x - 8 * sh0) : 0.0;
                    W1t[x] = x / 4 >= 2 * sh1 && x / 4 < cq1 ? __ldg(v1.W + (int64_t)I.i1 * v1.maxq * 4 + x - 8 * sh1) : 0.0;
                }
                __syncwarp();
            }
            // direction-2 basis pairs of the task's points (published with G)
            double2 b2v = make_double2(0.0, 0.0);
            const int b2pt = lane / NP, b2r = lane % NP;
            const int b2q = PTS * tau + b2pt;
            if (lane < PTS * NP && b2q < q_end) b2v = __ldg((const double2 *)(v2.B + (int64_t)(cqb + b2q) * BS) + b2r);
            zwait(&pfull[wp * NB + b], (NB == 2 ? use >> 1 : use) & 1, wt1);
            const double *bx = wbase + b * BOXD;  // [comp][c0][c1][pt]
            // ---------------- stage A: fibre (m, c1), both points, chains a2 = 0 (y0), 1 (y1)
            // Y: block m*2+a2 at CF::yoff, [c1][t0][pt] inside; interior: over the consumed box
            double *Y = YSEP ? Ybuf : wbase + b * BOXD + hp * CF::YTOT;
            #pragma unroll(CF::ZMB ? 1 : CF::NPASS)
            for (int pass = 0; pass < CF::NPASS; ++pass) {
                // boundary lines: the 3 #Q_1 fibres of this line packed densely (one pass when #Q_1 <= 10)
                if (BND && 32 * pass >= 3 * cq1) break;
                const int f = sl + 32 * pass;
                const int m = BND ? f / cq1 : f / QX, c1 = BND ? f % cq1 : f % QX;
                const bool fv = BND ? f < 3 * cq1 : f < NF;
                double y0[2][T0C], y1[2][T0C];
                #pragma unroll
                for (int pt = 0; pt < 2; ++pt)
                    #pragma unroll
                    for (int t = 0; t < T0C; ++t) { y0[pt][t] = 0.0; y1[pt][t] = 0.0; }
                if (fv && !ZDBG(4)) {
                    // components: a2 = 1 chain C_2m, a2 = 0 chain C_0m and C_1m (C_00 C_01 C_02 C_11 C_12 C_22)
                    const int ka = m == 0 ? 2 : (m == 1 ? 4 : 5);
                    const int kb = m == 0 ? 0 : (m == 1 ? 1 : 2);
                    const int kc = m == 0 ? 1 : (m == 1 ? 3 : 4);
                    const double2 w1p = PU ? make_double2(w1u0, w1u1)
                                           : *(const double2 *)(W1t + c1 * 4 + (m == 1 ? 2 : 0));  // w1^(0,b1), w1^(1,b1)
                    const double *T0s = T0 + (m == 0 ? 0 : QX * NPP);
                    const int w0o = m == 0 ? 2 : 0;
                    auto plane = [&](int c0, auto O) {
                        constexpr int o0 = decltype(O)::value;
                        const double2 w0p = PU ? make_double2(w0s[c0 % QI][0], w0s[c0 % QI][1])
                                               : *(const double2 *)(W0t + c0 * 4 + w0o);  // w0^(0,b0), w0^(1,b0)
                        const double s1 = w0p.x * w1p.x, s2 = w0p.y * w1p.x, s3 = w0p.x * w1p.y;
                        const double2 ca = *(const double2 *)(bx + ((ka * QX + c0) * QX + c1) * PTS + 2 * hp);
                        const double2 cb = *(const double2 *)(bx + ((kb * QX + c0) * QX + c1) * PTS + 2 * hp);
                        const double2 cc = *(const double2 *)(bx + ((kc * QX + c0) * QX + c1) * PTS + 2 * hp);
                        const double h1a = s1 * ca.x, h1b = s1 * ca.y;                                // l = 2
                        const double h0a = fma(s2, cb.x, s3 * cc.x), h0b = fma(s2, cb.y, s3 * cc.y);  // l = 0, 1
                        #pragma unroll
                        for (int rr = 0; rr < NPP / 2; ++rr) {
                            const double2 bp = PU ? make_double2(0.0, 0.0) : *(const double2 *)(T0s + c0 * NPP + 2 * rr);
                            #pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int r = 2 * rr + h;
                                if (r > P) continue;
                                const int t = o0 + r - T0A;  // compile time: t_1 in this chunk?
                                if (t < 0 || t >= T0N) continue;
                                const double bv = PU ? b0s[c0 & 1][r] : (h ? bp.y : bp.x);
                                y1[0][t] = fma(bv, h1a, y1[0][t]);
                                y1[1][t] = fma(bv, h1b, y1[1][t]);
                                y0[0][t] = fma(bv, h0a, y0[0][t]);
                                y0[1][t] = fma(bv, h0b, y0[1][t]);
                            }
                        }
                    };
                    if constexpr (CF::ZMA) {
                        // the group staircases as one unrolled interior staircase over a range of
                        // its points plus a rolled loop over the flat part (ZTy::group): left
                        // [0]*(P+1) + interior points 1..2P; right interior points 0..2P-2 + [P]*(P+2)
                        const int base = ty0 == P + 1 ? P : 0, clo = ty0 == P + 1 ? 1 : 0,
                                  chi = ty0 == 2 * P + 2 ? 2 * P - 2 : 2 * P;
                        unroll<QI>([&](auto C0) {
                            constexpr int c0 = decltype(C0)::value;
                            if (c0 >= clo && c0 <= chi) plane(base + c0, std::integral_constant<int, (c0 + 1) / 2>{});
                        });
                        if (ty0 == P + 1) {
                            #pragma unroll 1
                            for (int c0 = 0; c0 <= P; ++c0) plane(c0, std::integral_constant<int, 0>{});
                        } else if (ty0 == 2 * P + 2) {
                            #pragma unroll 1
                            for (int c0 = 2 * P - 1; c0 <= 3 * P; ++c0) plane(c0, std::integral_constant<int, P>{});
                        }
                    } else if constexpr (OGA) {
                        unroll<NP>([&](auto O) {
                            constexpr int o = decltype(O)::value;
                            #pragma unroll 1
                            for (int c0 = og0[o]; c0 < og0[o + 1]; ++c0) plane(c0, std::integral_constant<int, o>{});
                        });
                    } else if constexpr (BND) {
                        zdispatch<P>(ty0, [&](auto TT) {
                            constexpr int t = decltype(TT)::value;
                            unroll<ZTy<P>::nq(t)>([&](auto C0) {
                                constexpr int c0 = decltype(C0)::value;
                                plane(c0, std::integral_constant<int, ZTy<P>::off(t, c0)>{});
                            });
                        });
                    } else {
                        unroll<QI>([&](auto C0) {
                            constexpr int c0 = decltype(C0)::value;
                            plane(c0, std::integral_constant<int, (c0 + 1) / 2>{});
                        });
                    }
                }
                if (!YSEP) __syncwarp();  // every lane has read the box: Y may overwrite it
                if (fv) {
                    double *Y0 = Y + CF::yoff(m * 2 + 0) + c1 * T0C * 2;
                    double *Y1 = Y + CF::yoff(m * 2 + 1) + c1 * T0C * 2;
                    #pragma unroll
                    for (int t = 0; t < T0C; ++t) {
                        // ZMA: slot t of the group staircase is slot t - sh0 of the row (slots at
                        // and above #I_0 - sh0... are dead columns, never read as live)
                        const int td = CF::ZMA ? t - sh0 : t;
                        if (td >= 0) {
                            *(double2 *)(Y0 + td * 2) = make_double2(y0[0][t], y0[1][t]);
                            *(double2 *)(Y1 + td * 2) = make_double2(y1[0][t], y1[1][t]);
                        }
                    }
                }
            }
            __syncwarp();
            if constexpr (YSEP) {
                // the box is consumed (Y has its own buffer): start the next task's box load now.  The
                // box was only read through the generic proxy (no cross-proxy write to order), and
                // every lane's reads have completed (their values fed stage A) before the __syncwarp
                if (lane == 0) issue(b);
            }
            // ---------------- stage B: lane (g, t0): acc[x][pt][t1] over the Y blocks x = 0, 1
            double g[2][2][K];
            #pragma unroll
            for (int x = 0; x < 2; ++x)
                #pragma unroll
                for (int pt = 0; pt < 2; ++pt)
                    #pragma unroll
                    for (int t = 0; t < K; ++t) g[x][pt][t] = 0.0;
            if (fl && !ZDBG(4)) {
                const int t0 = fc;
                const double *Ya = Y + CF::yoff(ybx0) + t0 * 2;
                const double *Yb = Y + CF::yoff(ybx1) + t0 * 2;  // t0: this lane's t_1 within the chunk
                const double *Ta = T1 + QX * NPP, *Tb = T1 + tsel1 * QX * NPP;
                auto point1 = [&](int c1, auto O) {
                    constexpr int o1 = decltype(O)::value;
                    const double2 ya = *(const double2 *)(Ya + c1 * T0C * 2);
                    const double2 yb = *(const double2 *)(Yb + c1 * T0C * 2);
                    #pragma unroll
                    for (int rr = 0; rr < NPP / 2; ++rr) {
                        const double2 pa = PU ? make_double2(0.0, 0.0) : *(const double2 *)(Ta + c1 * NPP + 2 * rr);
                        const double2 pb = PU ? make_double2(0.0, 0.0) : *(const double2 *)(Tb + c1 * NPP + 2 * rr);
                        #pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int r = 2 * rr + h;
                            if (r > P) continue;
                            const double ba = PU ? u.b[1][c1 & 1][r][0] : (h ? pa.y : pa.x);
                            const double bb = PU ? b1x[c1 & 1][r] : (h ? pb.y : pb.x);
                            g[0][0][o1 + r] = fma(ba, ya.x, g[0][0][o1 + r]);
                            g[0][1][o1 + r] = fma(ba, ya.y, g[0][1][o1 + r]);
                            g[1][0][o1 + r] = fma(bb, yb.x, g[1][0][o1 + r]);
                            g[1][1][o1 + r] = fma(bb, yb.y, g[1][1][o1 + r]);
                        }
                    }
                };
                if constexpr (CF::ZMB) {
                    const int base = ty1 == P + 1 ? P : 0, clo = ty1 == P + 1 ? 1 : 0,
                              chi = ty1 == 2 * P + 2 ? 2 * P - 2 : 2 * P;
                    unroll<QI>([&](auto C1) {
                        constexpr int c1 = decltype(C1)::value;
                        if (c1 >= clo && c1 <= chi) point1(base + c1, std::integral_constant<int, (c1 + 1) / 2>{});
                    });
                    if (ty1 == P + 1) {
                        #pragma unroll 1
                        for (int c1 = 0; c1 <= P; ++c1) point1(c1, std::integral_constant<int, 0>{});
                    } else if (ty1 == 2 * P + 2) {
                        #pragma unroll 1
                        for (int c1 = 2 * P - 1; c1 <= 3 * P; ++c1) point1(c1, std::integral_constant<int, P>{});
                    }
                } else if constexpr (BND) {
                    zdispatch<P>(ty1, [&](auto TT) {
                        constexpr int t = decltype(TT)::value;
                        unroll<ZTy<P>::nq(t)>([&](auto C1) {
                            constexpr int c1 = decltype(C1)::value;
                            point1(c1, std::integral_constant<int, ZTy<P>::off(t, c1)>{});
                        });
                    });
                } else {
                    unroll<QI>([&](auto C1) {
                        constexpr int c1 = decltype(C1)::value;
                        point1(c1, std::integral_constant<int, (c1 + 1) / 2>{});
                    });
                }
            }
            // G of the slot ([pt][b2][col] (a2 = 0, 1) pairs): lanes g = 0, 1 store the sum of their
            // two chains as component a2 = g of b2 = 0; lanes g = 2 store both components of b2 = 1
            const uint32_t Tl = (uint32_t)T;
            const int slot_t = (int)(Tl % NTS);
            zwait(&gempty[slot_t], ((Tl / NTS) & 1) ^ 1, wt2);
            {
                // lanes g = 0 receive the a2 = 1 sums of lanes g = 1 and store (a2 = 0, a2 = 1) pairs of
                // b2 = 0; lanes g = 2 store their pairs of b2 = 1 (one 16-B store per lane and entry)
                const int t0 = fc;
                const double sum1 = fg < 2 ? 1.0 : 0.0;
                const int b2 = fg == 2 ? 1 : 0;
                #pragma unroll
                for (int pt = 0; pt < 2; ++pt) {
                    double2 *Gd = Gs + ((slot_t * PTS + 2 * hp + pt) * 2 + b2) * COLS + t0;
                    #pragma unroll
                    for (int t = 0; t < K; ++t) {  // t = t_2; column t0 + T0C t
                        const double v = fma(g[1][pt][t], sum1, g[0][pt][t]);
                        const double o = __shfl_down_sync(0xffffffffu, v, T0C, PTS == 4 ? 16 : 32);
                        const int td = CF::ZMB ? t - sh1 : t;  // slot of the row (see ZTy::shift)
                        if (fl && fg != 1 && td >= 0) Gd[T0C * td] = make_double2(v, fg == 0 ? o : g[1][pt][t]);
                    }
                }
            }
            if (lane < PTS * NP) B2r[(slot_t * PTS + b2pt) * NP + b2r] = b2v;
            mbar_arrive(&gfull[slot_t]);
            // the buffer is free again (all lanes done with Y): prefetch the task after next into it
            if constexpr (!YSEP) {
                fence_async_smem();
                __syncwarp();
                if (lane == 0) issue(b);
            }
        }
        prof_out();
        return;
    }

    // ============================================================ stage C consumers
    const int cw = ZMIXED ? warp - NWP : wrow * 2 + (smsp - 2);
    const DirView &v0 = a.v[0], &v1 = a.v[1];
    const int n0 = (int)v0.n, n01 = n0 * (int)v1.n;
    int colx[CPL], colr[CPL], t0c[CPL], t1c[CPL];
    #pragma unroll
    for (int j = 0; j < CPL; ++j) {
        colx[j] = lane + 32 * j;
        colr[j] = colx[j] < COLS ? colx[j] : COLS - 1;  // clamped column for shared-memory reads
        t0c[j] = T0A + colx[j] % T0C;  // global t_1 of the column
        t1c[j] = colx[j] / T0C;
    }
    double *W2b = W2all + cw * 2 * CF::W2D;  // [2][NR][mq2][4]
    const int mq2 = v2.maxq;
    // W2 rows of a batch are contiguous in global memory ([i][c][f]): one bulk copy per batch,
    // prefetched one batch ahead into a double buffer
    // a batch whose rows all take the uniform rules (CU) reads no W2 rows: no copy and no wait (the
    // issue and the wait side take the same decision per batch, so the buffer phases stay paired;
    // C4 p = 4 5.64 -> 5.39 ms)
    auto w2_need = [&](int r0) {
        if (!CU) return true;
        const int nr = n2l - r0 < NR ? n2l - r0 : NR;
        return !(i2b + r0 >= 2 * P && i2b + r0 + nr - 1 <= (int)v2.n - 1 - 2 * P);
    };
    auto w2_issue = [&](int r0, int buf) {
        if (!w2_need(r0)) return;
        const int nr = n2l - r0 < NR ? n2l - r0 : NR;
        const unsigned bytes = (unsigned)(nr * mq2 * 32);
        mbar_arrive_tx(&wfull[cw * 2 + buf], bytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(W2b + buf * CF::W2D)),
                     "l"(v2.W + (int64_t)(i2b + r0) * mq2 * 4), "r"(bytes), "r"(smem_u32(&wfull[cw * 2 + buf]))
                     : "memory");
    };
    // ROT: the batches of the CTA's items form one round-robin stream over the consumer warps (batch
    // b of item k is stream position k nb + b): the warp after the one that took a line's last batch
    // takes the next line's first, so the extra batch of a ragged line and the generic (non-uniform)
    // rows at the line ends rotate over the warps instead of always landing on warp 0 (measured: p = 2
    // 2.00 -> 1.74 ms at C4; p = 3 slower, 3.25 -> 3.39 ms; p = 4 unchanged: 52 batches per line)
    const int nbl = (n2l + NR - 1) / NR;
    auto first_row = [&](int64_t k) {
        return (int)((cw + NWC - (CF::ROT ? (int)((k * nbl) % NWC) : 0)) % NWC) * NR;
    };
    // first row of the first item >= k in which this warp has a batch (-1: none left)
    auto next_first = [&](int64_t k) {
        for (int64_t k2 = k; k2 < my_items && k2 < k + NWC; ++k2)
            if (first_row(k2) < n2l) return first_row(k2);
        return -1;
    };
    int wbuf = 0;
    unsigned wuse[2] = {0, 0};
    if (lane == 0) {
        const int f0 = next_first(0);
        if (f0 >= 0) w2_issue(f0, 0);
    }
    uint32_t got = 0, rel = 0, Tbase = 0;  // tasks waited for / released, first task of the item
    for (int64_t ik_ = 0; ik_ < my_items; ++ik_) {
        const ZItem I = z_item(a, item_of(ik_));
        bool live[CPL];
        int el[CPL], colb[CPL];
        #pragma unroll
        for (int j = 0; j < CPL; ++j) {
            live[j] = colx[j] < COLS && colx[j] % T0C < T0N && t0c[j] < I.ni0 && t1c[j] < I.ni1;
            el[j] = t0c[j] + I.ni0 * t1c[j];
            colb[j] = (I.jl0 + t0c[j]) + n0 * (I.jl1 + t1c[j]);
        }
        const int nc01 = I.ni0 * I.ni1;
        const int64_t A = v1.pref[I.i1] * a.L0 + (int64_t)I.ni1 * v0.pref[I.i0];
        const int64_t L01 = a.L0 * a.L1;
        for (int r0 = first_row(ik_); r0 < n2l; r0 += NWC * NR) {
            const int nr = n2l - r0 < NR ? n2l - r0 : NR;
            const int rl = r0 + nr - 1;
            const uint32_t t_hi = Tbase + (uint32_t)((qlo2[rl] + qlen2[rl] - 1) / PTS);
            const uint32_t t_lo = Tbase + (uint32_t)(qlo2[r0] / PTS);
            if (w2_need(r0)) {
                zwait(&wfull[cw * 2 + wbuf], wuse[wbuf] & 1, wt2);
                ++wuse[wbuf];
            }
            const double2 *W2w = (const double2 *)(W2b + wbuf * CF::W2D);  // [row][c][2] double2, row stride mq2
            if (lane == 0) {
                int nxt = r0 + NWC * NR;
                bool more = true;
                if (nxt >= n2l) { nxt = next_first(ik_ + 1); more = nxt >= 0; }
                if (more) w2_issue(nxt, wbuf ^ 1);
            }
            wbuf ^= 1;
            __syncwarp();
            while (rel < got && rel < t_lo) {
                if (lane == 0) mbar_arrive_relaxed(&gempty[rel % NTS]);
                ++rel;
            }
            while (got <= t_hi) {
                zwait(&gfull[got % NTS], (got / NTS) & 1, wt1);
                ++got;
                while (rel < got && rel < t_lo) {
                    if (lane == 0) mbar_arrive_relaxed(&gempty[rel % NTS]);
                    ++rel;
                }
            }
            __syncwarp();
            double acc[NR][CPL][K];
            #pragma unroll
            for (int k = 0; k < NR; ++k)
                #pragma unroll
                for (int j = 0; j < CPL; ++j)
                    #pragma unroll
                    for (int t = 0; t < K; ++t) acc[k][j][t] = 0.0;
            auto slot_of = [&](int q) { return (int)((Tbase * PTS + (uint32_t)q) % RING); };
            // fast path: a full batch of rows with the interior staircase; with CU only rows whose
            // rules are the uniform ones (the others go through the generic path)
            const int rlo = CU ? 2 * P : P + 1, rhi = CU ? (int)v2.n - 1 - 2 * P : (int)v2.n - P - 2;
            const bool interior = nr == NR && i2b + r0 >= rlo && i2b + r0 + NR - 1 <= rhi;
            if (interior && !ZDBG(2)) {
                const int slot0 = slot_of(qlo2[r0]);
                constexpr int UW = 2 * (NR - 1) + 2 * P + 1;
                #pragma unroll
                for (int u_ = 0; u_ < UW; ++u_) {
                    int slot = slot0 + u_;
                    if (slot >= RING) slot -= RING;
                    double2 g0[CPL], g1[CPL];
                    #pragma unroll
                    for (int j = 0; j < CPL; ++j) {
                        g0[j] = Gs[(slot * 2 + 0) * COLS + colr[j]];
                        g1[j] = Gs[(slot * 2 + 1) * COLS + colr[j]];
                    }
                    double2 bb[NP];
                    #pragma unroll
                    for (int r = 0; r <= P; ++r)
                        bb[r] = CU ? make_double2(u.b[2][u_ & 1][r][0], u.b[2][u_ & 1][r][1]) : B2r[slot * NP + r];
                    #pragma unroll
                    for (int k = 0; k < NR; ++k) {
                        if (u_ >= 2 * k && u_ <= 2 * k + 2 * P) {
                            const int c = u_ - 2 * k;
                            const int o0 = (c + 1) / 2;
                            const double2 *wr = W2w + (k * mq2 + c) * 2;
                            const double2 wA = CU ? make_double2(u.w[2][c][0], u.w[2][c][1]) : wr[0];
                            const double2 wB = CU ? make_double2(u.w[2][c][2], u.w[2][c][3]) : wr[1];
                            #pragma unroll
                            for (int j = 0; j < CPL; ++j) {
                                const double u0 = fma(wA.x, g0[j].x, wA.y * g0[j].y);
                                const double u1 = fma(wB.x, g1[j].x, wB.y * g1[j].y);
                                #pragma unroll
                                for (int r = 0; r <= P; ++r)
                                    acc[k][j][o0 + r] = fma(bb[r].x, u0, fma(bb[r].y, u1, acc[k][j][o0 + r]));
                            }
                        }
                    }
                }
            } else if (!interior && !ZDBG(16)) {
                #pragma unroll
                for (int k = 0; k < NR; ++k) {
                    if (k >= nr) break;
                    const int r = r0 + k;
                    const int qb = qlo2[r], nq = qlen2[r], jl = jlo2[r];
                    // an interior row takes the uniform rules here too, so that its values do not
                    // depend on how the rows were batched (bit-identical to the interior path)
                    const bool ru = CU && i2b + r >= 2 * P && i2b + r <= (int)v2.n - 1 - 2 * P;
                    #pragma unroll 1
                    for (int c = 0; c < nq; ++c) {
                        const int q = qb + c;
                        const int slot = slot_of(q);
                        const double2 *bp = ru ? (const double2 *)&u.b[2][c & 1][0][0] : B2r + slot * NP;
                        const double2 *wr = ru ? (const double2 *)&u.w[2][c][0] : W2w + (k * mq2 + c) * 2;
                        const double2 wA = wr[0], wB = wr[1];
                        double u0[CPL], u1[CPL];
                        #pragma unroll
                        for (int j = 0; j < CPL; ++j) {
                            const double2 g0 = Gs[(slot * 2 + 0) * COLS + colr[j]];
                            const double2 g1 = Gs[(slot * 2 + 1) * COLS + colr[j]];
                            u0[j] = fma(wA.x, g0.x, wA.y * g0.y);
                            u1[j] = fma(wB.x, g1.x, wB.y * g1.y);
                        }
                        const int off = span2[q] - jl;
                        dispatch<0, K - NP>(off, [&](auto O) {
                            constexpr int o0 = decltype(O)::value;
                            #pragma unroll
                            for (int r = 0; r <= P; ++r) {
                                const double2 bq = bp[r];
                                #pragma unroll
                                for (int j = 0; j < CPL; ++j)
                                    acc[k][j][o0 + r] = fma(bq.x, u0[j], fma(bq.y, u1[j], acc[k][j][o0 + r]));
                            }
                        });
                    }
                }
            }
            {
                const int nb = r0 + NWC * NR;
                const int low = nb < n2l ? qlo2[nb] : q_end;
                const uint32_t t_rel = Tbase + (uint32_t)(low / PTS);
                __syncwarp();
                while (rel < t_rel && rel < got) {
                    if (lane == 0) mbar_arrive_relaxed(&gempty[rel % NTS]);
                    ++rel;
                }
            }
            // stores straight from registers: for fixed (row, t2) the lanes' columns are consecutive;
            // interior lines have the compile-time stride K*K between the t2 slices of a row
            const int nc = BND ? nc01 : K * K;
            #pragma unroll
            for (int k = 0; k < NR; ++k) {
                if (k >= nr || ZDBG(1)) break;
                const int r = r0 + k;
                const int ni2 = jlen2[r];
                const int64_t ro = pref2[r] * L01 + (int64_t)ni2 * A - a.val_base;
                const int cb2 = n01 * jlo2[r];
                #pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    if (!live[j]) continue;
                    double *dv = a.val + ro + el[j];
                    int32_t *dc = a.col + ro + el[j];
                    const int c0 = colb[j] + cb2;
                    if (ni2 == K) {
                        #pragma unroll
                        for (int t = 0; t < K; ++t) __stcs(dv + nc * t, acc[k][j][t]);
                        if (a.col) {
                            #pragma unroll
                            for (int t = 0; t < K; ++t) __stcs(dc + nc * t, c0 + n01 * t);
                        }
                    } else {
                        #pragma unroll
                        for (int t = 0; t < K; ++t)
                            if (t < ni2) __stcs(dv + nc * t, acc[k][j][t]);
                        if (a.col) {
                            #pragma unroll
                            for (int t = 0; t < K; ++t)
                                if (t < ni2) __stcs(dc + nc * t, c0 + n01 * t);
                        }
                    }
                }
            }
        }
        const uint32_t t_end = Tbase + (uint32_t)NTASK;
        while (rel < t_end) {
            if (got <= rel) {
                mbar_wait(&gfull[got % NTS], (got / NTS) & 1);
                ++got;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&gempty[rel % NTS]);
            ++rel;
        }
        Tbase = t_end;
    }
    prof_out();
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 z_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}


template <int N, class F>
void hunroll(F &&f) {  // host-side compile-time loop
    if constexpr (N > 0) {
        hunroll<N - 1>(f);
        f(std::integral_constant<int, N - 1>{});
    }
}

int z_num_sms(int dev) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

template <int P, bool BND, bool PU, bool CU>
wq_status launch_zline_p(wq_plan_s *Pl, const int32_t *lines, int64_t n_lines, int64_t pl_lo, int64_t pl_hi,
                         double *val, int32_t *col, int64_t val_base, const ZUni &un, cudaStream_t s) {
    using CF = ZCfg<P, BND>;
    if constexpr (!CF::FITS) {
        wq_set_error("z-line kernel not configured for this degree");
        return WQ_EINVAL;
    } else {
        if (n_lines <= 0) return WQ_OK;
        ZArgs a;
        for (int l = 0; l < 3; ++l) a.v[l] = Pl->dir[l];
        a.L0 = Pl->L[0];
        a.L1 = Pl->L[1];
        a.slab_b = Pl->slab_b;
        a.i2b = Pl->slab_b + pl_lo;
        a.n2l = pl_hi - pl_lo;
        a.cq_b = Pl->cq_b;
        a.qoff = (wq_host_qlo(a.i2b, Pl->dir[2].E, Pl->p) - Pl->cq_b) & ~(int64_t)1;
        a.lines = lines;
        a.n_items = n_lines;
        a.bounds = BND && Pl->zbounds_dev && lines == Pl->zlines_dev + Pl->zlines_uni.size() + Pl->zlines_int.size() &&
                           n_lines == (int64_t)Pl->zlines_bnd.size() ? Pl->zbounds_dev : nullptr;
        a.val = val;
        a.col = col;
        a.val_base = val_base;
        a.prof = nullptr;
        a.dbg = getenv("WQ_ZL_DBG") ? atoi(getenv("WQ_ZL_DBG")) : 0;
        if (ZPROF && getenv("WQ_ZL_PROF")) {  // debug: per-warp wait accounting, read back with wq_debug_zprof
            if (!g_zprof) cudaMalloc(&g_zprof, sizeof(unsigned long long) * 148 * 32 * 3 * 3);
            const int slot = BND ? 2 : (PU ? 0 : 1);
            a.prof = g_zprof + (size_t)slot * 148 * 32 * 3;
            cudaMemsetAsync(a.prof, 0, sizeof(unsigned long long) * 148 * 32 * 3, s);
        }
        CUtensorMap m;
        auto fn = z_encode_fn();
        if (!fn) { wq_set_error("cuTensorMapEncodeTiled unavailable"); return WQ_ECUDA; }
        const int64_t nq0 = Pl->dir[0].nq, nq1 = Pl->dir[1].nq;
        cuuint64_t dims[4] = {(cuuint64_t)Pl->zld, (cuuint64_t)nq1, (cuuint64_t)nq0, 6};
        cuuint64_t strides[3] = {(cuuint64_t)Pl->zld * 8, (cuuint64_t)Pl->zld * nq1 * 8, (cuuint64_t)Pl->zcs * 8};
        cuuint32_t box[4] = {(cuuint32_t)CF::PTS, (cuuint32_t)CF::QX, (cuuint32_t)CF::QX, 6};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void *)Pl->coef, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            wq_set_error("cuTensorMapEncodeTiled failed for the z-layout coefficient field");
            return WQ_ECUDA;
        }
        const size_t smem = CF::SMEM + CF::d2_bytes(a.n2l, Pl->cq_e - Pl->cq_b - a.qoff);
        if (smem > 227 * 1024) {
            wq_set_error("z-line kernel: direction-2 tables exceed shared memory");
            return WQ_EINVAL;
        }
        int64_t grid = z_num_sms(Pl->device);
        if (grid > n_lines) grid = n_lines;
        if (a.bounds && grid != Pl->zbounds_n) a.bounds = nullptr;
        // one launch per column chunk of t_1
        wq_status st = WQ_OK;
        hunroll<CF::NCH>([&](auto CC) {
            constexpr int CH = decltype(CC)::value;
            if (st != WQ_OK) return;
            wq_smem_attr((const void *)k_zline<P, BND, PU, CU, CH>, smem);
            k_zline<P, BND, PU, CU, CH><<<(unsigned)grid, CF::NT, smem, s>>>(m, a, un);
            wq_count_launches(1);
            st = wq_cuda_status(cudaGetLastError(), "z-line assembly kernel");
        });
        return st;
    }
}

template <bool BND>
bool fits_z(int p, int64_t n2l, int64_t nq2l) {
    switch (p) {
    case 2: return ZCfg<2, BND>::FITS && ZCfg<2, BND>::SMEM + ZCfg<2, BND>::d2_bytes(n2l, nq2l) <= 227 * 1024;
    case 3: return ZCfg<3, BND>::FITS && ZCfg<3, BND>::SMEM + ZCfg<3, BND>::d2_bytes(n2l, nq2l) <= 227 * 1024;
    case 4: return ZCfg<4, BND>::FITS && ZCfg<4, BND>::SMEM + ZCfg<4, BND>::d2_bytes(n2l, nq2l) <= 227 * 1024;
    case 5: return ZCfg<5, BND>::FITS && ZCfg<5, BND>::SMEM + ZCfg<5, BND>::d2_bytes(n2l, nq2l) <= 227 * 1024;
    case 6: return ZCfg<6, BND>::FITS && ZCfg<6, BND>::SMEM + ZCfg<6, BND>::d2_bytes(n2l, nq2l) <= 227 * 1024;
    }
    return false;
}

}  // namespace
