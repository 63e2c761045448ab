// wq_assemble_line.cu -- step 7 for INTERIOR lines, warp-specialised
// persistent kernel (WQ_KERNEL_LINE), d = 3, stiffness, compile-time P.
//
// Arithmetic of the row-line kernel (Eq. sumfactorization P:837 / Alg. 3
// P:859-870): the rows of a line (i2, i3) share stages 3 and 2,
//   Y_{m,a1}(q1, c2, t3) = sum_c3 B3^{[m==2]}_{t3}(c3) H_{m,a1}(q1, c2, c3)      (stage 3)
//     H_{m,1} = w2^(0,b2) w3^(0,b3) C_0m,  H_{m,0} = w2^(1,b2) w3^(0,b3) C_1m + w2^(0,b2) w3^(1,b3) C_2m
//   G[b1][a1](q1, t2, t3) = sum_c2 sum_{m: [m==0]=b1} B2^{[m==1]}_{t2}(c2) Y_{m,a1}(q1, c2, t3)   (stage 2)
//   out(t1) = sum_c B1_{t1}(c) U0(c) + B1'_{t1}(c) U1(c),
//     U0 = w1^(0,0) G[0][0] + w1^(1,0) G[0][1],  U1 = w1^(0,1) G[1][0] + w1^(1,1) G[1][1]   (stage 1)
// with b2 = [m==1], b3 = [m==2].  A line is interior when its rows in
// directions 2 and 3 touch no boundary span: #Q = 2P+1 in both directions and
// the staircase offset of point c is (c+1)/2 (compile time).  Lines touching a
// boundary in direction 2 or 3 go to the generic kernels.
//
// Roles inside one persistent CTA per SM (no CTA-wide barrier after setup):
//   NWP producer warps, each fully independent: task = 2 consecutive points
//     q1 of a line.  The warp TMA-loads the task's coefficient box
//     (2 x (2P+1) x (2P+1) x 6 comps) into one of its two buffers one task
//     ahead, runs stage 3 with lanes = (m, c2), writes Y over the consumed
//     box, runs stage 2 with lanes = (m, t3) (m = 1, 2 partials combined by a
//     shuffle) and publishes G of the 2 points into a ring of NTS task slots
//     (mbarrier gfull / gempty).
//   NWC consumer warps: stage 1 exactly as in the warp-specialised kernel
//     (teams of TW warps over the K*K columns, NR rows per lane in registers,
//     per-warp staging + TMA bulk stores of values and columns).
// Tasks are numbered T = k * NTASK + tau over the CTA's items k (static
// round-robin over interior lines); producer warp w runs tasks T = w mod NWP.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include "wq_rows.cuh"
#include "wq_dev.cuh"

using namespace wqdev;

namespace {

struct LnPar {
    int nr, nteam, nwp, nts, nb;  // nb: coefficient box buffers per producer warp
};
// BND: lines touching a boundary span in direction 2 or 3 (#Q up to 3p+1, runtime staircase)
__host__ __device__ constexpr LnPar ln_par(int p, bool bnd) {
    if (bnd) {
        switch (p) {
        case 2: return {4, 8, 6, 20, 1};
        case 3: return {4, 4, 6, 16, 1};
        case 4: return {3, 2, 4, 11, 1};
        default: return {0, 0, 0, 0, 0};
        }
    }
    switch (p) {
    case 2: return {4, 8, 8, 24, 2};
    case 3: return {4, 4, 8, 18, 2};
    case 4: return {2, 3, 7, 14, 1};
    default: return {0, 0, 0, 0, 0};
    }
}

template <int P, bool BND>
struct LnCfg {
    static constexpr LnPar W = ln_par(P, BND);
    static constexpr bool ENABLED = W.nr > 0;
    static constexpr int K = 2 * P + 1;   // #I of an interior row = #Q of an interior row
    static constexpr int QI = 2 * P + 1;
    static constexpr int QB = 3 * P + 1;  // max #Q of a row (direction 1 boundary rows)
    static constexpr int NP = P + 1;
    static constexpr int COLS = K * K;
    static constexpr int TW = (COLS + 31) / 32;
    static constexpr int NR = ENABLED ? W.nr : 1;
    static constexpr int NTEAM = ENABLED ? W.nteam : 1;
    static constexpr int NWC = TW * NTEAM;
    static constexpr int NWP = ENABLED ? W.nwp : 1;
    // roles by SM sub-partition (warp % 4): 0, 1 producers, 2, 3 consumers, so that each SMSP runs
    // one role's code (instruction-cache locality) and the FP64 pipes split evenly between the roles
    static constexpr int RW = (NWP + NWC + 3) / 4;  // warps per SMSP
    static constexpr int NT = 32 * 4 * RW;
    static constexpr int NTS = ENABLED ? W.nts : 2;  // task slots (2 points each) in the G ring
    static constexpr int NB = ENABLED ? W.nb : 1;
    static constexpr int RING = 2 * NTS;
    static constexpr int QX = BND ? QB : QI;         // box / table extent in directions 2, 3
    static constexpr int NF = 3 * QX;                // stage-3 fibres (m, c2) per task
    static constexpr int NPASS = (NF + 31) / 32;     // stage-3 passes over the fibres
    // doubles per coefficient box buffer, padded so that every buffer starts 128-B aligned (TMA); the
    // interior kernel writes Y over the consumed box, BND (several stage-3 passes) into its own buffer
    static constexpr int BOXD = (6 * QX * QX * 2 + 15) / 16 * 16;
    static constexpr int YD = BND ? (3 * 2 * QX * K * 2 + 15) / 16 * 16 : 0;
    static constexpr int TABD = 4 * QX * NP + 4 * QX + 4 * QX + QX;  // per-warp line tables (doubles; + offsets)
    // team staging: one row of the team (K^3 entries max) per buffer, 2 buffers (row parity)
    static constexpr int SSTV = (K * K * K + 2 + 1) / 2 * 2;
    static constexpr int SSTC = (K * K * K + 4 + 3) / 4 * 4;
    __host__ __device__ static constexpr size_t al(size_t x) { return (x + 127) & ~(size_t)127; }
    static constexpr size_t O_BAR = 0;
    static constexpr size_t O_BOX = al(8 * (2 * NWP + 2 * NTS + 2 * NWC));
    static constexpr size_t O_TAB = al(O_BOX + (size_t)NWP * (NB * BOXD + YD) * 8);
    static constexpr size_t O_G = al(O_TAB + (size_t)NWP * TABD * 8);
    static constexpr size_t O_B1 = al(O_G + (size_t)4 * RING * COLS * 8);
    static constexpr size_t O_W1 = al(O_B1 + (size_t)RING * NP * 16);
    static constexpr size_t W1D = (size_t)NR * QB * 4;  // doubles per W1 buffer (rows x max #Q x 4 families)
    static constexpr size_t O_SV = al(O_W1 + (size_t)NWC * 2 * W1D * 8);
    static constexpr size_t O_SC = al(O_SV + (size_t)NTEAM * 2 * SSTV * 8);
    static constexpr size_t SMEM = al(O_SC + (size_t)NTEAM * 2 * SSTC * 4);
    // direction-1 index tables (qlo, qlen, jlo, jlen [n1] int32, pref [n1+1] int64, span [nq1] int32)
    // follow at SMEM (size depends on n1: d1_bytes)
    __host__ __device__ static constexpr size_t d1_bytes(int64_t n1, int64_t nq1) {
        return al(16 * (size_t)n1 + 8 * (size_t)(n1 + 1) + 4 * (size_t)nq1);
    }
    static constexpr bool FITS = ENABLED && (BND || NF <= 32) && 3 * K <= 32 &&  SMEM + d1_bytes(128, 2 * 128 + 2 * P + 1) <= 227 * 1024 &&
                                 NT <= 1024;
};

struct LnArgs {
    RowGeo g;
    DirView v[3];
    const int32_t *lines;  // interior lines (i2 + n2 * (i3 - slab_b)), relative to the plan's slab
    int64_t n_items;
    int64_t cq_b;
    double *val;
    int32_t *col;
    int64_t val_base;
    int dbg;  // debug ablation mask (WQ_LINE_DBG), 0 in production
    unsigned long long *prof;  // debug: per (block, warp) [total, wait A, wait B, wait C] cycles, or null
};

struct LItem {
    int i2, i3, ql2, ql3, jl2, jl3, nq2, nq3, ni2, ni3;
};

__device__ __forceinline__ LItem ln_item(const LnArgs &a, int64_t it) {
    LItem I;
    const int line = a.lines[it];
    const int n2 = (int)a.g.n[1];
    I.i2 = line % n2;
    I.i3 = (int)a.g.slab_b + line / n2;
    I.ql2 = a.v[1].qlo[I.i2];
    I.jl2 = a.v[1].jlo[I.i2];
    I.ql3 = a.v[2].qlo[I.i3];
    I.jl3 = a.v[2].jlo[I.i3];
    I.nq2 = a.v[1].qlen[I.i2];
    I.nq3 = a.v[2].qlen[I.i3];
    I.ni2 = a.v[1].jlen[I.i2];
    I.ni3 = a.v[2].jlen[I.i3];
    return I;
}

// debug builds (-DWQ_LINE_DEBUG): ablation mask WQ_LINE_DBG and per-warp wait-cycle accounting
// WQ_LINE_PROF (tools/prof_line.py); compiled out of the product build
#ifdef WQ_LINE_DEBUG
#define LDBG(bit) (a.dbg & (bit))
#define LPROF true
#else
#define LDBG(bit) false
#define LPROF false
#endif

__device__ __forceinline__ void twait(uint64_t *b, unsigned par, unsigned long long *acc) {
    if (LPROF && acc) {
        const long long t0 = clock64();
        mbar_wait(b, par);
        *acc += clock64() - t0;
    } else {
        mbar_wait(b, par);
    }
}

template <int P, bool BND>
__global__ void __launch_bounds__(LnCfg<P, BND>::NT, 1)
    k_line(const __grid_constant__ CUtensorMap tm, LnArgs a) {
    using CF = LnCfg<P, BND>;
    constexpr int QX = CF::QX;
    constexpr int K = CF::K, QI = CF::QI, QB = CF::QB, NP = CF::NP, COLS = CF::COLS, TW = CF::TW;
    constexpr int NR = CF::NR, NTEAM = CF::NTEAM, NWP = CF::NWP, NTS = CF::NTS, RING = CF::RING;
    constexpr int NF = CF::NF, BOXD = CF::BOXD;
    constexpr int BS = wq_bstride(P);
    extern __shared__ __align__(128) unsigned char smb[];
    uint64_t *pfull = (uint64_t *)(smb + CF::O_BAR);  // [NWP][2]
    uint64_t *gfull = pfull + 2 * NWP;                 // [NTS]
    uint64_t *gempty = gfull + NTS;                    // [NTS]
    uint64_t *wfull = gempty + NTS;                    // [NWC][2] W1 prefetch
    double *Boxes = (double *)(smb + CF::O_BOX);
    double *Tabs = (double *)(smb + CF::O_TAB);
    double *Gs = (double *)(smb + CF::O_G);
    double2 *B1r = (double2 *)(smb + CF::O_B1);
    double2 *W1all = (double2 *)(smb + CF::O_W1);
    double *Svall = (double *)(smb + CF::O_SV);
    int32_t *Scall = (int32_t *)(smb + CF::O_SC);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const DirView &v1 = a.v[0];
    const int n1 = (int)a.g.n[0];
    const int nq1 = (int)v1.nq;
    // direction-1 tables are shared by every line: one copy in shared memory per CTA
    int64_t *pref1 = (int64_t *)(smb + CF::SMEM);
    int *qlo1 = (int *)(pref1 + n1 + 1), *qlen1 = qlo1 + n1, *jlo1 = qlen1 + n1, *jlen1 = jlo1 + n1;
    int *span1 = jlen1 + n1;
    for (int x = tid; x < n1; x += blockDim.x) {
        qlo1[x] = v1.qlo[x]; qlen1[x] = v1.qlen[x]; jlo1[x] = v1.jlo[x]; jlen1[x] = v1.jlen[x];
    }
    for (int x = tid; x <= n1; x += blockDim.x) pref1[x] = a.g.pref[0][x];
    for (int x = tid; x < nq1; x += blockDim.x) span1[x] = v1.span[x];
    const int q0 = v1.qlo[0];
    const int q_end = v1.qlo[n1 - 1] + v1.qlen[n1 - 1];
    const int NTASK = (q_end - q0 + 1) / 2;
    const int64_t first = blockIdx.x, step = gridDim.x;
    const int64_t my_items = first < a.n_items ? (a.n_items - first + step - 1) / step : 0;
    const int64_t n_tasks = my_items * NTASK;
    const long long t_start = clock64();
    unsigned long long wA = 0, wB = 0, wC = 0;
    unsigned long long *pA = LPROF && a.prof ? &wA : nullptr, *pB = LPROF && a.prof ? &wB : nullptr,
                       *pC = LPROF && a.prof ? &wC : nullptr;
    auto prof_out = [&]() {
        if (LPROF && a.prof && lane == 0) {
            unsigned long long *o = a.prof + ((size_t)blockIdx.x * (blockDim.x / 32) + warp) * 4;
            o[0] = clock64() - t_start; o[1] = wA; o[2] = wB; o[3] = wC;
        }
    };

    if (tid == 0) {
        for (int s = 0; s < 2 * NWP; ++s) mbar_init(&pfull[s], 1);
        for (int s = 0; s < NTS; ++s) { mbar_init(&gfull[s], 32); mbar_init(&gempty[s], CF::NWC); }
        for (int s = 0; s < 2 * CF::NWC; ++s) mbar_init(&wfull[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // role of this warp: consumers fill SM sub-partitions 2 and 3 first (then 1, then 0, highest
    // warp first), producers take the remaining warps
    int cw = -1, wp = 0;
    {
        int pos = 0;
        for (int pass = 0; pass < 3 && cw < 0; ++pass)
            for (int w = pass == 0 ? 0 : CF::RW * 4 - 1; pass == 0 ? w < CF::RW * 4 : w >= 0; w += pass == 0 ? 1 : -1) {
                const int sp = w & 3;
                const bool take = pass == 0 ? sp >= 2 : (pass == 1 ? sp == 1 : sp == 0);
                if (!take) continue;
                if (pos >= CF::NWC) break;
                if (w == warp) { cw = pos; break; }
                ++pos;
            }
        if (cw < 0) {
            for (int w = 0; w < warp; ++w) {
                int p2 = 0, c2 = -1;
                for (int pass = 0; pass < 3 && c2 < 0; ++pass)
                    for (int x = pass == 0 ? 0 : CF::RW * 4 - 1; pass == 0 ? x < CF::RW * 4 : x >= 0; x += pass == 0 ? 1 : -1) {
                        const int sp = x & 3;
                        const bool take = pass == 0 ? sp >= 2 : (pass == 1 ? sp == 1 : sp == 0);
                        if (!take) continue;
                        if (p2 >= CF::NWC) break;
                        if (x == w) { c2 = p2; break; }
                        ++p2;
                    }
                if (c2 < 0) ++wp;
            }
        }
    }
    if (cw < 0) {
        // ============================================================ producer warp
        if (wp >= NWP) return;
        double *wbase = Boxes + wp * (CF::NB * BOXD + CF::YD);
        double *box[2] = {wbase, wbase + (CF::NB - 1) * BOXD};
        double *Ybuf = wbase + CF::NB * BOXD;  // BND only
        double *tab = Tabs + wp * CF::TABD;
        double *B2v = tab, *B2d = B2v + QX * NP, *B3v = B2d + QX * NP, *B3d = B3v + QX * NP;
        double *W2t = B3d + QX * NP, *W3t = W2t + 4 * QX;  // [c][f], f = a + 2b
        int *off2 = (int *)(W3t + 4 * QX), *off3 = off2 + QX;  // BND: staircase offsets span - jlo
        constexpr unsigned BOX_BYTES = 6 * QX * QX * 2 * 8;
        int64_t ik = -1;
        int iq2 = 0, iq3 = 0;
        auto issue = [&](int64_t T, int b) {  // lane 0: TMA of task T into buffer b
            if (T >= n_tasks || LDBG(1)) return;
            const int64_t k = T / NTASK;
            const int tau = (int)(T % NTASK);
            if (k != ik) {
                const LItem I = ln_item(a, first + k * step);
                ik = k; iq2 = I.ql2; iq3 = (int)(I.ql3 - a.cq_b);
            }
            mbar_arrive_tx(&pfull[wp * 2 + b], BOX_BYTES);
            tma_load_4d(box[b], &tm, &pfull[wp * 2 + b], q0 + 2 * tau + 1, iq2, iq3, 0);
        };
        if (lane == 0) {
            issue(wp, 0);
            if (CF::NB == 2) issue(wp + NWP, 1);
        }
        int64_t cur_item = -1;
        // lane roles: stage 3 fibre (m, c2) (pass-strided for BND), stage 2 fibre (m, t3)
        const int fm = lane / K, fc = lane % K;  // stage 2 (and interior stage 3, QI == K)
        const bool fl = lane < 3 * K;
        int cq2 = QI, cq3 = QI;  // #Q of the current item in directions 2, 3
        int use = 0;
        for (int64_t T = wp; T < n_tasks; T += NWP, ++use) {
            const int b = CF::NB == 2 ? (use & 1) : 0;
            const int64_t k = T / NTASK;
            const int tau = (int)(T % NTASK);
            if (k != cur_item) {
                // line tables of the new item (warp-private)
                cur_item = k;
                const LItem I = ln_item(a, first + k * step);
                const DirView &v2 = a.v[1], &v3 = a.v[2];
                __syncwarp();
                if (BND) { cq2 = I.nq2; cq3 = I.nq3; }
                for (int x = lane; x < QX * NP; x += 32) {
                    const int c = x / NP, r = x % NP;
                    const double2 b2 = c < cq2 ? __ldg((const double2 *)(v2.B + (int64_t)(I.ql2 + c) * BS) + r) : make_double2(0.0, 0.0);
                    const double2 b3 = c < cq3 ? __ldg((const double2 *)(v3.B + (int64_t)(I.ql3 + c) * BS) + r) : make_double2(0.0, 0.0);
                    B2v[x] = b2.x; B2d[x] = b2.y; B3v[x] = b3.x; B3d[x] = b3.y;
                }
                for (int x = lane; x < 4 * QX; x += 32) {
                    W2t[x] = x / 4 < cq2 ? __ldg(v2.W + (int64_t)I.i2 * v2.maxq * 4 + x) : 0.0;
                    W3t[x] = x / 4 < cq3 ? __ldg(v3.W + (int64_t)I.i3 * v3.maxq * 4 + x) : 0.0;
                }
                if (BND)
                    for (int x = lane; x < QX; x += 32) {
                        off2[x] = x < cq2 ? v2.span[I.ql2 + x] - I.jl2 : 0;
                        off3[x] = x < cq3 ? v3.span[I.ql3 + x] - I.jl3 : 0;
                    }
                __syncwarp();
            }
            // direction-1 basis pairs of the task's points (consumed at the end of the task)
            double2 b1v = make_double2(0.0, 0.0);
            const int b1pt = lane / NP, b1r = lane % NP;
            const int b1q = q0 + 2 * tau + b1pt;
            if (lane < 2 * NP && b1q < q_end) b1v = __ldg((const double2 *)(v1.B + (int64_t)b1q * BS) + b1r);
            if (!LDBG(1)) twait(&pfull[wp * 2 + b], (CF::NB == 2 ? use >> 1 : use) & 1, pA);
            const double *bx = box[b];  // [comp][c3][c2][pt]
            // ---------------- stage 3: fibre (m, c2), both points, chains a1 = 0 (y0), 1 (y1)
            // Y layout: [m][a1][c2][t3][pt]; interior: over the consumed box, BND: own buffer
            double *Y = BND ? Ybuf : box[b];
            #pragma unroll
            for (int pass = 0; pass < CF::NPASS; ++pass) {
                const int f = lane + 32 * pass;
                const int m = f / QX, c2 = f % QX;
                const bool fv = f < CF::NF && (!BND || c2 < cq2);
                double y0[2][K], y1[2][K];
                #pragma unroll
                for (int pt = 0; pt < 2; ++pt)
                    #pragma unroll
                    for (int t = 0; t < K; ++t) { y0[pt][t] = 0.0; y1[pt][t] = 0.0; }
                if (fv && !LDBG(4)) {
                    const int ka = m, kb = m == 0 ? 1 : (m == 1 ? 3 : 4), kc = m == 0 ? 2 : (m == 1 ? 4 : 5);
                    const double w2a = W2t[c2 * 4 + (m == 1 ? 2 : 0)];  // w2^(0,b2)
                    const double w2b = W2t[c2 * 4 + (m == 1 ? 3 : 1)];  // w2^(1,b2)
                    const double *B3c = m == 2 ? B3d : B3v;
                    const int b3o = m == 2 ? 2 : 0;
                    auto plane = [&](int c3, auto O) {
                        constexpr int o0 = decltype(O)::value;
                        const double w3a = W3t[c3 * 4 + b3o], w3b = W3t[c3 * 4 + b3o + 1];  // w3^(0,b3), w3^(1,b3)
                        const double s1 = w2a * w3a, s2 = w2b * w3a, s3 = w2a * w3b;
                        const double2 ca = *(const double2 *)(bx + ((ka * QX + c3) * QX + c2) * 2);
                        const double2 cb = *(const double2 *)(bx + ((kb * QX + c3) * QX + c2) * 2);
                        const double2 cc = *(const double2 *)(bx + ((kc * QX + c3) * QX + c2) * 2);
                        const double h1a = s1 * ca.x, h1b = s1 * ca.y;                                // l = 0
                        const double h0a = fma(s2, cb.x, s3 * cc.x), h0b = fma(s2, cb.y, s3 * cc.y);  // l = 1, 2
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) {
                            const double bv = B3c[c3 * NP + r];
                            y1[0][o0 + r] = fma(bv, h1a, y1[0][o0 + r]);
                            y1[1][o0 + r] = fma(bv, h1b, y1[1][o0 + r]);
                            y0[0][o0 + r] = fma(bv, h0a, y0[0][o0 + r]);
                            y0[1][o0 + r] = fma(bv, h0b, y0[1][o0 + r]);
                        }
                    };
                    if constexpr (BND) {
                        #pragma unroll 1
                        for (int c3 = 0; c3 < cq3; ++c3)
                            dispatch<0, K - NP>(off3[c3], [&](auto O) { plane(c3, O); });
                    } else {
                        unroll<QI>([&](auto C3) {
                            constexpr int c3 = decltype(C3)::value;
                            plane(c3, std::integral_constant<int, (c3 + 1) / 2>{});
                        });
                    }
                }
                if (!BND) __syncwarp();  // every lane has read the box: Y may overwrite it
                if (fv) {
                    double *Y0 = Y + ((m * 2 + 0) * QX + c2) * K * 2;
                    double *Y1 = Y + ((m * 2 + 1) * QX + c2) * K * 2;
                    #pragma unroll
                    for (int t = 0; t < K; ++t) {
                        *(double2 *)(Y0 + t * 2) = make_double2(y0[0][t], y0[1][t]);
                        *(double2 *)(Y1 + t * 2) = make_double2(y1[0][t], y1[1][t]);
                    }
                }
            }
            __syncwarp();
            // ---------------- stage 2: lane (m, t3): g[a1][pt][t2]
            double g[2][2][K];
            #pragma unroll
            for (int a1 = 0; a1 < 2; ++a1)
                #pragma unroll
                for (int pt = 0; pt < 2; ++pt)
                    #pragma unroll
                    for (int t = 0; t < K; ++t) g[a1][pt][t] = 0.0;
            if (fl && !LDBG(8)) {
                const int m = fm, t3 = fc;
                const double *B2c = m == 1 ? B2d : B2v;
                const double *Ya0 = Y + ((m * 2 + 0) * QX) * K * 2 + t3 * 2;
                const double *Ya1 = Y + ((m * 2 + 1) * QX) * K * 2 + t3 * 2;
                auto point2 = [&](int c2, auto O) {
                    constexpr int o0 = decltype(O)::value;
                    const double2 ya0 = *(const double2 *)(Ya0 + c2 * K * 2);
                    const double2 ya1 = *(const double2 *)(Ya1 + c2 * K * 2);
                    #pragma unroll
                    for (int r = 0; r <= P; ++r) {
                        const double bv = B2c[c2 * NP + r];
                        g[0][0][o0 + r] = fma(bv, ya0.x, g[0][0][o0 + r]);
                        g[0][1][o0 + r] = fma(bv, ya0.y, g[0][1][o0 + r]);
                        g[1][0][o0 + r] = fma(bv, ya1.x, g[1][0][o0 + r]);
                        g[1][1][o0 + r] = fma(bv, ya1.y, g[1][1][o0 + r]);
                    }
                };
                if constexpr (BND) {
                    #pragma unroll 1
                    for (int c2 = 0; c2 < cq2; ++c2) dispatch<0, K - NP>(off2[c2], [&](auto O) { point2(c2, O); });
                } else {
                    unroll<QI>([&](auto C2) {
                        constexpr int c2 = decltype(C2)::value;
                        point2(c2, std::integral_constant<int, (c2 + 1) / 2>{});
                    });
                }
            }
            // b1 = 0 collects m = 1 and m = 2: lane (1, t3) += lane (2, t3)
            #pragma unroll
            for (int a1 = 0; a1 < 2; ++a1)
                #pragma unroll
                for (int pt = 0; pt < 2; ++pt)
                    #pragma unroll
                    for (int t = 0; t < K; ++t) {
                        const double o = __shfl_down_sync(0xffffffffu, g[a1][pt][t], K);
                        if (fm == 1) g[a1][pt][t] += o;
                    }
            const uint32_t Tl = (uint32_t)T;  // slot accounting in task units
            const int slot_t = (int)(Tl % NTS);
            twait(&gempty[slot_t], ((Tl / NTS) & 1) ^ 1, pB);
            if (fl && fm < 2) {
                const int b1 = fm == 0 ? 1 : 0, t3 = fc;
                #pragma unroll
                for (int a1 = 0; a1 < 2; ++a1)
                    #pragma unroll
                    for (int pt = 0; pt < 2; ++pt) {
                        double *Gd = Gs + ((b1 * 2 + a1) * RING + slot_t * 2 + pt) * COLS + K * t3;
                        #pragma unroll
                        for (int t = 0; t < K; ++t) Gd[t] = g[a1][pt][t];
                    }
            }
            if (lane < 2 * NP && b1q < q_end) B1r[(slot_t * 2 + b1pt) * NP + b1r] = b1v;
            mbar_arrive(&gfull[slot_t]);
            // the buffer is free again (all lanes done with Y): prefetch the task after next into it
            fence_async_smem();
            __syncwarp();
            if (lane == 0) issue(T + CF::NB * NWP, b);
        }
        prof_out();
        return;
    }

    // ============================================================ stage 1 consumers

    const int team = cw / TW, wt = cw % TW;
    const int colx = wt * 32 + lane;
    const int t2c = colx % K, t3c = colx / K;
    bool live = colx < COLS;
    double *W1b = (double *)W1all + cw * 2 * CF::W1D;  // [2][NR][maxq][4]
    double *Sv0 = Svall + team * 2 * CF::SSTV;  // [2][SSTV] team staging (row parity)
    int32_t *Sc0 = Scall + team * 2 * CF::SSTC;
    int spar = 0;
    const int mq1 = v1.maxq;
    // W1 rows of a batch are contiguous in global memory ([i][c][f]): one bulk copy per batch,
    // prefetched one batch ahead into a double buffer
    auto w1_issue = [&](int r0, int buf) {
        const int nr = n1 - r0 < NR ? n1 - r0 : NR;
        const unsigned bytes = (unsigned)(nr * mq1 * 32);
        mbar_arrive_tx(&wfull[cw * 2 + buf], bytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(W1b + buf * CF::W1D)),
                     "l"(v1.W + (int64_t)r0 * mq1 * 4), "r"(bytes), "r"(smem_u32(&wfull[cw * 2 + buf]))
                     : "memory");
    };
    const int my_first = team * NR;
    int wbuf = 0;
    unsigned wuse[2] = {0, 0};
    if (lane == 0 && my_first < n1 && first < a.n_items) w1_issue(my_first, 0);
    // entry of column (t2, t3) in a row, in units of ni1: t2 + ni2 * t3 (interior: colx)
    int el = colx, nc23 = K * K;
    uint32_t got = 0, rel = 0, Tbase = 0;  // tasks waited for / released, first task of the item
    for (int64_t it = first; it < a.n_items; it += step) {
        const LItem I = ln_item(a, it);
        if (BND) {
            live = colx < COLS && t2c < I.ni2 && t3c < I.ni3;
            el = t2c + I.ni2 * t3c;
            nc23 = I.ni2 * I.ni3;
        }
        const int64_t line_off = a.g.offset(0, I.i2, I.i3) - a.val_base;
        const int colbase = n1 * ((I.jl2 + t2c) + (int)a.g.n[1] * (I.jl3 + t3c));
        for (int r0 = team * NR; r0 < n1; r0 += NTEAM * NR) {
            const int nr = n1 - r0 < NR ? n1 - r0 : NR;
            const int rl = r0 + nr - 1;
            const uint32_t t_hi = Tbase + (uint32_t)((qlo1[rl] + qlen1[rl] - 1 - q0) / 2);
            const uint32_t t_lo = Tbase + (uint32_t)((qlo1[r0] - q0) / 2);
            // this batch's weights: wait for the prefetch, then prefetch the next batch of the team
            twait(&wfull[cw * 2 + wbuf], wuse[wbuf] & 1, pC);
            ++wuse[wbuf];
            const double2 *W1w = (const double2 *)(W1b + wbuf * CF::W1D);  // [row][c][2] double2, row stride mq1
            if (lane == 0) {
                int nxt = r0 + NTEAM * NR;
                bool more = true;
                if (nxt >= n1) { nxt = my_first; more = it + step < a.n_items; }
                if (more) w1_issue(nxt, wbuf ^ 1);
            }
            wbuf ^= 1;
            __syncwarp();
            while (rel < got && rel < t_lo) {
                if (lane == 0) mbar_arrive(&gempty[rel % NTS]);
                ++rel;
            }
            while (got <= t_hi) {
                twait(&gfull[got % NTS], (got / NTS) & 1, pA);
                ++got;
                while (rel < got && rel < t_lo) {
                    if (lane == 0) mbar_arrive(&gempty[rel % NTS]);
                    ++rel;
                }
            }
            __syncwarp();
            double acc[NR][K];
            #pragma unroll
            for (int k = 0; k < NR; ++k)
                #pragma unroll
                for (int t = 0; t < K; ++t) acc[k][t] = 0.0;
            auto slot_of = [&](int q) { return (int)((Tbase * 2 + (uint32_t)(q - q0)) % RING); };
            auto gload = [&](int slot, double &g00, double &g01, double &g10, double &g11) {
                g00 = Gs[(0 * RING + slot) * COLS + colx];
                g01 = Gs[(1 * RING + slot) * COLS + colx];
                g10 = Gs[(2 * RING + slot) * COLS + colx];
                g11 = Gs[(3 * RING + slot) * COLS + colx];
            };
            const bool interior = nr == NR && r0 >= P + 1 && r0 + NR - 1 <= n1 - P - 2;
            if (live && !LDBG(16)) {
                if (interior) {
                    const int slot0 = slot_of(qlo1[r0]);
                    constexpr int UW = 2 * (NR - 1) + 2 * P + 1;
                    #pragma unroll
                    for (int u = 0; u < UW; ++u) {
                        int slot = slot0 + u;
                        if (slot >= RING) slot -= RING;
                        double g00, g01, g10, g11;
                        gload(slot, g00, g01, g10, g11);
                        double2 bb[NP];
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) bb[r] = B1r[slot * NP + r];
                        #pragma unroll
                        for (int k = 0; k < NR; ++k) {
                            if (u >= 2 * k && u <= 2 * k + 2 * P) {
                                const int c = u - 2 * k;
                                const int o0 = (c + 1) / 2;
                                const double2 *wr = W1w + (k * mq1 + c) * 2;
                                const double2 wA = wr[0], wB = wr[1];
                                const double u0 = fma(wA.x, g00, wA.y * g01);
                                const double u1 = fma(wB.x, g10, wB.y * g11);
                                #pragma unroll
                                for (int r = 0; r <= P; ++r)
                                    acc[k][o0 + r] = fma(bb[r].x, u0, fma(bb[r].y, u1, acc[k][o0 + r]));
                            }
                        }
                    }
                } else {
                    #pragma unroll
                    for (int k = 0; k < NR; ++k) {
                        if (k >= nr) break;
                        const int i1 = r0 + k;
                        const int qb = qlo1[i1], nq1 = qlen1[i1], jl1 = jlo1[i1];
                        #pragma unroll 1
                        for (int c = 0; c < nq1; ++c) {
                            const int q = qb + c;
                            const int slot = slot_of(q);
                            const double2 *bp = B1r + slot * NP;
                            const double2 *wr = W1w + (k * mq1 + c) * 2;
                            double g00, g01, g10, g11;
                            gload(slot, g00, g01, g10, g11);
                            const double2 wA = wr[0], wB = wr[1];
                            const double u0 = fma(wA.x, g00, wA.y * g01);
                            const double u1 = fma(wB.x, g10, wB.y * g11);
                            const int off = span1[q] - jl1;
                            dispatch<0, K - NP>(off, [&](auto O) {
                                constexpr int o0 = decltype(O)::value;
                                #pragma unroll
                                for (int r = 0; r <= P; ++r) {
                                    const double2 bq = bp[r];
                                    acc[k][o0 + r] = fma(bq.x, u0, fma(bq.y, u1, acc[k][o0 + r]));
                                }
                            });
                        }
                    }
                }
            }
            {
                const int nb = r0 + NTEAM * NR;
                const int low = nb < n1 ? qlo1[nb] : q_end;
                const uint32_t t_rel = Tbase + (uint32_t)((low - q0) / 2);
                __syncwarp();
                while (rel < t_rel && rel < got) {
                    if (lane == 0) mbar_arrive(&gempty[rel % NTS]);
                    ++rel;
                }
            }
            // write the batch's rows: the team's warps stage their slices of a row in CSR order in the
            // team buffer; one lane of the team's first warp copies the row (contiguous in the CSR)
            // with TMA bulk stores, the <= 1 + 1 unaligned values and <= 3 + 3 unaligned columns at
            // the ends by single lanes; two named barriers per row (team only)
            {
                const int nall = TW * 32;
                #pragma unroll
                for (int k = 0; k < NR; ++k) {
                    if (k >= nr) break;
                    const int i1 = r0 + k;
                    const int ni1 = jlen1[i1];
                    const int64_t dst0 = line_off + (int64_t)nc23 * pref1[i1];
                    const int len = ni1 * nc23;
                    const int hv = (int)dst0 & 1, hc = (int)dst0 & 3;
                    double *Sv = Sv0 + spar * CF::SSTV;
                    int32_t *Sc = Sc0 + spar * CF::SSTC;
                    if (wt == 0 && lane == 0) bulk_wait_read<1>();  // this buffer's copy (two rows ago) is done
                    bar_sync(1 + team, nall);
                    if (live) {
                        double *svl = Sv + hv + ni1 * el;
                        int32_t *scl = Sc + hc + ni1 * el;
                        const int cb = jlo1[i1] + colbase;
                        if (ni1 == K) {
                            #pragma unroll
                            for (int t = 0; t < K; ++t) { svl[t] = acc[k][t]; scl[t] = cb + t; }
                        } else {
                            #pragma unroll
                            for (int t = 0; t < K; ++t)
                                if (t < ni1) { svl[t] = acc[k][t]; scl[t] = cb + t; }
                        }
                    }
                    fence_async_smem();
                    bar_sync(1 + team, nall);
                    if (wt == 0) {
                        const int nbv = (len - hv) & ~1, tv = hv + nbv;
                        const int h4 = min((4 - hc) & 3, len);
                        const int nbc = (len - h4) & ~3, tc = h4 + nbc;
                        double *dv = a.val + dst0;
                        int32_t *dc = a.col + dst0;
                        if (lane == 0) {
                            if (nbv > 0) bulk_s2g(dv + hv, Sv + 2 * hv, (unsigned)nbv * 8u);
                            if (a.col && nbc > 0) bulk_s2g(dc + h4, Sc + hc + h4, (unsigned)nbc * 4u);
                            bulk_commit();
                        } else if (lane == 1) {
                            if (hv) dv[0] = Sv[1];
                        } else if (lane == 2) {
                            if (tv < len) dv[tv] = Sv[hv + tv];
                        } else if (a.col && lane >= 4 && lane < 7) {
                            if (lane - 4 < h4) dc[lane - 4] = Sc[hc + lane - 4];
                        } else if (a.col && lane >= 8 && lane < 12) {
                            if (tc + lane - 8 < len) dc[tc + lane - 8] = Sc[hc + tc + lane - 8];
                        }
                    }
                    spar ^= 1;
                }
            }
        }
        const uint32_t t_end = Tbase + (uint32_t)NTASK;
        while (rel < t_end) {
            if (got <= rel) {
                twait(&gfull[got % NTS], (got / NTS) & 1, pB);
                ++got;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&gempty[rel % NTS]);
            ++rel;
        }
        Tbase = t_end;
    }
    if (lane == 0) bulk_wait<0>();
    prof_out();
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

unsigned long long *g_prof_buf = nullptr;

int num_sms(int dev) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

template <int P, bool BND>
wq_status launch_line_p(wq_plan_s *Pl, const int32_t *lines, int64_t n_lines, double *val, int32_t *col,
                        int64_t val_base, cudaStream_t s) {
    using CF = LnCfg<P, BND>;
    if constexpr (!CF::FITS) {
        wq_set_error("line kernel not configured for this degree");
        return WQ_EINVAL;
    } else {
        if (n_lines <= 0) return WQ_OK;
        LnArgs a;
        a.g.init(Pl);
        for (int l = 0; l < 3; ++l) a.v[l] = Pl->dir[l];
        a.lines = lines;
        a.n_items = n_lines;
        a.cq_b = Pl->cq_b;
        a.val = val;
        a.col = col;
        a.val_base = val_base;
        a.dbg = getenv("WQ_LINE_DBG") ? atoi(getenv("WQ_LINE_DBG")) : 0;
        a.prof = nullptr;
        if (LPROF && getenv("WQ_LINE_PROF")) {  // debug: cycle accounting per warp, read back with wq_debug_prof
            static unsigned long long *buf = nullptr;
            if (!buf) cudaMalloc(&buf, sizeof(unsigned long long) * 148 * 32 * 4);
            cudaMemset(buf, 0, sizeof(unsigned long long) * 148 * 32 * 4);
            a.prof = buf;
            g_prof_buf = buf;
        }
        CUtensorMap m;
        auto fn = encode_fn();
        if (!fn) { wq_set_error("cuTensorMapEncodeTiled unavailable"); return WQ_ECUDA; }
        cuuint64_t dims[4] = {(cuuint64_t)(Pl->dir[0].nq + Pl->c0off), (cuuint64_t)Pl->dir[1].nq,
                              (cuuint64_t)(Pl->cq_e - Pl->cq_b), (cuuint64_t)Pl->ncomp_std};
        cuuint64_t strides[3] = {(cuuint64_t)Pl->cld1 * 8, (cuuint64_t)Pl->cld1 * Pl->dir[1].nq * 8,
                                 (cuuint64_t)Pl->cstride * 8};
        cuuint32_t box[4] = {2, (cuuint32_t)CF::QX, (cuuint32_t)CF::QX, 6};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void *)Pl->coef, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            wq_set_error("cuTensorMapEncodeTiled failed for the coefficient field");
            return WQ_ECUDA;
        }
        const size_t smem = CF::SMEM + CF::d1_bytes(Pl->dir[0].n, Pl->dir[0].nq);
        if (smem > 227 * 1024) {
            wq_set_error("line kernel: direction-1 tables exceed shared memory");
            return WQ_EINVAL;
        }
        cudaFuncSetAttribute(k_line<P, BND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int64_t grid = num_sms(Pl->device);
        if (grid > n_lines) grid = n_lines;
        k_line<P, BND><<<(unsigned)grid, CF::NT, smem, s>>>(m, a);
        wq_count_launches(1);
        return wq_cuda_status(cudaGetLastError(), "line assembly kernel");
    }
}


template <bool BND>
bool fits_line(int p, int64_t n1, int64_t nq1) {
    switch (p) {
    case 2: return LnCfg<2, BND>::FITS && LnCfg<2, BND>::SMEM + LnCfg<2, BND>::d1_bytes(n1, nq1) <= 227 * 1024;
    case 3: return LnCfg<3, BND>::FITS && LnCfg<3, BND>::SMEM + LnCfg<3, BND>::d1_bytes(n1, nq1) <= 227 * 1024;
    case 4: return LnCfg<4, BND>::FITS && LnCfg<4, BND>::SMEM + LnCfg<4, BND>::d1_bytes(n1, nq1) <= 227 * 1024;
    }
    return false;
}

}  // namespace

bool line_supported(const wq_plan_s *P, int matrix, bool bnd) {
    if (matrix != WQ_STIFFNESS || P->d != 3 || !P->need_stiff || P->zlayout) return false;
    if (!encode_fn()) return false;
    for (int l = 0; l < 3; ++l)
        if (P->dir[l].maxq > 3 * P->p + 1) return false;  // a support holding both boundary spans
    return bnd ? fits_line<true>(P->p, P->dir[0].n, P->dir[0].nq) : fits_line<false>(P->p, P->dir[0].n, P->dir[0].nq);
}

wq_status launch_assemble_line(wq_plan_s *P, int matrix, bool bnd, const int32_t *lines, int64_t n_lines, double *val,
                               int32_t *col, int64_t val_base, cudaStream_t s) {
    if (!line_supported(P, matrix, bnd)) {
        wq_set_error("line kernel not available for this plan");
        return WQ_EINVAL;
    }
    switch (P->p * 2 + (bnd ? 1 : 0)) {
    case 4: return launch_line_p<2, false>(P, lines, n_lines, val, col, val_base, s);
    case 5: return launch_line_p<2, true>(P, lines, n_lines, val, col, val_base, s);
    case 6: return launch_line_p<3, false>(P, lines, n_lines, val, col, val_base, s);
    case 7: return launch_line_p<3, true>(P, lines, n_lines, val, col, val_base, s);
    case 8: return launch_line_p<4, false>(P, lines, n_lines, val, col, val_base, s);
    case 9: return launch_line_p<4, true>(P, lines, n_lines, val, col, val_base, s);
    }
    return WQ_EINVAL;
}

// debug only (WQ_LINE_PROF): copy the per-warp cycle accounting of the last line-kernel launch
extern "C" int wq_debug_prof(unsigned long long *host, int n) {
    if (!g_prof_buf) return -1;
    cudaDeviceSynchronize();
    return (int)cudaMemcpy(host, g_prof_buf, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
}
