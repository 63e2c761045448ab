// wq_assemble_ws.cu -- step 7, warp-specialised persistent row-line kernel
// (WQ_KERNEL_WS), d = 3, compile-time degree P.
//
// Same arithmetic as the row-line kernel of wq_assemble_tile.cu (Eq.
// sumfactorization P:837 / Alg. 3 P:859-870 re-organised so that the rows of
// a line (i2, i3) share every stage but the last; stiffness terms merged into
// 6 chains through modes 3 and 2, 4 arrays G[b1][a1] into mode 1; DESIGN.md
// §6), scheduled as a pipeline of three warp roles inside one persistent CTA
// per SM:
//
//   warp 0        TMA: streams the coefficient field of the current line, one
//                 q3-plane box (NQSB q1 points x nq2 x NCOMP) per stage, into a
//                 ring of NSTAGE shared-memory buffers (mbarrier full/empty).
//   NWP warps     stage 3 (contract q3, test weights of directions 2, 3 pushed
//                 pointwise) and stage 2 (contract q2) for sub-batches of NQS
//                 points q1, software-pipelined: stage 2 of sub-batch S and
//                 stage 3 of S+1 run between two named barriers.  Results go
//                 to a ring of NSB sub-batch slots of G (mbarrier gfull/gempty).
//   NWC warps     stage 1 (contract q1) for the rows of the line: teams of TW
//                 warps cover the COLS = K x T3C columns (t2, t3) of a row, each
//                 lane NR rows in registers; values + columns are staged per
//                 warp in shared memory and written with TMA bulk stores.
//
// The sequence of (line, t3-chunk) items of a CTA is one continuous stream, so
// the pipeline does not drain between lines.  (a, b) = (test, trial)
// derivative order (reading R3); directions 1..3 are indices 0..2.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include "wq_rows.cuh"
#include "wq_dev.cuh"

using namespace wqdev;

namespace {

struct WsPar {
    int t3c, nr, nteam, nwp, nqs, nsb, nstage;
};

// hand-tuned per (P, matrix); see DESIGN.md §6 (t3c = 0: kernel not instantiated)
__host__ __device__ constexpr WsPar ws_par(int p, bool stiff) {
    if (stiff) {
        switch (p) {
        case 1: return {3, 4, 8, 4, 8, 16, 6};
        case 2: return {5, 4, 8, 7, 8, 12, 6};
        case 3: return {7, 4, 4, 7, 6, 11, 6};
        case 4: return {9, 3, 2, 6, 4, 9, 6};
        default: return {0, 0, 0, 0, 0, 0, 0};
        }
    }
    switch (p) {
    case 1: return {3, 6, 8, 3, 16, 10, 6};
    case 2: return {5, 6, 8, 3, 16, 8, 6};
    case 3: return {7, 6, 4, 4, 12, 8, 6};
    case 4: return {9, 4, 2, 4, 12, 6, 6};
    default: return {0, 0, 0, 0, 0, 0, 0};
    }
}

template <int P, bool STIFF>
struct WsCfg {
    static constexpr WsPar W = ws_par(P, STIFF);
    static constexpr bool ENABLED = W.t3c > 0;
    static constexpr int K = 2 * P + 1;   // max #I
    static constexpr int QI = 2 * P + 1;  // #Q of an interior row
    static constexpr int QB = 3 * P + 1;  // max #Q (supports with one boundary span)
    static constexpr int NP = P + 1;
    static constexpr int T3C = ENABLED ? W.t3c : 1;
    static constexpr int NCH = (K + T3C - 1) / T3C;
    static constexpr int COLS = K * T3C;
    static constexpr int TW = (COLS + 31) / 32;  // consumer warps per team
    static constexpr int NR = ENABLED ? W.nr : 1;
    static constexpr int NTEAM = ENABLED ? W.nteam : 1;
    static constexpr int NWC = TW * NTEAM;
    static constexpr int NWP = ENABLED ? W.nwp : 1;
    static constexpr int NTP = 32 * NWP;
    static constexpr int NT = 32 * (1 + NWP + NWC);
    static constexpr int NQS = ENABLED ? W.nqs : 2;
    // TMA box width: the box starts at the even q1 at or below the sub-batch (TMA needs a 16-B
    // aligned start in the innermost dimension), so it spans NQS + 1 points rounded up to even
    static constexpr int NQSB = (NQS + 2) & ~1;
    static constexpr int NSB = ENABLED ? W.nsb : 2;
    static constexpr int RING = NSB * NQS;
    static constexpr int NSTAGE = ENABLED ? W.nstage : 2;
    static constexpr int NM = STIFF ? 3 : 1;     // trial-derivative directions m (stage-3 fibres)
    static constexpr int NA = STIFF ? 2 : 1;     // a1 variants (stage-2 fibres)
    static constexpr int NY = STIFF ? 6 : 1;     // chains through stage 3
    static constexpr int NG = STIFF ? 4 : 1;     // G arrays
    static constexpr int NCOMP = STIFF ? 6 : 1;  // coefficient components
    // producer work items per sub-batch: stage-2 fibres (t3l, a1, q1s), then stage-3 fibres (q1s, c2, m)
    static constexpr int N2 = T3C * NA * NQS;
    static constexpr int N3MAX = NQS * NM * QB;
    static constexpr int IPT = (N2 + N3MAX + NTP - 1) / NTP;  // items per producer thread
    static constexpr int FPT = (N3MAX + NTP - 1) / NTP < IPT ? (N3MAX + NTP - 1) / NTP : IPT;  // stage-3 items per thread
    static constexpr int SSTV = 32 * K + 2;  // staging doubles per warp buffer
    static constexpr int SSTC = 32 * K + 4;  // staging int32 per warp buffer
    // shared memory layout (bytes, 128-B aligned regions)
    __host__ __device__ static constexpr size_t al(size_t x) { return (x + 127) & ~(size_t)127; }
    static constexpr size_t STAGE_BYTES = al((size_t)NCOMP * QB * NQSB * 8);
    static constexpr size_t O_BAR = 0;
    static constexpr size_t O_CST = al(8 * (2 * NSTAGE + 2 * NSB));
    static constexpr size_t O_Y = O_CST + NSTAGE * STAGE_BYTES;
    static constexpr size_t Y_BUF = (size_t)NQS * NY * QB * T3C;  // doubles per Y buffer
    static constexpr size_t O_G = al(O_Y + 2 * Y_BUF * 8);
    static constexpr size_t O_B1 = al(O_G + (size_t)NG * RING * COLS * 8);
    static constexpr size_t O_TAB = al(O_B1 + (size_t)RING * NP * 16);
    static constexpr size_t TAB_D2 = 2 * (size_t)QB * NP + 2 * (size_t)QB * NP + 2 * QB + 2 * QB;  // double2 per buffer
    static constexpr size_t O_W1 = al(O_TAB + 2 * TAB_D2 * 16);
    static constexpr size_t O_SV = al(O_W1 + (size_t)NWC * NR * QB * 2 * 16);
    static constexpr size_t O_SC = al(O_SV + (size_t)NWC * 2 * SSTV * 8);
    static constexpr size_t SMEM = al(O_SC + (size_t)NWC * 2 * SSTC * 4);
    static constexpr bool FITS = ENABLED && SMEM <= 227 * 1024 && NT <= 1024;
};

struct WsArgs {
    RowGeo g;
    DirView v[3];
    int64_t cq_b;
    int comp0;  // first coefficient component loaded (mass: index of c)
    double *val;
    int32_t *col;
    int64_t val_base;
    int64_t plane_lo;  // first slab plane (relative) of this launch
    int64_t n_items;   // lines * NCH
    int dbg;           // debug bisection mask (WQ_WS_DBG), 0 in production
};

// per-item (line, t3 chunk) geometry
struct Item {
    int i2, i3, ql2, nq2, ql3, nq3, jl2, jl3, ni2, ni3, t3a, nt3;
    bool int2, int3;
};

template <int P, int NCH, int T3C>
__device__ __forceinline__ Item get_item(const WsArgs &a, int64_t it) {
    Item I;
    const int chunk = (int)(it % NCH);
    const int64_t line = it / NCH;
    const int n2 = (int)a.g.n[1], n3 = (int)a.g.n[2];
    I.i2 = (int)(line % n2);
    I.i3 = (int)(a.g.slab_b + a.plane_lo + line / n2);
    const DirView &v2 = a.v[1], &v3 = a.v[2];
    I.ql2 = v2.qlo[I.i2];
    I.nq2 = v2.qlen[I.i2];
    I.jl2 = v2.jlo[I.i2];
    I.ni2 = v2.jlen[I.i2];
    I.ql3 = v3.qlo[I.i3];
    I.nq3 = v3.qlen[I.i3];
    I.jl3 = v3.jlo[I.i3];
    I.ni3 = v3.jlen[I.i3];
    I.t3a = chunk * T3C;
    I.nt3 = I.ni3 - I.t3a < T3C ? I.ni3 - I.t3a : T3C;
    I.int2 = I.nq2 == 2 * P + 1 && I.i2 >= P + 1 && I.i2 <= n2 - P - 2;
    I.int3 = I.nq3 == 2 * P + 1 && I.i3 >= P + 1 && I.i3 <= n3 - P - 2;
    return I;
}

template <int P, bool STIFF>
__global__ void __launch_bounds__(WsCfg<P, STIFF>::NT, 1)
    k_ws(const __grid_constant__ CUtensorMap tm_s, const __grid_constant__ CUtensorMap tm_b, WsArgs a) {
    using CF = WsCfg<P, STIFF>;
    constexpr int K = CF::K, QI = CF::QI, QB = CF::QB, NP = CF::NP, T3C = CF::T3C, NCH = CF::NCH;
    constexpr int COLS = CF::COLS, TW = CF::TW, NR = CF::NR, NTEAM = CF::NTEAM, NWP = CF::NWP, NTP = CF::NTP;
    constexpr int NQS = CF::NQS, NQSB = CF::NQSB, NSB = CF::NSB, RING = CF::RING, NSTAGE = CF::NSTAGE;
    constexpr int NM = CF::NM, NA = CF::NA, NY = CF::NY, NG = CF::NG, NCOMP = CF::NCOMP;
    constexpr int N2 = CF::N2, IPT = CF::IPT, FPT = CF::FPT;
    constexpr int BS = wq_bstride(P);
    extern __shared__ __align__(128) unsigned char smb[];
    uint64_t *full = (uint64_t *)(smb + CF::O_BAR);
    uint64_t *empty = full + NSTAGE;
    uint64_t *gfull = empty + NSTAGE;
    uint64_t *gempty = gfull + NSB;
    double *Cst = (double *)(smb + CF::O_CST);
    double *Ys = (double *)(smb + CF::O_Y);
    double *Gs = (double *)(smb + CF::O_G);
    double2 *B1r = (double2 *)(smb + CF::O_B1);
    double2 *Tab = (double2 *)(smb + CF::O_TAB);
    double2 *W1all = (double2 *)(smb + CF::O_W1);
    double *Svall = (double *)(smb + CF::O_SV);
    int32_t *Scall = (int32_t *)(smb + CF::O_SC);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const DirView &v1 = a.v[0];
    const int n1 = (int)a.g.n[0];
    const int q0 = v1.qlo[0];
    const int q_end = v1.qlo[n1 - 1] + v1.qlen[n1 - 1];
    const int NSUB = (q_end - q0 + NQS - 1) / NQS;  // sub-batches per item (same for every line)
    const int64_t first = blockIdx.x, step = gridDim.x;

    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NWP); }
        for (int s = 0; s < NSB; ++s) { mbar_init(&gfull[s], NTP); mbar_init(&gempty[s], CF::NWC); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ======================================================== TMA producer
        if (lane == 0) {
            int st = 0;
            unsigned ph = 0;
            for (int64_t it = first; it < a.n_items; it += step) {
                const Item I = get_item<P, NCH, T3C>(a, it);
                const bool small = I.nq2 <= QI;
                const void *tm = small ? (const void *)&tm_s : (const void *)&tm_b;
                const unsigned bytes = (unsigned)(NCOMP * (small ? QI : QB) * NQSB * 8);
                const int z0 = (int)(I.ql3 - a.cq_b);
                for (int s = 0; s < NSUB; ++s)
                    for (int c3 = 0; c3 < I.nq3; ++c3) {
                        mbar_wait(&empty[st], ph ^ 1);
                        if (a.dbg & 1) { mbar_arrive(&full[st]); if (++st == NSTAGE) { st = 0; ph ^= 1; } continue; }
                        mbar_arrive_tx(&full[st], bytes);
                        tma_load_4d(Cst + st * (CF::STAGE_BYTES / 8), tm, &full[st], (q0 + s * NQS + 1) & ~1, I.ql2, z0 + c3,
                                    a.comp0);
                        if (++st == NSTAGE) { st = 0; ph ^= 1; }
                    }
            }
        }
        return;
    }

    if (warp <= NWP) {
        // ======================================================== stage 3 / stage 2 producers
        const int ptid = tid - 32;
        int st = 0;
        unsigned ph = 0;
        // stage-3 accumulators of the thread's fibres for the sub-batch in flight
        double y0[FPT][T3C], y1[FPT][T3C];
        // the flat stream: sub-batch S of item k = S / NSUB; stage 3 of S+1 overlaps stage 2 of S
        int64_t it3 = first;  // item of the next stage-3 sub-batch
        int s3 = 0;           // its sub-batch index
        Item I3 = get_item<P, NCH, T3C>(a, it3), I2 = I3;
        int tb3 = 0, tb2 = 0;  // table buffers
        auto tabs = [&](int b) { return Tab + b * CF::TAB_D2; };
        // load the direction-2/3 tables of an item into buffer b (producer threads)
        auto load_tabs = [&](const Item &I, int b) {
            double2 *B2s = tabs(b), *B3s = B2s + QB * NP, *W2s = B3s + QB * NP, *W3s = W2s + 2 * QB;
            const DirView &v2 = a.v[1], &v3 = a.v[2];
            for (int x = ptid; x < QB * NP; x += NTP) {
                const int c = x / NP, r = x % NP;
                B2s[x] = c < I.nq2 ? __ldg((const double2 *)(v2.B + (int64_t)(I.ql2 + c) * BS) + r) : make_double2(0.0, 0.0);
                B3s[x] = c < I.nq3 ? __ldg((const double2 *)(v3.B + (int64_t)(I.ql3 + c) * BS) + r) : make_double2(0.0, 0.0);
            }
            for (int x = ptid; x < QB * 2; x += NTP) {
                const int c = x / 2;
                W2s[x] = c < I.nq2 ? __ldg((const double2 *)(v2.W + ((int64_t)I.i2 * v2.maxq + c) * 4) + (x & 1))
                                   : make_double2(0.0, 0.0);
                W3s[x] = c < I.nq3 ? __ldg((const double2 *)(v3.W + ((int64_t)I.i3 * v3.maxq + c) * 4) + (x & 1))
                                   : make_double2(0.0, 0.0);
            }
        };

        // ---- stage 3 of one sub-batch (item I, sub-batch s) into Y buffer yb
        auto stage3 = [&](const Item &I, int s, int tb, int yb) {
            const double2 *B3s = tabs(tb) + QB * NP, *W2s = B3s + QB * NP, *W3s = W2s + 2 * QB;
            const int nq2 = I.nq2, nq3 = I.nq3;
            const int n3 = NQS * NM * nq2;
            const int cs = (I.nq2 <= QI ? QI : QB) * NQSB;  // component stride in a stage buffer
            const int sh = (q0 + s * NQS + 1) & 1;          // point q1 is column q1 + 1; box starts at an even column
            int fq[FPT], fc2[FPT], fm[FPT];
            bool fv[FPT];
            double2 w2v[FPT];
            #pragma unroll
            for (int k = 0; k < FPT; ++k) {
                // stage-3 items of this thread: flat items ptid + j*NTP at or beyond N2
                int cnt = 0, f = -1;
                #pragma unroll
                for (int j = 0; j < IPT; ++j) {
                    const int itm = ptid + j * NTP;
                    if (itm >= N2 && itm < N2 + n3) {
                        if (cnt == k) f = itm - N2;
                        ++cnt;
                    }
                }
                fv[k] = f >= 0;
                const int ff = f >= 0 ? f : 0;
                fq[k] = ff % NQS;
                fc2[k] = (ff / NQS) % nq2;
                fm[k] = STIFF ? ff / (NQS * nq2) : 0;
                w2v[k] = W2s[fc2[k] * 2 + (STIFF && fm[k] == 1 ? 1 : 0)];  // (w2^(0,b2), w2^(1,b2))
                #pragma unroll
                for (int t = 0; t < T3C; ++t) { y0[k][t] = 0.0; y1[k][t] = 0.0; }
            }
            auto plane = [&](int c3, auto O) {  // O: staircase offset (compile time) or INT_MIN (runtime)
                mbar_wait(&full[st], ph);
                const double *buf = Cst + st * (CF::STAGE_BYTES / 8);
                #pragma unroll
                for (int k = 0; k < FPT; ++k) {
                    if (!fv[k]) continue;
                    const int m = fm[k];
                    const int b3 = STIFF && m == 2 ? 1 : 0;
                    const int ka = STIFF ? m : 0;
                    const int kb = m == 0 ? 1 : (m == 1 ? 3 : 4);
                    const int kc = m == 0 ? 2 : (m == 1 ? 4 : 5);
                    const double *cb0 = buf + fc2[k] * NQSB + fq[k] + sh;
                    const double ca = cb0[ka * cs];
                    const double cbv = STIFF ? cb0[kb * cs] : 0.0;
                    const double ccv = STIFF ? cb0[kc * cs] : 0.0;
                    const double2 w3v = W3s[c3 * 2 + b3];  // (w3^(0,b3), w3^(1,b3))
                    const double *bp = (const double *)(B3s + c3 * NP) + b3;
                    double h1, h0;
                    if (STIFF) {
                        h1 = w2v[k].x * w3v.x * ca;                             // l = 0      (a1 = 1)
                        h0 = fma(w2v[k].y * w3v.x, cbv, w2v[k].x * w3v.y * ccv);  // l = 1, 2  (a1 = 0)
                    } else {
                        h0 = w2v[k].x * w3v.x * ca;
                        h1 = 0.0;
                    }
                    auto acc = [&](auto OO) {
                        constexpr int o0 = decltype(OO)::value;
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) {
                            const int t = o0 + r;
                            if (t >= 0 && t < T3C) {
                                const double bv = bp[2 * r];
                                y0[k][t] = fma(bv, h0, y0[k][t]);
                                if (STIFF) y1[k][t] = fma(bv, h1, y1[k][t]);
                            }
                        }
                    };
                    if constexpr (decltype(O)::value != -1000) {
                        acc(O);
                    } else {
                        const int off = a.v[2].span[I.ql3 + c3] - I.jl3 - I.t3a;
                        if (NCH == 1) dispatch<0, K - NP>(off, acc);
                        else dispatch<-P, T3C - 1>(off, acc);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == NSTAGE) { st = 0; ph ^= 1; }
            };
            if (NCH == 1 && I.int3) {
                unroll<QI>([&](auto C3) {
                    constexpr int c3 = decltype(C3)::value;
                    plane(c3, std::integral_constant<int, (c3 + 1) / 2>{});
                });
            } else {
                #pragma unroll 1
                for (int c3 = 0; c3 < nq3; ++c3) plane(c3, std::integral_constant<int, -1000>{});
            }
            // Y[yb][q1s][chain][c2][t3l], chain = m * NA + a1 (a1 = 0: y0, a1 = 1: y1)
            double *Y = Ys + yb * CF::Y_BUF;
            #pragma unroll
            for (int k = 0; k < FPT; ++k) {
                if (!fv[k]) continue;
                double *Y0 = Y + ((fq[k] * NY + fm[k] * NA + 0) * QB + fc2[k]) * T3C;
                #pragma unroll
                for (int t = 0; t < T3C; ++t) Y0[t] = y0[k][t];
                if (STIFF) {
                    double *Y1 = Y0 + QB * T3C;
                    #pragma unroll
                    for (int t = 0; t < T3C; ++t) Y1[t] = y1[k][t];
                }
            }
        };

        // ---- stage 2 of one sub-batch (item I, sub-batch s, global slot sb) from Y buffer yb
        auto stage2 = [&](const Item &I, int s, int tb, int yb, uint32_t S) {
            const double2 *B2s = tabs(tb);
            const int qs = q0 + s * NQS;
            const int nqs = q_end - qs < NQS ? q_end - qs : NQS;
            const int slot_sb = (int)(S % NSB);
            // the slot's previous use must have been released by every consumer warp
            mbar_wait(&gempty[slot_sb], ((S / NSB) & 1) ^ 1);
            const double *Y = Ys + yb * CF::Y_BUF;
            #pragma unroll
            for (int j = 0; j < IPT; ++j) {
                const int f = ptid + j * NTP;
                if (f >= N2) break;
                const int t3l = f % T3C;
                const int rest = f / T3C;
                const int a1 = STIFF ? rest % NA : 0;
                const int q1s = rest / NA;
                if (q1s >= nqs) continue;
                double g0[K], g1[K];
                #pragma unroll
                for (int t = 0; t < K; ++t) { g0[t] = 0.0; g1[t] = 0.0; }
                const double *Yb0 = Y + ((q1s * NY + 0 * NA + a1) * QB) * T3C + t3l;  // m = 0 (mass: the chain)
                const double *Yb1 = Y + ((q1s * NY + 1 * NA + a1) * QB) * T3C + t3l;  // m = 1
                const double *Yb2 = Y + ((q1s * NY + 2 * NA + a1) * QB) * T3C + t3l;  // m = 2
                auto point2 = [&](int c2, auto O) {
                    constexpr int o0 = decltype(O)::value;
                    const double2 *bp = B2s + c2 * NP;
                    if (STIFF) {
                        const double ya = Yb0[c2 * T3C], yb_ = Yb1[c2 * T3C], yc = Yb2[c2 * T3C];
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) {
                            const double2 b = bp[r];
                            g1[o0 + r] = fma(b.x, ya, g1[o0 + r]);                 // b1 = 1: m = 0
                            g0[o0 + r] = fma(b.y, yb_, fma(b.x, yc, g0[o0 + r]));  // b1 = 0: m = 1, 2
                        }
                    } else {
                        const double y = Yb0[c2 * T3C];
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) g0[o0 + r] = fma(bp[r].x, y, g0[o0 + r]);
                    }
                };
                if (t3l < I.nt3) {
                    if (I.int2) {
                        unroll<QI>([&](auto C2) {
                            constexpr int c2 = decltype(C2)::value;
                            point2(c2, std::integral_constant<int, (c2 + 1) / 2>{});
                        });
                    } else {
                        for (int c2 = 0; c2 < I.nq2; ++c2) {
                            const int off = a.v[1].span[I.ql2 + c2] - I.jl2;
                            dispatch<0, K - NP>(off, [&](auto O) { point2(c2, O); });
                        }
                    }
                }
                const int slot = slot_sb * NQS + q1s;
                double *G0 = Gs + ((0 * NA + a1) * RING + slot) * COLS + K * t3l;  // b1 = 0
                #pragma unroll
                for (int t = 0; t < K; ++t) G0[t] = g0[t];
                if (STIFF) {
                    double *G1 = Gs + ((1 * NA + a1) * RING + slot) * COLS + K * t3l;  // b1 = 1
                    #pragma unroll
                    for (int t = 0; t < K; ++t) G1[t] = g1[t];
                }
            }
            // direction-1 basis pairs of the sub-batch's points
            for (int x = ptid; x < nqs * NP; x += NTP) {
                const int q1s = x / NP, r = x % NP;
                B1r[(slot_sb * NQS + q1s) * NP + r] = __ldg((const double2 *)(a.v[0].B + (int64_t)(qs + q1s) * BS) + r);
            }
            mbar_arrive(&gfull[slot_sb]);
        };

        // prologue: tables of the first item, stage 3 of sub-batch 0
        if (it3 < a.n_items) {
            load_tabs(I3, 0);
            bar_sync(1, NTP);
            stage3(I3, 0, 0, 0);
        }
        bar_sync(1, NTP);
        uint32_t S = 0;
        for (int64_t it2 = first; it2 < a.n_items; it2 += step) {
            I2 = get_item<P, NCH, T3C>(a, it2);
            for (int s2 = 0; s2 < NSUB; ++s2, ++S) {
                // next stage-3 sub-batch
                int s3n = s2 + 1;
                int64_t it3n = it2;
                if (s3n == NSUB) { s3n = 0; it3n = it2 + step; }
                const bool have3 = it3n < a.n_items;
                if (have3 && s3n == 0) {
                    tb3 ^= 1;
                    I3 = get_item<P, NCH, T3C>(a, it3n);
                    load_tabs(I3, tb3);
                    bar_sync(1, NTP);
                }
                if (a.dbg & 8) { mbar_wait(&gempty[S % NSB], ((S / NSB) & 1) ^ 1); mbar_arrive(&gfull[S % NSB]); }
                else stage2(I2, s2, tb2, (int)(S & 1), S);
                if (have3) stage3(I3, s3n, tb3, (int)((S + 1) & 1));
                bar_sync(1, NTP);
                if (have3 && s3n == 0) tb2 = tb3;
            }
        }
        (void)s3;
        return;
    }

    // ============================================================ stage 1 consumers
    const int cw = warp - 1 - NWP;
    const int team = cw / TW, wt = cw % TW;
    const int colx = wt * 32 + lane;
    const int t2c = colx % K, t3c = colx / K;
    double2 *W1w = W1all + cw * (NR * QB * 2);
    double *Sv = Svall + cw * 2 * CF::SSTV;
    int32_t *Sc = Scall + cw * 2 * CF::SSTC;
    const int *__restrict__ qlo1 = v1.qlo, *__restrict__ qlen1 = v1.qlen, *__restrict__ jlo1 = v1.jlo;
    const int *__restrict__ jlen1 = v1.jlen, *__restrict__ span1 = v1.span;
    const int64_t *__restrict__ pref1 = a.g.pref[0];
    const int mq1 = v1.maxq;
    uint32_t got = 0, rel = 0, Sbase = 0;
    int sbuf = 0;
    for (int64_t it = first; it < a.n_items; it += step) {
        const Item I = get_item<P, NCH, T3C>(a, it);
        const bool live = colx < COLS && t2c < I.ni2 && t3c < I.nt3;
        const int el = t2c + I.ni2 * t3c;  // entry of (t2, t3l) in units of ni1 within the row chunk
        const unsigned lm = __ballot_sync(0xffffffffu, live);
        const int e_lo = lm ? __shfl_sync(0xffffffffu, el, __ffs(lm) - 1) : 0;
        const int e_hi = lm ? __shfl_sync(0xffffffffu, el, 31 - __clz(lm)) + 1 : 0;
        const int64_t line_off = a.g.offset(0, I.i2, I.i3) - a.val_base;
        const int colbase = n1 * ((I.jl2 + t2c) + (int)a.g.n[1] * (I.jl3 + I.t3a + t3c));
        for (int r0 = team * NR; r0 < n1; r0 += NTEAM * NR) {
            const int nr = n1 - r0 < NR ? n1 - r0 : NR;
            const int rl = r0 + nr - 1;
            const uint32_t s_hi = Sbase + (uint32_t)((qlo1[rl] + qlen1[rl] - 1 - q0) / NQS);
            // row weights of the batch -> warp-private shared memory
            for (int x = lane; x < NR * QB * 2; x += 32) {
                const int b = x / (QB * 2), c = (x / 2) % QB, i1 = r0 + b;
                W1w[x] = (b < nr && c < qlen1[i1]) ? __ldg((const double2 *)(v1.W + ((int64_t)i1 * mq1 + c) * 4) + (x & 1))
                                                  : make_double2(0.0, 0.0);
            }
            // wait for the batch's sub-batches; the ones below its window (needed only by other
            // teams) are released as soon as they have been waited for, so that a warp never holds
            // more than its own window while it waits (no cross-team deadlock on the ring)
            const uint32_t s_lo = Sbase + (uint32_t)((qlo1[r0] - q0) / NQS);
            __syncwarp();
            while (rel < got && rel < s_lo) {
                if (lane == 0) mbar_arrive(&gempty[rel % NSB]);
                ++rel;
            }
            while (got <= s_hi) {
                mbar_wait(&gfull[got % NSB], (got / NSB) & 1);
                ++got;
                while (rel < got && rel < s_lo) {
                    if (lane == 0) mbar_arrive(&gempty[rel % NSB]);
                    ++rel;
                }
            }
            __syncwarp();
            double acc[NR][K];
            #pragma unroll
            for (int k = 0; k < NR; ++k)
                #pragma unroll
                for (int t = 0; t < K; ++t) acc[k][t] = 0.0;
            auto slot_of = [&](int q) { return (int)((Sbase * NQS + (uint32_t)(q - q0)) % RING); };
            auto gload = [&](int slot, double &g00, double &g01, double &g10, double &g11) {
                g00 = Gs[((0 * NA + 0) * RING + slot) * COLS + colx];
                if (STIFF) {
                    g01 = Gs[((0 * NA + 1) * RING + slot) * COLS + colx];
                    g10 = Gs[((1 * NA + 0) * RING + slot) * COLS + colx];
                    g11 = Gs[((1 * NA + 1) * RING + slot) * COLS + colx];
                }
            };
            const bool interior = nr == NR && r0 >= P + 1 && r0 + NR - 1 <= n1 - P - 2;
            if (live && !(a.dbg & 16)) {
                if (interior) {
                    // rows of the batch have the interior pattern: 2P+1 points, consecutive rows
                    // shifted by 2 points, staircase offset (c+1)/2
                    const int slot0 = slot_of(qlo1[r0]);
                    constexpr int UW = 2 * (NR - 1) + 2 * P + 1;
                    #pragma unroll
                    for (int u = 0; u < UW; ++u) {
                        int slot = slot0 + u;
                        if (slot >= RING) slot -= RING;
                        double g00, g01 = 0.0, g10 = 0.0, g11 = 0.0;
                        gload(slot, g00, g01, g10, g11);
                        double2 bb[NP];
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) bb[r] = B1r[slot * NP + r];
                        #pragma unroll
                        for (int k = 0; k < NR; ++k) {
                            if (u >= 2 * k && u <= 2 * k + 2 * P) {
                                const int c = u - 2 * k;
                                const int o0 = (c + 1) / 2;
                                const double2 *wr = W1w + (k * QB + c) * 2;
                                if (STIFF) {
                                    const double2 wA = wr[0], wB = wr[1];
                                    const double u0 = fma(wA.x, g00, wA.y * g01);
                                    const double u1 = fma(wB.x, g10, wB.y * g11);
                                    #pragma unroll
                                    for (int r = 0; r <= P; ++r)
                                        acc[k][o0 + r] = fma(bb[r].x, u0, fma(bb[r].y, u1, acc[k][o0 + r]));
                                } else {
                                    const double u0 = wr[0].x * g00;
                                    #pragma unroll
                                    for (int r = 0; r <= P; ++r) acc[k][o0 + r] = fma(bb[r].x, u0, acc[k][o0 + r]);
                                }
                            }
                        }
                    }
                } else {
                    #pragma unroll
                    for (int k = 0; k < NR; ++k) {
                        if (k >= nr) break;
                        const int i1 = r0 + k;
                        const int qb = qlo1[i1], nq1 = qlen1[i1], jl1 = jlo1[i1];
                        for (int c = 0; c < nq1; ++c) {
                            const int q = qb + c;
                            const int slot = slot_of(q);
                            const double2 *bp = B1r + slot * NP;
                            const double2 *wr = W1w + (k * QB + c) * 2;
                            double g00, g01 = 0.0, g10 = 0.0, g11 = 0.0;
                            gload(slot, g00, g01, g10, g11);
                            double u0, u1 = 0.0;
                            if (STIFF) {
                                const double2 wA = wr[0], wB = wr[1];
                                u0 = fma(wA.x, g00, wA.y * g01);
                                u1 = fma(wB.x, g10, wB.y * g11);
                            } else {
                                u0 = wr[0].x * g00;
                            }
                            const int off = span1[q] - jl1;
                            dispatch<0, K - NP>(off, [&](auto O) {
                                constexpr int o0 = decltype(O)::value;
                                #pragma unroll
                                for (int r = 0; r <= P; ++r) {
                                    const double2 b = bp[r];
                                    acc[k][o0 + r] = STIFF ? fma(b.x, u0, fma(b.y, u1, acc[k][o0 + r]))
                                                           : fma(b.x, u0, acc[k][o0 + r]);
                                }
                            });
                        }
                    }
                }
            }
            // release the sub-batches that no later batch of this team needs
            {
                const int nb = r0 + NTEAM * NR;
                const int low = nb < n1 ? qlo1[nb] : q_end;
                const uint32_t s_rel = Sbase + (uint32_t)((low - q0) / NQS);
                __syncwarp();
                while (rel < s_rel && rel < got) {
                    if (lane == 0) mbar_arrive(&gempty[rel % NSB]);
                    ++rel;
                }
            }
            // write the batch's rows: stage in CSR order, TMA bulk copy of the warp's segment
            #pragma unroll
            for (int k = 0; k < NR; ++k) {
                if (k >= nr) break;
                const int i1 = r0 + k;
                const int ni1 = jlen1[i1];
                const int64_t goff = line_off + (int64_t)(I.ni2 * I.ni3) * pref1[i1] + (int64_t)ni1 * I.ni2 * I.t3a;
                const int64_t dst0 = goff + (int64_t)ni1 * e_lo;  // first entry of the warp segment
                const int len = ni1 * (e_hi - e_lo);
                const int hv = (int)(dst0 & 1), hc = (int)(dst0 & 3);
                double *sv = Sv + sbuf * CF::SSTV + hv;
                int32_t *sc = Sc + sbuf * CF::SSTC + hc;
                if (lane == 0) bulk_wait_read<1>();  // the buffer's previous copy has read shared memory
                __syncwarp();
                if (live) {
                    const int e0 = ni1 * (el - e_lo);
                    const int cb = jlo1[i1] + colbase;
                    #pragma unroll
                    for (int t = 0; t < K; ++t)
                        if (t < ni1) {
                            sv[e0 + t] = acc[k][t];
                            sc[e0 + t] = cb + t;
                        }
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0 && len > 0) {
                    double *dv = a.val + dst0;
                    const int nbv = (len - hv) & ~1;
                    if (hv) dv[0] = sv[0];
                    if (nbv > 0 && !(a.dbg & 2)) bulk_s2g(dv + hv, sv + hv, (unsigned)nbv * 8u);
                    for (int e = hv + nbv; e < len; ++e) dv[e] = sv[e];
                    if (a.col) {
                        int32_t *dc = a.col + dst0;
                        const int h4 = (4 - hc) & 3;
                        const int hcn = h4 < len ? h4 : len;
                        const int nbc = (len - hcn) & ~3;
                        for (int e = 0; e < hcn; ++e) dc[e] = sc[e];
                        if (nbc > 0 && !(a.dbg & 2)) bulk_s2g(dc + hcn, sc + hcn, (unsigned)nbc * 4u);
                        for (int e = hcn + nbc; e < len; ++e) dc[e] = sc[e];
                    }
                    bulk_commit();
                }
                sbuf ^= 1;
            }
        }
        // release everything left of this item (waiting for each first keeps the phases in order)
        const uint32_t s_end = Sbase + (uint32_t)NSUB;
        while (rel < s_end) {
            if (got <= rel) {
                mbar_wait(&gfull[got % NSB], (got / NSB) & 1);
                ++got;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&gempty[rel % NSB]);
            ++rel;
        }
        Sbase = s_end;
    }
    if (lane == 0) bulk_wait<0>();
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

// coefficient field as a 4D tensor (q1, q2, q3 - cq_b, comp), q1 padded to cld1
bool make_map(CUtensorMap *m, const wq_plan_s *Pl, int box_q1, int box_q2, int box_comp) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)(Pl->dir[0].nq + Pl->c0off), (cuuint64_t)Pl->dir[1].nq, (cuuint64_t)(Pl->cq_e - Pl->cq_b),
                          (cuuint64_t)Pl->ncomp_std};
    cuuint64_t strides[3] = {(cuuint64_t)Pl->cld1 * 8, (cuuint64_t)Pl->cld1 * Pl->dir[1].nq * 8,
                             (cuuint64_t)Pl->cstride * 8};
    cuuint32_t box[4] = {(cuuint32_t)box_q1, (cuuint32_t)box_q2, 1, (cuuint32_t)box_comp};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void *)Pl->coef, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int num_sms(int dev) {
    static int cached[64] = {0};
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) cudaDeviceGetAttribute(&cached[dev], cudaDevAttrMultiProcessorCount, dev);
    return cached[dev];
}

template <int P, bool STIFF>
wq_status launch_ws_p(wq_plan_s *Pl, double *val, int32_t *col, int64_t pl_lo, int64_t pl_hi, int64_t val_base,
                      cudaStream_t s) {
    using CF = WsCfg<P, STIFF>;
    if constexpr (!CF::FITS) {
        wq_set_error("warp-specialised kernel not configured for this degree");
        return WQ_EINVAL;
    } else {
        WsArgs a;
        a.g.init(Pl);
        for (int l = 0; l < 3; ++l) a.v[l] = Pl->dir[l];
        a.cq_b = Pl->cq_b;
        a.comp0 = STIFF ? 0 : Pl->comp_mass;
        a.val = val;
        a.col = col;
        a.val_base = val_base;
        a.plane_lo = pl_lo;
        const int64_t lines = Pl->dir[1].n * (pl_hi - pl_lo);
        a.n_items = lines * CF::NCH;
        a.dbg = getenv("WQ_WS_DBG") ? atoi(getenv("WQ_WS_DBG")) : 0;
        if (a.n_items <= 0) return WQ_OK;
        CUtensorMap ms, mb;
        if (!make_map(&ms, Pl, CF::NQSB, CF::QI, CF::NCOMP) || !make_map(&mb, Pl, CF::NQSB, CF::QB, CF::NCOMP)) {
            wq_set_error("cuTensorMapEncodeTiled failed for the coefficient field");
            return WQ_ECUDA;
        }
        static bool set = false;
        if (!set) {
            cudaFuncSetAttribute(k_ws<P, STIFF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
            set = true;
        }
        int64_t grid = num_sms(Pl->device);
        if (grid > a.n_items) grid = a.n_items;
        k_ws<P, STIFF><<<(unsigned)grid, CF::NT, CF::SMEM, s>>>(ms, mb, a);
        wq_count_launches(1);
        return wq_cuda_status(cudaGetLastError(), "warp-specialised assembly kernel");
    }
}

template <bool STIFF>
wq_status dispatch_ws(wq_plan_s *Pl, double *val, int32_t *col, int64_t lo, int64_t hi, int64_t vb, cudaStream_t s) {
    switch (Pl->p) {
    case 1: return launch_ws_p<1, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 2: return launch_ws_p<2, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 3: return launch_ws_p<3, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 4: return launch_ws_p<4, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 5: return launch_ws_p<5, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 6: return launch_ws_p<6, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 7: return launch_ws_p<7, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 8: return launch_ws_p<8, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 9: return launch_ws_p<9, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 10: return launch_ws_p<10, STIFF>(Pl, val, col, lo, hi, vb, s);
    }
    wq_set_error("warp-specialised kernel: unsupported degree");
    return WQ_EINVAL;
}

template <bool STIFF>
bool fits_p(int p) {
    switch (p) {
    case 1: return WsCfg<1, STIFF>::FITS;
    case 2: return WsCfg<2, STIFF>::FITS;
    case 3: return WsCfg<3, STIFF>::FITS;
    case 4: return WsCfg<4, STIFF>::FITS;
    case 5: return WsCfg<5, STIFF>::FITS;
    case 6: return WsCfg<6, STIFF>::FITS;
    case 7: return WsCfg<7, STIFF>::FITS;
    case 8: return WsCfg<8, STIFF>::FITS;
    case 9: return WsCfg<9, STIFF>::FITS;
    case 10: return WsCfg<10, STIFF>::FITS;
    }
    return false;
}

}  // namespace

bool ws_supported(const wq_plan_s *P, int matrix) {
    if (P->d != 3 || P->p < 1 || P->p > 10) return false;
    if (matrix == WQ_STIFFNESS && P->zlayout) return false;  // stiffness components are in the z layout
    for (int l = 0; l < 3; ++l)
        if (P->dir[l].maxq > 3 * P->p + 1) return false;  // a support holding both boundary spans
    if (P->dir[0].n < 2) return false;
    if (!encode_fn()) return false;
    return matrix == WQ_MASS ? fits_p<false>(P->p) : fits_p<true>(P->p);
}

wq_status launch_assemble_ws(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo, int64_t plane_hi,
                             int64_t val_base, cudaStream_t s) {
    if (!ws_supported(P, matrix)) {
        wq_set_error("warp-specialised kernel not available for this plan");
        return WQ_EINVAL;
    }
    return matrix == WQ_MASS ? dispatch_ws<false>(P, val, col, plane_lo, plane_hi, val_base, s)
                             : dispatch_ws<true>(P, val, col, plane_lo, plane_hi, val_base, s);
}

#ifdef WQ_DIAG
// debug builds only: route stuck-wait records to a host-mapped buffer
extern "C" int wq_diag_set(unsigned long long *mapped) {
    return (int)cudaMemcpyToSymbol(g_wq_diag, &mapped, sizeof(mapped));
}
#endif
