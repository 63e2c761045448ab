#pragma once
// wq_zhp.cuh -- step 7, the z-line kernel for every degree and both matrices (WQ_KERNEL_ZHP):
// lines along direction 3 like k_zline, with a producer and a consumer thread group per CTA, built
// so that the shared-memory pipeline fits the SM at every degree.
//
// Arithmetic (Eq. sumfactorization P:837 / Alg. 3; stiffness reading R8, families R3).
// A LINE is the set of rows i = (i0, i1, i2), (i0, i1) fixed, i2 over the plan's slab; an ITEM is a
// line and a chunk of T consecutive values of t_1 (the second trial index).  With the weights of
// directions 0 and 1 pushed onto the coefficient field pointwise:
//   stiffness (6 chains (m, a2): m = trial-derivative direction, a2 = test derivative in dir. 2)
//     H_{m,1} = w0^(0,b0) w1^(0,b1) C_2m,  H_{m,0} = w0^(1,b0) w1^(0,b1) C_0m + w0^(0,b0) w1^(1,b1) C_1m,
//     b_k = [m == k];
//     stage A (contract c1):  Y_{m,a2}(c0, t1) = sum_c1 D^{b1}B1_{t1}(c1) H_{m,a2}(c0, c1)
//     stage B (contract c0):  G[b2][a2](t0, t1) = sum_{m: [m==2]=b2} sum_c0 D^{b0}B0_{t0}(c0) Y_{m,a2}(c0, t1)
//     stage C (contract c2, per row i2):
//       S(i; t0, t1, t2) = sum_c2 B2_{t2}(c2) U0(c2) + B2'_{t2}(c2) U1(c2),
//       U0 = w2^(0,0) G[0][0] + w2^(1,0) G[0][1],  U1 = w2^(0,1) G[1][0] + w2^(1,1) G[1][1];
//   mass (one chain): H = w0^(0,0) w1^(0,0) c, Y = sum_c1 B1 H, G = sum_c0 B0 Y,
//       M(i; t) = sum_c2 w2^(0,0) B2_{t2}(c2) G(c2).
// (H is pointwise in (c0, c1), so the order of the first two contractions is free; contracting c1
// first lets an item own whole runs of t0, the fastest index of a CSR row segment: a chunk CTA writes
// every 32-B sector of its runs alone instead of sharing it with the neighbouring t0 chunk, which
// had cost a read-modify-write of most written sectors at p = 8.)
// Staircases for every row type: the points c of a row are grouped by their staircase offset
// o(c) = span(c) - jlo (non-decreasing in c, 0 <= o <= p for every row of every knot vector), and
// the kernel loops over o at compile time and over the points of the group at run time, so each
// accumulator index o + r is a compile-time register index while the group bounds come from
// small per-row tables: one code path for interior, boundary and graded rows.
//
// CTA (256 producer + 256 consumer threads, one per SM, persistent over items): per step of R rows
//   producers: the G planes the step needs, pair of points by pair of points (the coefficient box of
//     a pair, 2 x QX x QX x ncomp, is one 4D TMA tile of the z layout, several in flight):
//     stage A (threads = fibres (m, c0) of a pair), barrier, next box loads, stage B (threads =
//     (point, family, t1)) into a ring of G planes (+ the planes' direction-2 basis pairs);
//   consumers (stage C): threads = (row, column (t0, t1)), acc[t2] in registers, plain coalesced
//     stores of values (and fused columns) straight from registers.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include "wq_rows.cuh"
#include "wq_dev.cuh"

namespace zhp {
using namespace wqdev;

// fully unrolled interior staircases (bits: 1 stage A, 2 stage B, 4 stage C); the rolled offset-group
// form is smaller code (instruction-cache misses are the top stall of both roles at high p)
#ifndef WQ_ZHP_UNROLL
#define WQ_ZHP_UNROLL 7
#endif
constexpr bool kIntA = (WQ_ZHP_UNROLL & 1) != 0, kIntB = (WQ_ZHP_UNROLL & 2) != 0, kIntC = (WQ_ZHP_UNROLL & 4) != 0;

constexpr int NPRO = 256;             // producer threads (stages A, B)
constexpr int NCON = 256;             // consumer threads (stage C)
constexpr int NT = NPRO + NCON;

// column chunks of t_0 per degree (the G ring of a chunk, T (2p+1) x 4 doubles per point, and the
// coefficient boxes must fit the SM's shared memory)
__host__ __device__ constexpr int nch_of(int p) { return p <= 6 ? 1 : (p <= 7 ? 2 : (p <= 8 ? 3 : (p == 9 ? 5 : 7))); }
template <int P>
struct Chunks {
    static constexpr int K = 2 * P + 1, NCH = nch_of(P), T = (K + NCH - 1) / NCH;
    __host__ __device__ static constexpr int ta(int ch) { return ch * K / NCH; }  // balanced: widths T or T-1
    __host__ __device__ static constexpr int tn(int ch) { return ta(ch + 1) - ta(ch); }
};

template <int P, bool MASS, int T, int QX>
struct Cfg {
    static constexpr int K = 2 * P + 1;
    static constexpr int NP = P + 1;
    static constexpr int NCH = nch_of(P);
    static_assert(T == Chunks<P>::T, "chunk width");
    static constexpr int NC = MASS ? 1 : 6;       // coefficient components in the box
    static constexpr int NCHAIN = MASS ? 1 : 6;   // stage-A chains
    static constexpr int NGF = MASS ? 1 : 4;      // G families per column
    static constexpr int COLS = T * K;            // columns (t0, t1 local) of an item, t0 fastest
    static constexpr int BOXD = (NC * QX * QX * 2 + 15) / 16 * 16;  // doubles per box buffer (128-B aligned TMA dst)
    static constexpr int YPAIR = 2 * NCHAIN * QX * T;  // doubles of Y per pair [pt][chain][c1][t0]
    static constexpr int SLOT = COLS * NGF;       // doubles of a G ring slot [col][family]
    static constexpr int QR = 3 * P + 1;          // max #Q of a row (n_EL >= p+2)
#ifdef WQ_ZHP_SPA
    static constexpr bool SPA = WQ_ZHP_SPA;
#else
    // stage-A threads per pair fibre: one per point for the mass matrix at 4 <= p <= 8, where a batch
    // has few fibres (#Q_0 per pair) for the 256 producer threads (measured, C4: p = 4 5.93 -> 5.76 ms,
    // p = 8 37.2 -> 36.6; slower at p = 10 and for the stiffness matrix, whose three fibres per c0
    // fill the threads better and whose 16-B loads serve both points: p = 8 113 -> 138 ms)
    static constexpr bool SPA = MASS && P >= 4 && P <= 8;
#endif
#ifdef WQ_ZHP_CPT
    static constexpr int CPT = WQ_ZHP_CPT;
#else
    // stage-C columns per consumer thread (measured, C4: stiffness p = 8 129 -> 112 ms with one column,
    // mass p = 6 13.2 -> 11.5 ms with three, p = 10 121 -> 100 ms with two)
    static constexpr int CPT = MASS ? (P == 5 || P == 6 ? 3 : 2) : (P >= 8 ? 1 : 2);
#endif
};

struct Args {
    DirView v[3];
    int64_t n0, n1;          // DOFs in directions 0, 1
    int64_t L0, L1;          // sum_i #I_{0,i}, sum_i #I_{1,i}
    int64_t slab_b;          // first owned plane of i2 (CSR offsets relative to it)
    int64_t i2b, n2l;        // rows of this launch: planes [i2b, i2b + n2l) of the slab
    int64_t cq_b;            // first q2 of the coefficient sub-grid
    int64_t qoff;            // even local q2 (relative to cq_b) of this launch's first pair
    const int32_t *lines;    // line = i0 + n0 * i1
    int64_t n_lines;
    int ns;                  // G ring slots
    int depth;               // pipeline depth D: the producers run up to D-1 steps ahead (2..4)
    int R;                   // rows per step
    int nb;                  // box buffers
    double *val;
    int32_t *col;
    int64_t val_base;
    int cl;                  // launched as clusters of the NCH chunk CTAs of a line (lockstep per step)
    int rollc;               // stage C in the rolled sliding-window form (env WQ_ZHP_ROLLC; default p >= 6)
    int abl;                 // measurement switch (env WQ_ZHP_ABLATE), bits: 1 = no stage C, 2 = no stages A, B, 4 = no box loads
};

// shared-memory carve-up (byte offsets), identical on host and device
struct Layout {
    size_t bar, box, y, ring, rb2, t0, t1, w0, w1, o0, o1, g0, g1, w2, g2, d2, total;
};
template <int P, bool MASS, int T, int QX>
__host__ __device__ inline Layout layout(int nb, int R, int ns, int64_t n2l) {
    using CF = Cfg<P, MASS, T, QX>;
    Layout L;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 127) & ~(size_t)127; return r; };
    L.bar = take(8 * 16);
    L.box = take(8 * (size_t)nb * CF::BOXD);
    L.y = take(8 * (size_t)R * CF::YPAIR);
    L.ring = take(8 * (size_t)ns * CF::SLOT);
    L.rb2 = take(16 * (size_t)ns * CF::NP);
    L.t0 = take(16 * (size_t)QX * CF::NP);
    L.t1 = take(16 * (size_t)QX * CF::NP);
    L.w0 = take(8 * 4 * (size_t)QX);
    L.w1 = take(8 * 4 * (size_t)QX);
    L.o0 = take(4 * (size_t)QX);
    L.o1 = take(4 * (size_t)QX);
    L.g0 = take(4 * (size_t)(CF::NP + 1));
    L.g1 = take(4 * (size_t)(CF::NP + 1));
    L.w2 = take(8 * 4 * 2 * (size_t)R * CF::QR);
    L.g2 = take(4 * (size_t)n2l * (CF::NP + 1));
    L.d2 = take(8 * (size_t)(n2l + 1) + 16 * (size_t)n2l);
    L.total = o;
    return L;
}

// split cluster barrier: keeps the chunk CTAs of a line (one cluster) within a step of each other
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// group bounds of a point range: g[o] = first point c with off[c] >= o, o = 0..NP (g[NP] = n)
template <int NP>
__device__ __forceinline__ void groups(const int *off, int n, int *g, int tid) {
    if (tid <= NP) {
        int c = 0;
        while (c < n && off[c] < tid) ++c;
        g[tid] = tid == NP ? n : c;
    }
}

// f(c, integral_constant<o>) for every point c of a row in order, o = staircase offset of c.
// INT: an interior row (the 2P+1 points mid, knot, mid, .., with offsets (c+1)/2, P:537-542 and
// Remark 1), fully unrolled with compile-time c; else the points of each offset group at run time.
template <int P, bool INT, class F>
__device__ __forceinline__ void staircase(const int *g, F &&f) {
    if constexpr (INT) {
        unroll<2 * P + 1>([&](auto C) {
            constexpr int c = decltype(C)::value;
            f(c, std::integral_constant<int, (c + 1) / 2>{});
        });
    } else {
        unroll<P + 1>([&](auto O) {
            constexpr int o = decltype(O)::value;
            for (int c = g[o]; c < g[o + 1]; ++c) f(c, O);
        });
    }
}

// stage A of the pairs pp0 .. pp0 + nbat - 1 (box of pair pp in buffer pp % nb, Y of batch pair k):
// contracts c1 for the chunk's t1 range; a thread = fibre (m, c0) of one pair, both points (the box
// holds the pair's points side by side, so one 16-B load serves both and the tables are loaded once
// per two points), or with SPA one point of the pair (twice the threads, half the serial work per
// thread: at high degree a batch has fewer fibres than producer threads)
template <int P, bool MASS, int T, int QX, int CH, bool SPA>
__device__ __forceinline__ void stage_a(const double *Boxes, int nb, int pp0, int nbat, double *Yall,
                                        const double2 *B1t, const double *W0t, const double *W1t, const int *g1,
                                        int nq0, int tid) {
    using CF = Cfg<P, MASS, T, QX>;
    constexpr int TA = Chunks<P>::ta(CH), TN = Chunks<P>::tn(CH);  // t1 range of the chunk
    constexpr int NPT = SPA ? 1 : 2;                                // points per thread
    const int nfib = (MASS ? 1 : 3) * nq0;
    const int nit = nfib * (SPA ? 2 : 1);
    for (int fx = tid; fx < nbat * nit; fx += NPRO) {
        const int k = fx / nit, f0 = fx % nit;
        const int pt0 = SPA ? f0 / nfib : 0, f = SPA ? f0 - pt0 * nfib : f0;
        const double *box = Boxes + ((pp0 + k) % nb) * CF::BOXD;
        double *Y = Yall + k * CF::YPAIR;
        const int c0 = f % nq0, m = f / nq0;
        // the thread's points of the box entry at e (both points, or point pt0)
        auto ld = [&](int e, double (&v)[NPT]) {
            if constexpr (SPA) {
                v[0] = box[e * 2 + pt0];
            } else {
                const double2 w = *(const double2 *)(box + e * 2);
                v[0] = w.x;
                v[1] = w.y;
            }
        };
        double y0[NPT][T], y1[NPT][T];
        #pragma unroll
        for (int t = 0; t < T; ++t)
            #pragma unroll
            for (int h = 0; h < NPT; ++h) { y0[h][t] = 0.0; y1[h][t] = 0.0; }
        if constexpr (MASS) {
            const double w0 = W0t[c0 * 4 + 0];
            staircase<P, kIntA && QX == 2 * P + 1>(g1, [&](int c1, auto O) {
                constexpr int o = decltype(O)::value;
                double cv[NPT];
                ld(c0 * QX + c1, cv);
                const double s = W1t[c1 * 4 + 0] * w0;
                double ha[NPT];
                #pragma unroll
                for (int h = 0; h < NPT; ++h) ha[h] = s * cv[h];
                const double2 *bp = B1t + c1 * CF::NP;
                #pragma unroll
                for (int r = 0; r <= P; ++r) {
                    const int t = o + r - TA;
                    if (t >= 0 && t < TN) {
                        const double bv = bp[r].x;
                        #pragma unroll
                        for (int h = 0; h < NPT; ++h) y0[h][t] = fma(bv, ha[h], y0[h][t]);
                    }
                }
            });
            #pragma unroll
            for (int h = 0; h < NPT; ++h) {
                double *Yo = Y + (((pt0 + h) * CF::NCHAIN + 0) * QX + c0) * T;
                #pragma unroll
                for (int t = 0; t < T; ++t) Yo[t] = y0[h][t];
            }
        } else {
            // components C00 C01 C02 C11 C12 C22: ka = C_2m, kb = C_0m, kc = C_1m
            const int ka = m == 0 ? 2 : (m == 1 ? 4 : 5);
            const int kb = m == 0 ? 0 : (m == 1 ? 1 : 2);
            const int kc = m == 0 ? 1 : (m == 1 ? 3 : 4);
            const double2 w0p = *(const double2 *)(W0t + c0 * 4 + (m == 0 ? 2 : 0));  // (w0^(0,b0), w0^(1,b0))
            const int w1o = m == 1 ? 2 : 0;
            const bool der1 = m == 1;
            staircase<P, kIntA && QX == 2 * P + 1>(g1, [&](int c1, auto O) {
                constexpr int o = decltype(O)::value;
                const double2 w1p = *(const double2 *)(W1t + c1 * 4 + w1o);  // (w1^(0,b1), w1^(1,b1))
                const double s1 = w0p.x * w1p.x, s2 = w0p.y * w1p.x, s3 = w0p.x * w1p.y;
                double ca[NPT], cb[NPT], cc[NPT], h1[NPT], h0[NPT];
                ld((ka * QX + c0) * QX + c1, ca);
                ld((kb * QX + c0) * QX + c1, cb);
                ld((kc * QX + c0) * QX + c1, cc);
                #pragma unroll
                for (int h = 0; h < NPT; ++h) {
                    h1[h] = s1 * ca[h];                    // a2 = 1 (l = 2)
                    h0[h] = fma(s2, cb[h], s3 * cc[h]);    // a2 = 0 (l = 0, 1)
                }
                const double2 *bp = B1t + c1 * CF::NP;
                #pragma unroll
                for (int r = 0; r <= P; ++r) {
                    const int t = o + r - TA;
                    if (t >= 0 && t < TN) {
                        const double bv = der1 ? bp[r].y : bp[r].x;
                        #pragma unroll
                        for (int h = 0; h < NPT; ++h) {
                            y0[h][t] = fma(bv, h0[h], y0[h][t]);
                            y1[h][t] = fma(bv, h1[h], y1[h][t]);
                        }
                    }
                }
            });
            #pragma unroll
            for (int h = 0; h < NPT; ++h) {
                double *Y0 = Y + (((pt0 + h) * CF::NCHAIN + m * 2 + 0) * QX + c0) * T;
                double *Y1 = Y + (((pt0 + h) * CF::NCHAIN + m * 2 + 1) * QX + c0) * T;
                #pragma unroll
                for (int t = 0; t < T; ++t) { Y0[t] = y0[h][t]; Y1[t] = y1[h][t]; }
            }
        }
    }
}

template <int P, bool MASS, int T, int QX>
__global__ void __launch_bounds__(NT, 1) k_zhp(const __grid_constant__ CUtensorMap tm, Args a) {
    using CF = Cfg<P, MASS, T, QX>;
    constexpr int K = CF::K, NP = CF::NP, NCH = CF::NCH, COLS = CF::COLS, NGF = CF::NGF;
    constexpr int BS = wq_bstride(P);
    extern __shared__ __align__(128) unsigned char smb[];
    const int tid = threadIdx.x;
    const int R = a.R, NS = a.ns, NB = a.nb;
    const int n2l = (int)a.n2l;
    const Layout Ly = layout<P, MASS, T, QX>(NB, R, NS, a.n2l);
    uint64_t *full = (uint64_t *)(smb + Ly.bar);  // [NB] box loads
    uint64_t *ready = full + 8;                   // [D] step planes produced (count NPRO)
    uint64_t *freeb = full + 12;                  // [D] step consumed (count NCON)
    const int D = a.depth;
    double *Box = (double *)(smb + Ly.box);
    double *Y = (double *)(smb + Ly.y);
    double *Ring = (double *)(smb + Ly.ring);
    double2 *RB2 = (double2 *)(smb + Ly.rb2);
    double2 *B0t = (double2 *)(smb + Ly.t0), *B1t = (double2 *)(smb + Ly.t1);
    double *W0t = (double *)(smb + Ly.w0), *W1t = (double *)(smb + Ly.w1);
    int *off0 = (int *)(smb + Ly.o0), *off1 = (int *)(smb + Ly.o1);
    int *g0 = (int *)(smb + Ly.g0), *g1 = (int *)(smb + Ly.g1);
    double *W2s = (double *)(smb + Ly.w2);  // [2 parities][R][QR][4]
    int *g2s = (int *)(smb + Ly.g2);        // [n2l][NP+1] staircase groups of every row (direction 2)
    int64_t *pref2 = (int64_t *)(smb + Ly.d2);
    int *qlo2 = (int *)(pref2 + n2l + 1), *qlen2 = qlo2 + n2l, *jlo2 = qlen2 + n2l, *jlen2 = jlo2 + n2l;

    const DirView &v0 = a.v[0], &v1 = a.v[1], &v2 = a.v[2];
    const int i2b = (int)a.i2b;
    const int cqb = (int)(a.cq_b + a.qoff);  // global index of local point 0 (even offset in the z field)
    for (int x = tid; x < n2l; x += NT) {
        qlo2[x] = v2.qlo[i2b + x] - cqb; qlen2[x] = v2.qlen[i2b + x]; jlo2[x] = v2.jlo[i2b + x]; jlen2[x] = v2.jlen[i2b + x];
    }
    for (int x = tid; x <= n2l; x += NT) pref2[x] = v2.pref[i2b + x] - v2.pref[a.slab_b];
    // the rows' groups depend on i2 only: formed once per CTA for every line
    for (int x = tid; x < n2l * (NP + 1); x += NT) {
        const int rr = x / (NP + 1), o = x % (NP + 1);
        const int q0 = v2.qlo[i2b + rr], n = v2.qlen[i2b + rr], j = v2.jlo[i2b + rr];
        int c = 0;
        while (c < n && v2.span[q0 + c] - j < o) ++c;
        g2s[x] = o == NP ? n : c;
    }
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) mbar_init(&full[b], 1);
        for (int b = 0; b < D; ++b) { mbar_init(&ready[b], NPRO); mbar_init(&freeb[b], NCON); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int q_end = qlo2[n2l - 1] + qlen2[n2l - 1];  // local end of the last row's Q
    const int npairs = (q_end + 1) / 2;
    const int nsteps = (n2l + R - 1) / R;
    int narr = 0;  // cluster-barrier arrivals of this thread (NCH > 1: one per step)
    auto step_sync = [&]() {
        if (NCH > 1 && a.cl) {
            if (narr > 0) cl_wait();
            cl_arrive();
            ++narr;
        }
    };
    constexpr unsigned BOX_BYTES = CF::NC * QX * QX * 2 * 8;
    constexpr bool SPA = CF::SPA;

    if (tid < NPRO) {
        // ================================================================ producers
        const int ptid = tid;
        unsigned use_bits = 0;  // phase parity of each box buffer's next use (bit b)
        int64_t gs = 0;         // global step counter (shared sequence with the consumers)
        for (int64_t li = blockIdx.x / NCH; li < a.n_lines; li += gridDim.x / NCH) {
            const int line = a.lines[li];
            const int ch = (int)(blockIdx.x % NCH);  // the CTA's rank in its cluster (NCH > 1)
            const int i0 = (int)(line % a.n0), i1 = (int)(line / a.n0);
            const int ql0 = v0.qlo[i0], nq0 = v0.qlen[i0], jl0 = v0.jlo[i0];
            const int ql1 = v1.qlo[i1], nq1 = v1.qlen[i1], jl1 = v1.jlo[i1];
            // the ring restarts at plane 0: wait until the consumers have finished the previous item
            if (gs >= 1) mbar_wait_sleep(&freeb[(gs - 1) % D], ((gs - 1) / D) & 1);
            bar_sync(1, NPRO);  // every producer is past the previous item (tables free)
            if (ptid == 0 && !(a.abl & 4)) {
                for (int b = 0; b < NB && b < npairs; ++b) {
                    mbar_arrive_tx(&full[b], BOX_BYTES);
                    tma_load_4d(Box + b * CF::BOXD, &tm, &full[b], (int)a.qoff + 2 * b, ql1, ql0, 0);
                }
            }
            for (int x = ptid; x < QX * NP; x += NPRO) {
                const int c = x / NP, r = x % NP;
                B0t[x] = c < nq0 ? __ldg((const double2 *)(v0.B + (int64_t)(ql0 + c) * BS) + r) : make_double2(0.0, 0.0);
                B1t[x] = c < nq1 ? __ldg((const double2 *)(v1.B + (int64_t)(ql1 + c) * BS) + r) : make_double2(0.0, 0.0);
            }
            for (int x = ptid; x < 4 * QX; x += NPRO) {
                W0t[x] = x / 4 < nq0 ? __ldg(v0.W + (int64_t)i0 * v0.maxq * 4 + x) : 0.0;
                W1t[x] = x / 4 < nq1 ? __ldg(v1.W + (int64_t)i1 * v1.maxq * 4 + x) : 0.0;
            }
            for (int x = ptid; x < QX; x += NPRO) {
                off0[x] = x < nq0 ? v0.span[ql0 + x] - jl0 : 1 << 20;
                off1[x] = x < nq1 ? v1.span[ql1 + x] - jl1 : 1 << 20;
            }
            bar_sync(1, NPRO);
            groups<NP>(off0, nq0, g0, ptid);
            if (ptid >= 32 && ptid <= 32 + NP) groups<NP>(off1, nq1, g1, ptid - 32);
            bar_sync(1, NPRO);
            int pairs_done = 0;
            for (int st = 0; st < nsteps; ++st, ++gs) {
                const int r0 = st * R;
                const int rl = (r0 + R <= n2l ? r0 + R : n2l) - 1;
                const int need = (qlo2[rl] + qlen2[rl] + 1) / 2;  // pairs covering the step's last point
                // the slots this step writes were last read D steps ago
                if (gs >= D) mbar_wait_sleep(&freeb[gs % D], ((gs - D) / D) & 1);
                while (pairs_done < need) {
                    const int nbat = need - pairs_done < R ? need - pairs_done : R;
                    for (int k = 0; k < nbat; ++k) {
                        const int b = (pairs_done + k) % NB;
                        if (!(a.abl & 4)) mbar_wait(&full[b], (use_bits >> b) & 1);
                    }
                    if (!(a.abl & 2)) switch (ch) {
                    case 0: stage_a<P, MASS, T, QX, 0, SPA>(Box, NB, pairs_done, nbat, Y, B1t, W0t, W1t, g1, nq0, ptid); break;
                    case 1: if constexpr (NCH > 1) stage_a<P, MASS, T, QX, 1, SPA>(Box, NB, pairs_done, nbat, Y, B1t, W0t, W1t, g1, nq0, ptid); break;
                    case 2: if constexpr (NCH > 2) stage_a<P, MASS, T, QX, 2, SPA>(Box, NB, pairs_done, nbat, Y, B1t, W0t, W1t, g1, nq0, ptid); break;
                    case 3: if constexpr (NCH > 3) stage_a<P, MASS, T, QX, 3, SPA>(Box, NB, pairs_done, nbat, Y, B1t, W0t, W1t, g1, nq0, ptid); break;
                    case 4: if constexpr (NCH > 4) stage_a<P, MASS, T, QX, 4, SPA>(Box, NB, pairs_done, nbat, Y, B1t, W0t, W1t, g1, nq0, ptid); break;
                    case 5: if constexpr (NCH > 5) stage_a<P, MASS, T, QX, 5, SPA>(Box, NB, pairs_done, nbat, Y, B1t, W0t, W1t, g1, nq0, ptid); break;
                    case 6: if constexpr (NCH > 6) stage_a<P, MASS, T, QX, 6, SPA>(Box, NB, pairs_done, nbat, Y, B1t, W0t, W1t, g1, nq0, ptid); break;
                    default: break;
                    }
                    bar_sync(1, NPRO);  // the batch's boxes consumed, Y written
                    for (int k = 0; k < nbat; ++k) {
                        const int pp = pairs_done + k, b = pp % NB;
                        use_bits ^= 1u << b;
                        if (ptid == 0 && pp + NB < npairs && !(a.abl & 4)) {
                            if (k == 0) fence_async_smem();
                            mbar_arrive_tx(&full[b], BOX_BYTES);
                            tma_load_4d(Box + b * CF::BOXD, &tm, &full[b], (int)a.qoff + 2 * (pp + NB), ql1, ql0, 0);
                        }
                    }
                    // stage B for the batch: items (plane j, t1 of the chunk, family g), contracting c0 for
                    // every t0 -> G ring (column t0 + K t1l), + the planes' B2 pairs
                    const int nitem = (a.abl & 2) ? 0 : nbat * 2 * NGF * T;
                    for (int x = ptid; x < nitem; x += NPRO) {
                        const int g = x % NGF, tl = (x / NGF) % T, j = x / (NGF * T);
                        const int k = j >> 1, pt = j & 1;
                        const int q = 2 * (pairs_done + k) + pt;  // local point
                        const double *Yk = Y + k * CF::YPAIR + pt * CF::NCHAIN * QX * T;
                        double *G = Ring + (size_t)(q % NS) * CF::SLOT;
                        double acc[K];
                        #pragma unroll
                        for (int t = 0; t < K; ++t) acc[t] = 0.0;
                        if constexpr (MASS) {
                            staircase<P, kIntB && QX == 2 * P + 1>(g0, [&](int c0, auto O) {
                                constexpr int o = decltype(O)::value;
                                const double yv = Yk[c0 * T + tl];
                                const double2 *bp = B0t + c0 * NP;
                                #pragma unroll
                                for (int r = 0; r <= P; ++r) acc[o + r] = fma(bp[r].x, yv, acc[o + r]);
                            });
                        } else {
                            // g = a2 + 2 b2: b2 = 0 sums chains m = 1 (B0 values) and m = 0 (B0
                            // derivatives), b2 = 1 is chain m = 2 (B0 values)
                            const int a2 = g & 1, b2 = g >> 1;
                            const double *Ya = Yk + ((b2 ? 4 : 2) + a2) * QX * T;
                            const double *Yb = Yk + a2 * QX * T;
                            staircase<P, kIntB && QX == 2 * P + 1>(g0, [&](int c0, auto O) {
                                constexpr int o = decltype(O)::value;
                                const double ya = Ya[c0 * T + tl];
                                const double yb = b2 ? 0.0 : Yb[c0 * T + tl];
                                const double2 *bp = B0t + c0 * NP;
                                #pragma unroll
                                for (int r = 0; r <= P; ++r) acc[o + r] = fma(bp[r].y, yb, fma(bp[r].x, ya, acc[o + r]));
                            });
                        }
                        #pragma unroll
                        for (int t = 0; t < K; ++t) {
                            // ring slot [b2][column][a2] (stage C loads (a2 = 0, 1) pairs with a 16-B
                            // lane stride: conflict-free)
                            const int cl = t + K * tl;
                            if constexpr (MASS) G[cl] = acc[t];
                            else G[((g >> 1) * COLS + cl) * 2 + (g & 1)] = acc[t];
                        }
                    }
                    for (int x = ptid; x < nbat * 2 * NP; x += NPRO) {
                        const int q = 2 * pairs_done + x / NP, r = x % NP;
                        RB2[(q % NS) * NP + r] = q < q_end ? __ldg((const double2 *)(v2.B + (int64_t)(cqb + q) * BS) + r)
                                                           : make_double2(0.0, 0.0);
                    }
                    bar_sync(1, NPRO);  // Y free for the next batch
                    pairs_done += nbat;
                }
                mbar_arrive(&ready[gs % D]);  // release: this step's planes are in the ring
                step_sync();
            }
        }
        if (NCH > 1 && a.cl && narr > 0) cl_wait();
        return;
    }
    // ==================================================================== consumers
    const int ctid = tid - NPRO;
    int64_t gs = 0;
    // direction-2 weights of a step's rows (they depend on i2 only), copied asynchronously one step
    // ahead into the buffer of that step's parity: [2 parities][R][QR][4]
    auto load_w2 = [&](int st, int par) {
        const int r0 = st * R, nr = r0 + R <= n2l ? R : n2l - r0;
        double *W2p = W2s + (size_t)par * R * CF::QR * 4;
        for (int x = ctid; x < nr * CF::QR * 2; x += NCON) {  // 16-B pieces: (point, half)
            const int rho = x / (CF::QR * 2), e = x % (CF::QR * 2);
            const int i2 = i2b + r0 + rho;
            const bool in = e / 2 < qlen2[r0 + rho];
            cp_async16(W2p + (size_t)rho * CF::QR * 4 + 2 * e, in ? (const void *)(v2.W + (int64_t)i2 * v2.maxq * 4 + 2 * e) : (const void *)v2.W,
                       in ? 16u : 0u);
        }
    };
    if (a.n_lines > blockIdx.x / NCH) load_w2(0, 0);
    for (int64_t li = blockIdx.x / NCH; li < a.n_lines; li += gridDim.x / NCH) {
        const int line = a.lines[li];
        const int ch = (int)(blockIdx.x % NCH);
        const int i0 = (int)(line % a.n0), i1 = (int)(line / a.n0);
        const int jl0 = v0.jlo[i0], ni0 = v0.jlen[i0];
        const int jl1 = v1.jlo[i1], ni1 = v1.jlen[i1];
        const int ta = Chunks<P>::ta(ch), tn = Chunks<P>::tn(ch);
        // CSR offset of row (i0, i1, i2) relative to the first owned row minus val_base:
        // (pref2[i2] - pref2[slab_b]) L1 L0 + ni2 pref1[i1] L0 + ni2 ni1 pref0[i0]
        const int64_t p1L0 = v1.pref[i1] * a.L0, p0n1 = v0.pref[i0] * (int64_t)ni1;
        for (int st = 0; st < nsteps; ++st, ++gs) {
            const int r0 = st * R;
            const int nr = r0 + R <= n2l ? R : n2l - r0;
            const int par = (int)(gs & 1);
            double *W2p = W2s + (size_t)par * R * CF::QR * 4;
            const int *g2p = g2s + r0 * (NP + 1);
            bool all_int = true;
            for (int rho = 0; rho < nr; ++rho) {
                const int i2 = i2b + r0 + rho;
                all_int = all_int && i2 >= P + 1 && i2 <= (int)v2.n - P - 2 && qlen2[r0 + rho] == 2 * P + 1;
            }
            cp_async_wait_all();  // this thread's pieces of the step's weights
            bar_sync(2, NCON);    // everyone's pieces; every consumer is past the previous step
            {   // next step's weights (the next line's first step after the last one)
                const bool last_item = li + gridDim.x / NCH >= a.n_lines;
                if (st + 1 < nsteps) load_w2(st + 1, par ^ 1);
                else if (!last_item) load_w2(0, par ^ 1);
            }
            mbar_wait_sleep(&ready[gs % D], (gs / D) & 1);  // acquire: the step's planes
            // stage C: CPT adjacent columns per thread (the row's point weights and basis pairs are
            // loaded once for them)
            auto stage_c = [&](auto IC) {
                constexpr bool INTC = decltype(IC)::value;
                constexpr int CPT = CF::CPT, NCP = (COLS + CPT - 1) / CPT;
                for (int x = ctid; x < nr * NCP; x += NCON) {
                    const int rho = x / NCP, cl0 = x % NCP;  // columns cl0 + j NCP (consecutive lanes, consecutive columns)
                    const int rr = r0 + rho;
                    const int q0 = qlo2[rr], s0 = q0 % NS;  // ring slot of the row's first point
                    const double *Wr = W2p + rho * CF::QR * 4;
                    const int *gg = g2p + rho * (NP + 1);
                    int clc[CPT];
                    #pragma unroll
                    for (int j = 0; j < CPT; ++j) clc[j] = cl0 + j * NCP < COLS ? cl0 + j * NCP : COLS - 1;
                    double acc[CPT][K];
                    #pragma unroll
                    for (int j = 0; j < CPT; ++j)
                        #pragma unroll
                        for (int t = 0; t < K; ++t) acc[j][t] = 0.0;
                    staircase<P, INTC>(gg, [&](int c, auto O) {
                        constexpr int o = decltype(O)::value;
                        const int s = s0 + c < NS ? s0 + c : s0 + c - NS;  // c < #Q <= NS
                        const double2 *bp = RB2 + s * NP;
                        const double *Gs = Ring + (size_t)s * CF::SLOT;
                        if constexpr (MASS) {
                            const double wv = Wr[c * 4];
                            double uu[CPT];
                            #pragma unroll
                            for (int j = 0; j < CPT; ++j) uu[j] = wv * Gs[clc[j]];
                            #pragma unroll
                            for (int r = 0; r <= P; ++r) {
                                const double bx = bp[r].x;
                                #pragma unroll
                                for (int j = 0; j < CPT; ++j) acc[j][o + r] = fma(bx, uu[j], acc[j][o + r]);
                            }
                        } else {
                            const double4 w = *(const double4 *)(Wr + c * 4);
                            double u0[CPT], u1[CPT];
                            #pragma unroll
                            for (int j = 0; j < CPT; ++j) {
                                const double2 Ga = *(const double2 *)(Gs + clc[j] * 2);               // b2 = 0: a2 = 0, 1
                                const double2 Gb = *(const double2 *)(Gs + (COLS + clc[j]) * 2);      // b2 = 1
                                u0[j] = fma(w.x, Ga.x, w.y * Ga.y);
                                u1[j] = fma(w.z, Gb.x, w.w * Gb.y);
                            }
                            #pragma unroll
                            for (int r = 0; r <= P; ++r) {
                                const double2 b2 = bp[r];
                                #pragma unroll
                                for (int j = 0; j < CPT; ++j) acc[j][o + r] = fma(b2.y, u1[j], fma(b2.x, u0[j], acc[j][o + r]));
                            }
                        }
                    });
                    const int ni2 = INTC ? K : jlen2[rr];  // interior rows: 2p+1 trial indices t2
                    const int64_t row = pref2[rr] * a.L1 * a.L0 + (int64_t)ni2 * (p1L0 + p0n1) - a.val_base;
                    const int stp = ni0 * ni1;
                    #pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        const int cl = cl0 + j * NCP;
                        const int t0 = cl % K, tl = cl / K, t1 = ta + tl;  // chunks over t1: whole t0 runs
                        if (cl < COLS && tl < tn && t0 < ni0 && t1 < ni1) {
                            const int64_t e0 = row + t0 + (int64_t)ni0 * t1;
                            double *vp = a.val + e0;  // pointer walk: one 64-bit add per store
                            #pragma unroll
                            for (int t = 0; t < K; ++t) {
                                if (INTC || t < ni2) *vp = acc[j][t];
                                vp += stp;
                            }
                            if (a.col) {
                                const int jb = (jl0 + t0) + (int)a.n0 * ((jl1 + t1) + (int)a.n1 * jlo2[rr]);
                                const int js = (int)(a.n0 * a.n1);
                                int32_t *cp = a.col + e0;
                                #pragma unroll
                                for (int t = 0; t < K; ++t) {
                                    if (INTC || t < ni2) *cp = jb + js * t;
                                    cp += stp;
                                }
                            }
                        }
                    }
                }
            };
            // stage C, rolled form: one loop over the staircase offsets o = 0..p with the row's
            // accumulators as a sliding window win[r] <-> t2 = o + r (offsets are non-decreasing in c,
            // so t2 = o is final once group o is done: stored, and the window shifts by one).  The
            // loop body is one point: a few hundred bytes of code for every row type, instead of
            // the fully unrolled staircases (instruction-cache misses were the top stall of both
            // thread groups at p = 8).
            auto stage_c_roll = [&](auto IC) {
                constexpr bool INTC = decltype(IC)::value;  // every row of the step interior: groups
                                                           // {0}, {1, 2}, .., {2p-1, 2p}
                constexpr int CPT = CF::CPT, NCP = (COLS + CPT - 1) / CPT;
                const int stp = ni0 * ni1;
                for (int x = ctid; x < nr * NCP; x += NCON) {
                    const int rho = x / NCP, cl0 = x % NCP;  // columns cl0 + j NCP
                    const int rr = r0 + rho;
                    const int q0 = qlo2[rr], s0 = q0 % NS;
                    const double *Wr = W2p + rho * CF::QR * 4;
                    const int *gg = g2p + rho * (NP + 1);
                    const int ni2 = jlen2[rr];
                    const int64_t row = pref2[rr] * a.L1 * a.L0 + (int64_t)ni2 * (p1L0 + p0n1) - a.val_base;
                    int clc[CPT];
                    bool ok[CPT];
                    double *vp[CPT];
                    int32_t *cp[CPT];
                    int jb[CPT];
                    #pragma unroll
                    for (int j = 0; j < CPT; ++j) {
                        const int cl = cl0 + j * NCP;
                        clc[j] = cl < COLS ? cl : COLS - 1;
                        const int t0 = cl % K, tl = cl / K, t1 = ta + tl;
                        ok[j] = cl < COLS && tl < tn && t0 < ni0 && t1 < ni1;
                        const int64_t e0 = row + t0 + (int64_t)ni0 * t1;
                        vp[j] = a.val + e0;
                        cp[j] = a.col ? a.col + e0 : nullptr;
                        jb[j] = (jl0 + t0) + (int)a.n0 * ((jl1 + t1) + (int)a.n1 * jlo2[rr]);
                    }
                    const int js = (int)(a.n0 * a.n1);
                    double win[CPT][NP];
                    #pragma unroll
                    for (int j = 0; j < CPT; ++j)
                        #pragma unroll
                        for (int r = 0; r < NP; ++r) win[j][r] = 0.0;
                    auto put = [&](int t, int j, double v) {  // value (and column) of t2 = jlo + t
                        if (ok[j] && t < ni2) {
                            vp[j][(int64_t)stp * t] = v;
                            if (cp[j]) cp[j][(int64_t)stp * t] = jb[j] + js * t;
                        }
                    };
                    auto point = [&](int c) {
                            const int s = s0 + c < NS ? s0 + c : s0 + c - NS;  // c < #Q <= NS
                            const double2 *bp = RB2 + s * NP;
                            const double *Gs = Ring + (size_t)s * CF::SLOT;
                            if constexpr (MASS) {
                                const double wv = Wr[c * 4];
                                double uu[CPT];
                                #pragma unroll
                                for (int j = 0; j < CPT; ++j) uu[j] = wv * Gs[clc[j]];
                                #pragma unroll
                                for (int r = 0; r <= P; ++r) {
                                    const double bx = bp[r].x;
                                    #pragma unroll
                                    for (int j = 0; j < CPT; ++j) win[j][r] = fma(bx, uu[j], win[j][r]);
                                }
                            } else {
                                const double4 w = *(const double4 *)(Wr + c * 4);
                                double u0[CPT], u1[CPT];
                                #pragma unroll
                                for (int j = 0; j < CPT; ++j) {
                                    const double2 Ga = *(const double2 *)(Gs + clc[j] * 2);
                                    const double2 Gb = *(const double2 *)(Gs + (COLS + clc[j]) * 2);
                                    u0[j] = fma(w.x, Ga.x, w.y * Ga.y);
                                    u1[j] = fma(w.z, Gb.x, w.w * Gb.y);
                                }
                                #pragma unroll
                                for (int r = 0; r <= P; ++r) {
                                    const double2 b2 = bp[r];
                                    #pragma unroll
                                    for (int j = 0; j < CPT; ++j) win[j][r] = fma(b2.y, u1[j], fma(b2.x, u0[j], win[j][r]));
                                }
                            }
                    };
                    int c = 0;
                    for (int o = 0; o <= P; ++o) {
                        if constexpr (INTC) {
                            if (o == 0) point(0);
                            else { point(2 * o - 1); point(2 * o); }
                        } else {
                            for (const int ce = gg[o + 1]; c < ce; ++c) point(c);
                        }
                        #pragma unroll
                        for (int j = 0; j < CPT; ++j) {
                            put(o, j, win[j][0]);
                            #pragma unroll
                            for (int r = 0; r < P; ++r) win[j][r] = win[j][r + 1];
                            win[j][P] = 0.0;
                        }
                    }
                    #pragma unroll
                    for (int r = 0; r < P; ++r)
                        #pragma unroll
                        for (int j = 0; j < CPT; ++j) put(P + 1 + r, j, win[j][r]);
                }
            };
            if (a.abl & 1) {
            } else if (a.rollc) {
                if (all_int) stage_c_roll(std::true_type{});
                else stage_c_roll(std::false_type{});
            }
            else if (kIntC && all_int) stage_c(std::true_type{});
            else stage_c(std::false_type{});
            // this step's ring slots may be overwritten.  Relaxed: every value this thread read from
            // the ring fed the accumulators of the stores it has already issued, so the reads are
            // complete; a release arrive would also wait for those global stores to be acknowledged
            // (ncu: 'membar' stalls of the consumers, C4 p = 8).  Bit-repeatability stress test:
            // tests/test_gpu_parity.py::test_zline_repeatable_bit_exact (ZHP cases).
            mbar_arrive_relaxed(&freeb[gs % D]);
            step_sync();
        }
    }
    if (NCH > 1 && a.cl && narr > 0) cl_wait();
}

}  // namespace zhp

// ---------------------------------------------------------------- host side
namespace zhp {

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

struct Plan2 {  // launch geometry along the slab direction for the planes [pl_lo, pl_hi)
    int64_t i2b, n2l, qoff;
    std::vector<int32_t> qlo, qhi;  // local (relative to cq_b + qoff)
};
inline Plan2 plan2(const wq_plan_s *Pl, int64_t pl_lo, int64_t pl_hi) {
    Plan2 g;
    const int p = Pl->p;
    const int64_t E = Pl->dir[2].E;
    g.i2b = Pl->slab_b + pl_lo;
    g.n2l = pl_hi - pl_lo;
    g.qoff = (wq_host_qlo(g.i2b, E, p) - Pl->cq_b) & ~(int64_t)1;
    for (int64_t i = g.i2b; i < g.i2b + g.n2l; ++i) {
        g.qlo.push_back((int32_t)(wq_host_qlo(i, E, p) - Pl->cq_b - g.qoff));
        g.qhi.push_back((int32_t)(wq_host_qhi(i, E, p) - Pl->cq_b - g.qoff));
    }
    return g;
}
// ring slots for R rows per step: the production of a step overwrites slot (q mod NS) of planes q <
// 2 need while the step's rows read planes >= qlo(first row)
// (the producers write the planes of step s+1 while the consumers read those of step s)
inline int ring_slots(const Plan2 &g, int R, int D) {
    int ns = 2;
    for (int64_t r0 = 0; r0 < g.n2l; r0 += R) {
        const int64_t r1 = std::min<int64_t>(r0 + (int64_t)D * R, g.n2l) - 1;  // last row D-1 steps ahead
        const int need = (g.qhi[r1] + 2) / 2;
        ns = std::max(ns, 2 * need - g.qlo[r0]);
    }
    return ns;
}

// pipeline depth (measurement switch WQ_ZHP_D, 2..4)
inline int zhp_depth() {
    const char *e = getenv("WQ_ZHP_D");
    const int d = e ? atoi(e) : 2;
    return d < 2 ? 2 : (d > 4 ? 4 : d);
}

template <int P, bool MASS, int QX>
bool choose(const Plan2 &g, int &nb, int &R, int &ns, size_t &smem, int optin) {
    constexpr int T = Chunks<P>::T;
    using CF = Cfg<P, MASS, T, QX>;
    // rows per step: as many as one pass of the consumer threads covers (stage C items = rows x COLS);
    // box buffers: a batch of R pairs (stage A runs over the whole batch), doubled for prefetch
    int rbest = NCON / ((CF::COLS + CF::CPT - 1) / CF::CPT);
    rbest = rbest < 1 ? 1 : (rbest > 6 ? 6 : rbest);
    if (getenv("WQ_ZHP_R")) rbest = atoi(getenv("WQ_ZHP_R"));
    const int nb_env = getenv("WQ_ZHP_NB") ? atoi(getenv("WQ_ZHP_NB")) : 0;
    for (int r = rbest; r >= 1; --r)
        for (int b = 2 * r; b >= r; --b) {
            if (b > 8 || (nb_env && b != nb_env)) continue;
            const int n = ring_slots(g, r, zhp_depth());
            const Layout L = layout<P, MASS, T, QX>(b, r, n, g.n2l);
            if (L.total <= (size_t)optin) {
                nb = b;
                R = r;
                ns = n;
                smem = L.total;
                return true;
            }
        }
    return false;
}

template <int P, bool MASS, int QX>
wq_status launch_cls(wq_plan_s *Pl, const int32_t *lines, int64_t n_lines, const Plan2 &g, double *val, int32_t *col,
                     int64_t val_base, cudaStream_t s) {
    constexpr int T = Chunks<P>::T, NCH = Chunks<P>::NCH;
    using CF = Cfg<P, MASS, T, QX>;
    if (n_lines <= 0 || g.n2l <= 0) return WQ_OK;
    int optin = 0, nsm = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, Pl->device);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, Pl->device);
    Args a;
    int nb = 0, R = 0, ns = 0;
    size_t smem = 0;
    if (!choose<P, MASS, QX>(g, nb, R, ns, smem, optin)) {
        wq_set_error("ZHP kernel: shared memory does not fit this slab");
        return WQ_EINVAL;
    }
    for (int l = 0; l < 3; ++l) a.v[l] = Pl->dir[l];
    a.n0 = Pl->dir[0].n;
    a.n1 = Pl->dir[1].n;
    a.L0 = Pl->L[0];
    a.L1 = Pl->L[1];
    a.slab_b = Pl->slab_b;
    a.i2b = g.i2b;
    a.n2l = g.n2l;
    a.cq_b = Pl->cq_b;
    a.qoff = g.qoff;
    a.lines = lines;
    a.n_lines = n_lines;
    a.ns = ns;
    a.R = R;
    a.nb = nb;
    a.depth = zhp_depth();
    a.val = val;
    a.col = col;
    a.val_base = val_base;
    auto fn = encode_fn();
    if (!fn) { wq_set_error("cuTensorMapEncodeTiled unavailable"); return WQ_ECUDA; }
    CUtensorMap m;
    const int64_t nq0 = Pl->dir[0].nq, nq1 = Pl->dir[1].nq;
    const double *base = Pl->coef + (MASS ? (int64_t)Pl->comp_mass * Pl->zcs : 0);
    cuuint64_t dims[4] = {(cuuint64_t)Pl->zld, (cuuint64_t)nq1, (cuuint64_t)nq0, (cuuint64_t)CF::NC};
    cuuint64_t strides[3] = {(cuuint64_t)Pl->zld * 8, (cuuint64_t)Pl->zld * nq1 * 8, (cuuint64_t)Pl->zcs * 8};
    cuuint32_t box[4] = {2, (cuuint32_t)QX, (cuuint32_t)QX, (cuuint32_t)CF::NC};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void *)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
        wq_set_error("cuTensorMapEncodeTiled failed for the coefficient field");
        return WQ_ECUDA;
    }
    // one cluster of NCH CTAs per line (the chunks of a line side by side, kept within a step of each
    // other so that their interleaved partial-sector stores merge in L2)
    const int64_t nclusters = std::max<int64_t>(1, std::min<int64_t>(n_lines, nsm / NCH));
    cudaError_t ce = wq_smem_attr((const void *)k_zhp<P, MASS, T, QX>, smem);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "ZHP smem attribute");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nclusters * NCH));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = NCH;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    // measured: lockstep clusters pay with two chunks (C4 p = 7 mass 42.9 -> 34.6 ms) and cost with
    // three or more (p = 8 stiffness 155 -> 298 ms)
    a.cl = NCH == 2 && !getenv("WQ_ZHP_NOCLUSTER");
    a.abl = getenv("WQ_ZHP_ABLATE") ? atoi(getenv("WQ_ZHP_ABLATE")) : 0;
    // measured (C4): the rolled stage C pays from p = 6 on (stiffness p = 7 74 -> 69 ms, p = 8 161 ->
    // 129, p = 9 312 -> 227; mass p = 6 14.1 -> 13.2, p = 10 133 -> 121) and is neutral below; a
    // rolled stage B was slower at every degree
    a.rollc = getenv("WQ_ZHP_ROLLC") ? atoi(getenv("WQ_ZHP_ROLLC")) : (P >= 6);
    cfg.numAttrs = a.cl ? 1 : 0;
    ce = cudaLaunchKernelEx(&cfg, k_zhp<P, MASS, T, QX>, m, a);
    wq_count_launches(1);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "ZHP assembly kernel");
    return wq_cuda_status(cudaGetLastError(), "ZHP assembly kernel");
}

template <int P>
bool supported_p(const wq_plan_s *Pl, int matrix) {
    const Plan2 g = plan2(Pl, 0, Pl->slab_e - Pl->slab_b);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, Pl->device);
    if (optin <= 0) optin = 227 * 1024;
    int nb, R, ns;
    size_t sm;
    return matrix == WQ_MASS ? choose<P, true, 3 * P + 1>(g, nb, R, ns, sm, optin) &&
                                   choose<P, true, 2 * P + 1>(g, nb, R, ns, sm, optin)
                             : choose<P, false, 3 * P + 1>(g, nb, R, ns, sm, optin) &&
                                   choose<P, false, 2 * P + 1>(g, nb, R, ns, sm, optin);
}

template <int P>
wq_status launch_p(wq_plan_s *Pl, int matrix, int64_t pl_lo, int64_t pl_hi, double *val, int32_t *col,
                   int64_t val_base, cudaStream_t s, int classes) {
    // classes: bit 0 = interior lines (boxes of 2p+1 points), bit 1 = the rest (boundary lines)
    const Plan2 g = plan2(Pl, pl_lo, pl_hi);
    const int64_t ni = (int64_t)Pl->zh_int.size(), nbd = (int64_t)Pl->zh_bnd.size();
    wq_status st = WQ_OK;
    if (matrix == WQ_MASS) {
        if (classes & 1) st = launch_cls<P, true, 2 * P + 1>(Pl, Pl->zh_dev, ni, g, val, col, val_base, s);
        if (!st && (classes & 2)) st = launch_cls<P, true, 3 * P + 1>(Pl, Pl->zh_dev + ni, nbd, g, val, col, val_base, s);
    } else {
        if (classes & 1) st = launch_cls<P, false, 2 * P + 1>(Pl, Pl->zh_dev, ni, g, val, col, val_base, s);
        if (!st && (classes & 2)) st = launch_cls<P, false, 3 * P + 1>(Pl, Pl->zh_dev + ni, nbd, g, val, col, val_base, s);
    }
    return st;
}

}  // namespace zhp

#define WQ_ZHP_DEG_DECL(PP)                                                                                          \
    bool zhp_supported_deg_##PP(const wq_plan_s *Pl, int matrix);                                                 \
    wq_status zhp_launch_deg_##PP(wq_plan_s *Pl, int matrix, int64_t pl_lo, int64_t pl_hi, double *val, int32_t *col, \
                                  int64_t val_base, cudaStream_t s, int classes);
#define WQ_ZHP_DEG_DEF(PP)                                                                                           \
    bool zhp_supported_deg_##PP(const wq_plan_s *Pl, int matrix) { return zhp::supported_p<PP>(Pl, matrix); }      \
    wq_status zhp_launch_deg_##PP(wq_plan_s *Pl, int matrix, int64_t pl_lo, int64_t pl_hi, double *val, int32_t *col, \
                                  int64_t val_base, cudaStream_t s, int classes) {                                  \
        return zhp::launch_p<PP>(Pl, matrix, pl_lo, pl_hi, val, col, val_base, s, classes);                          \
    }
WQ_ZHP_DEG_DECL(1) WQ_ZHP_DEG_DECL(2) WQ_ZHP_DEG_DECL(3) WQ_ZHP_DEG_DECL(4) WQ_ZHP_DEG_DECL(5)
WQ_ZHP_DEG_DECL(6) WQ_ZHP_DEG_DECL(7) WQ_ZHP_DEG_DECL(8) WQ_ZHP_DEG_DECL(9) WQ_ZHP_DEG_DECL(10)
