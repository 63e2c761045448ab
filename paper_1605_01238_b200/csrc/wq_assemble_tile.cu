// wq_assemble_tile.cu -- step 7, sum-factorised row-line kernel (WQ_KERNEL_TILE),
// d = 3, compile-time degree P.  Eq. sumfactorization / Alg. 3
// (P:859-870), re-organised so that rows share every stage but the last
// (DESIGN.md §6 "Row-line kernel"):
//
// CTA = one line (i2, i3) of the row grid (all i1, processed in batches of RB
// rows) x one chunk of T3C trial indices t3.  Per point q1 of the line:
//   stage 3 (+ test weights of directions 2, 3 applied pointwise), fibre (q1, c2):
//     stiffness chains (m, a1); m = trial-derivative direction, a1 = [l == 0]:
//       Y_{m,a1}(c2,t3) = sum_{c3} B3^{[m==2]}_{t3}(c3) *
//                         sum_{l: [l==0]=a1} w2^{([l==1],[m==1])}(c2) w3^{([l==2],[m==2])}(c3) C_lm(q1,c2,c3)
//     mass: Y(c2,t3) = sum_{c3} B3_{t3}(c3) w2^(0,0)(c2) w3^(0,0)(c3) c(q1,c2,c3)
//   stage 2, fibre (q1, t3): G[b1][a1](t2,t3) = sum_{c2} sum_{m: [m==0]=b1} B2^{[m==1]}_{t2}(c2) Y_{m,a1}(c2,t3)
// G lives in a shared-memory ring indexed by q1, so each point is done once per line.
//   stage 1, per row i1 (threads = columns (t2,t3), NR rows per thread in registers):
//     out(t1) = sum_{c1} B1_{t1}(c1) U0(c1) + B1'_{t1}(c1) U1(c1),
//     U0 = w1^(0,0) G[0][0] + w1^(1,0) G[0][1],  U1 = w1^(0,1) G[1][0] + w1^(1,1) G[1][1]
//     (mass: out = sum_{c1} B1_{t1}(c1) w1^(0,0)(c1) G).
// The B-spline factors are taken from the compact per-point tables: at point
// q the nonzero functions are span(q)..span(q)+P, so in a row with first
// column jlo the point contributes to t = span(q) - jlo + r, r = 0..P (a
// monotone staircase).  The staircase offset is dispatched to compile-time
// register indices (uniform across the CTA for stages 3/2, compile-time for
// rows whose support touches no boundary span).
// (a, b) = (test, trial) derivative order (reading R3); directions 1..3 are
// indices 0..2 in the code.
#include <type_traits>
#include "wq_rows.cuh"

namespace {

template <int P, bool STIFF>
struct Cfg {
    static constexpr int K = 2 * P + 1;   // max #I
    static constexpr int QB = 3 * P + 1;  // max #Q (supports with one boundary span)
    static constexpr int NP = P + 1;
    static constexpr int T3C = P <= 5 ? K : (P <= 7 ? 7 : (P <= 9 ? 5 : 3));  // t3 chunk
    static constexpr int NCH = (K + T3C - 1) / T3C;
    static constexpr int COLS = K * T3C;  // columns (t2 + K*t3l) of a chunk
    static constexpr int NT = 256;
    static constexpr int NR = P <= 2 ? 4 : (P <= 4 ? 3 : 2);  // rows per final-stage thread
    static constexpr int NY = STIFF ? 6 : 1;
    static constexpr int NG = STIFF ? 4 : 1;
    __host__ __device__ static constexpr int ev(int x) { return (x + 1) & ~1; }  // keep regions 16-B aligned
    static constexpr int STV = ev(K * COLS + 2);            // staging doubles per group buffer
    static constexpr int STC = (K * COLS + 4 + 3) / 4 * 2;  // staging int32 per group buffer, in doubles
    static constexpr size_t LIMIT = 224 * 1024;
    __host__ __device__ static constexpr size_t smem_for(int ng, int nqs) {
        const int rb = NR * ng, ring = QB + 2 * rb + P;
        const size_t tab = 2 * (2 * QB * NP) + 2 * (4 * QB) + 2 * ring * NP + rb * QB * 4;
        return sizeof(double) * ((size_t)ev(NY * nqs * QB * T3C) + (size_t)ev(NG * ring * COLS) +
                                 2 * (size_t)ng * (STV + STC) + tab + 4);
    }
    // row groups per batch: as many as threads allow and shared memory holds
    __host__ __device__ static constexpr int pick_ng() {
        for (int ng = NT / COLS; ng > 1; --ng)
            if (smem_for(ng, NR * ng) <= LIMIT) return ng;
        return 1;
    }
    static constexpr int NGRP = pick_ng();
    static constexpr int RB = NR * NGRP;          // rows per batch
    static constexpr int RING = QB + 2 * RB + P;  // >= q1 window of a batch
    // stage-3 sub-batch: all new points of a batch (2 RB) if it fits
    static constexpr int NQS = smem_for(NGRP, 2 * RB) <= LIMIT ? 2 * RB
                             : (smem_for(NGRP, RB) <= LIMIT ? RB : (RB / 2 > 2 ? RB / 2 : 2));
    static constexpr int Y_D = ev(NY * NQS * QB * T3C);
    static constexpr int G_D = ev(NG * RING * COLS);
    static constexpr size_t SMEM = smem_for(NGRP, NQS);
    static_assert(NT / COLS >= 1, "columns per chunk exceed the CTA");
    static_assert(SMEM <= 227 * 1024, "tile kernel shared memory");
};

// compile-time dispatch of a runtime offset o in [LO, HI] (|o| <= 31): f(integral_constant<o>);
// a dense switch, compiled to a jump table (one indirect branch, uniform across the CTA)
#define WQ_CASE(O) \
    case O:        \
        if constexpr ((O) >= LO && (O) <= HI) f(std::integral_constant<int, (O)>{}); \
        break;
#define WQ_CASE8(B) WQ_CASE(B) WQ_CASE(B + 1) WQ_CASE(B + 2) WQ_CASE(B + 3) WQ_CASE(B + 4) WQ_CASE(B + 5) WQ_CASE(B + 6) WQ_CASE(B + 7)
template <int LO, int HI, class F>
__device__ __forceinline__ void dispatch(int o, F &&f) {
    static_assert(LO >= -16 && HI < 32, "dispatch range");
    switch (o) {
        WQ_CASE8(-16) WQ_CASE8(-8) WQ_CASE8(0) WQ_CASE8(8) WQ_CASE8(16) WQ_CASE8(24)
    default: break;
    }
}
#undef WQ_CASE8

template <int N, class F>
__device__ __forceinline__ void unroll(F &&f) {
    if constexpr (N > 0) {
        unroll<N - 1>(f);
        f(std::integral_constant<int, N - 1>{});
    }
}

struct TileArgs {
    RowGeo g;
    DirView v[3];
    CoefView cv;       // coefficient field (any layout; q_1 contiguous in the fastest layout)
    int64_t cq_b;
    int comp_mass;
    double *val;
    int32_t *col;
    int64_t val_base;
    int64_t plane_lo;  // first slab plane (relative) of this launch
    const int32_t *lines;  // optional list of lines (i2 + n2 * (i3 - slab_b)); plane_lo = 0 then
};

__device__ __forceinline__ int comp_ix(int l, int m) {  // upper-triangle index, d = 3
    if (l > m) { int t = l; l = m; m = t; }
    return l * 3 - l * (l - 1) / 2 + (m - l);
}

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// shared -> global bulk copy (TMA, async proxy); addresses 16-B aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_s2g(void *g, const void *s, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes)
                 : "memory");
}

template <int P, bool STIFF>
__global__ void __launch_bounds__(256, 1) k_tile(TileArgs a) {
    using CF = Cfg<P, STIFF>;
    constexpr int K = CF::K, NP = CF::NP, T3C = CF::T3C, COLS = CF::COLS, NR = CF::NR, NGRP = CF::NGRP;
    constexpr int RB = CF::RB, RING = CF::RING, NQS = CF::NQS, QB = CF::QB, NT = CF::NT;
    constexpr int BS = wq_bstride(P);  // basis-table stride per point (even)
    constexpr int STV = CF::STV, STC = CF::STC;
    extern __shared__ __align__(16) double sm[];
    double *Ys = sm;                                    // [NY][NQS][QB][T3C]
    double *Gs = Ys + CF::Y_D;                          // [NG][RING][COLS]
    double *Sv = Gs + CF::G_D;                          // [2][NGRP][STV]
    int32_t *Sc = (int32_t *)(Sv + 2 * NGRP * STV);     // [2][NGRP][2*STC]
    double2 *B2s = (double2 *)(Sv + 2 * NGRP * (STV + STC));  // [QB][NP] (value, derivative)
    double2 *B3s = B2s + QB * NP;                       // [QB][NP]
    double2 *W2s = B3s + QB * NP;                       // [QB][2] (f0,f1),(f2,f3)
    double2 *W3s = W2s + QB * 2;                        // [QB][2]
    double2 *B1w = W3s + QB * 2;                        // [RING][NP] per q1 slot
    double2 *W1b = B1w + RING * NP;                     // [RB][QB][2] rows of the batch

    const int tid = threadIdx.x;
    const int chunk = (int)(blockIdx.x % CF::NCH);
    const int line = a.lines ? a.lines[blockIdx.x / CF::NCH] : (int)(blockIdx.x / CF::NCH);
    const int n1 = (int)a.g.n[0], n2 = (int)a.g.n[1];
    const int i2 = line % n2, i3 = (int)(a.g.slab_b + a.plane_lo) + line / n2;
    const DirView &v1 = a.v[0], &v2 = a.v[1], &v3 = a.v[2];
    const int ni2 = v2.jlen[i2], nq2 = v2.qlen[i2];
    const int ni3 = v3.jlen[i3], nq3 = v3.qlen[i3];
    const int jl2 = v2.jlo[i2], ql2 = v2.qlo[i2], jl3 = v3.jlo[i3], ql3 = v3.qlo[i3];
    const int t3a = chunk * T3C;
    if (t3a >= ni3) return;
    const int nt3 = ni3 - t3a < T3C ? ni3 - t3a : T3C;
    const int64_t plane_stride = a.cv.s3;
    const int *__restrict__ qlo1 = v1.qlo, *__restrict__ qlen1 = v1.qlen, *__restrict__ jlo1 = v1.jlo;
    const int *__restrict__ jlen1 = v1.jlen, *__restrict__ span1 = v1.span;
    const int mq1 = v1.maxq;
    // directions 2 and 3 are fixed for the CTA: stage their tables in shared memory
    for (int x = tid; x < QB * NP; x += NT) {
        const int c = x / NP, r = x % NP;
        B2s[x] = c < nq2 ? __ldg((const double2 *)(v2.B + (int64_t)(ql2 + c) * BS) + r) : make_double2(0.0, 0.0);
        B3s[x] = c < nq3 ? __ldg((const double2 *)(v3.B + (int64_t)(ql3 + c) * BS) + r) : make_double2(0.0, 0.0);
    }
    for (int x = tid; x < QB * 2; x += NT) {
        const int c = x / 2;
        W2s[x] = c < nq2 ? __ldg((const double2 *)(v2.W + ((int64_t)i2 * v2.maxq + c) * 4) + (x & 1)) : make_double2(0.0, 0.0);
        W3s[x] = c < nq3 ? __ldg((const double2 *)(v3.W + ((int64_t)i3 * v3.maxq + c) * 4) + (x & 1)) : make_double2(0.0, 0.0);
    }
    const int off2_0 = v2.span[ql2] - jl2;  // staircase start (dir 2)
    const int off3_0 = v3.span[ql3] - jl3;
    const bool int2 = nq2 == 2 * P + 1 && i2 >= P + 1 && i2 <= n2 - P - 2;  // interior pattern in dir 2
    const bool int3 = nq3 == 2 * P + 1 && i3 >= P + 1 && i3 <= (int)a.g.n[2] - P - 2 && CF::NCH == 1;
    // coefficient field restricted to this line
    const double *__restrict__ Cl = a.cv.ptr(0, 0, ql2, ql3 - a.cq_b);

    // CSR offset of row (0, i2, i3) relative to the first owned row; row i1 adds ni2*ni3*P1(i1)
    const int64_t line_off = a.g.offset(0, i2, i3) - a.val_base;
    const int64_t *__restrict__ pref1 = a.g.pref[0];
    // final-stage thread role: group grp, column colx = t2 + K*t3l
    const int grp = tid / COLS, colx = tid % COLS;
    const int t2c = colx % K, t3c = colx / K;
    const bool fin = grp < NGRP && t2c < ni2 && t3c < nt3;
    int sbuf = 0;  // staging buffer parity

    int q_done = qlo1[0] - 1;  // last q1 whose G is in the ring
    for (int r0 = 0; r0 < n1; r0 += RB) {
        const int rl = (r0 + RB < n1 ? r0 + RB : n1) - 1;
        const int q_hi = qlo1[rl] + qlen1[rl] - 1;
        // direction-1 tables of the batch: basis pairs of the new points, weights of the rows
        for (int x = tid; x < (q_hi - q_done) * NP; x += NT) {
            const int q = q_done + 1 + x / NP, r = x % NP;
            B1w[(q % RING) * NP + r] = __ldg((const double2 *)(v1.B + (int64_t)q * BS) + r);
        }
        for (int x = tid; x < RB * QB * 2; x += NT) {
            const int b = x / (QB * 2), c = (x / 2) % QB, i1 = r0 + b;
            W1b[x] = (i1 < n1 && c < qlen1[i1]) ? __ldg((const double2 *)(v1.W + ((int64_t)i1 * mq1 + c) * 4) + (x & 1))
                                              : make_double2(0.0, 0.0);
        }
        __syncthreads();
        // ---------------- stages 3 and 2 for the new points (q_done, q_hi]
        for (int qs = q_done + 1; qs <= q_hi; qs += NQS) {
            const int nqs = q_hi - qs + 1 < NQS ? q_hi - qs + 1 : NQS;
            // stage 3: fibres (q1s, m, c2), q1s fastest; compile-time divisors only
            const int nfib = NQS * (STIFF ? 3 : 1) * nq2;
            for (int f = tid; f < nfib; f += NT) {
                const int q1s = f % NQS;
                const int rest = f / NQS;
                const int m = STIFF ? rest % 3 : 0;
                const int c2 = STIFF ? rest / 3 : rest;
                if (q1s >= nqs) continue;
                double y0[T3C], y1[T3C];
                #pragma unroll
                for (int t = 0; t < T3C; ++t) { y0[t] = 0.0; y1[t] = 0.0; }
                const int b3 = STIFF && m == 2 ? 1 : 0;
                const double2 w2v = W2s[c2 * 2 + (STIFF && m == 1 ? 1 : 0)];  // (w2^(0,b2), w2^(1,b2))
                // components C_{0m}, C_{1m}, C_{2m} (upper-triangle storage) or c
                const int ka = STIFF ? m : a.comp_mass;
                const int kb = m == 0 ? 1 : (m == 1 ? 3 : 4);
                const int kc = m == 0 ? 2 : (m == 1 ? 4 : 5);
                const int64_t fo = (int64_t)c2 * a.cv.s2 + (int64_t)(qs + q1s) * a.cv.s1;
                const double *pa = Cl + (int64_t)ka * a.cv.cs + fo;
                const double *pb = Cl + (int64_t)kb * a.cv.cs + fo;
                const double *pc = Cl + (int64_t)kc * a.cv.cs + fo;
                const double *B3b = (const double *)B3s + b3;  // value (b3 = 0) or derivative column
                // contribution of point c3 (coefficients ca, cb, cc) at staircase offset O (compile time)
                auto point3 = [&](int c3, double ca, double cb, double cc, auto O) {
                    constexpr int o0 = decltype(O)::value;
                    const double2 w3v = W3s[c3 * 2 + b3];  // (w3^(0,b3), w3^(1,b3))
                    const double *bp = B3b + c3 * 2 * NP;
                    if (STIFF) {
                        const double h1 = w2v.x * w3v.x * ca;                        // l = 0
                        const double h0 = fma(w2v.y * w3v.x, cb, w2v.x * w3v.y * cc);  // l = 1, 2
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) {
                            const int t = o0 + r;
                            if (t >= 0 && t < T3C) {
                                const double bv = bp[2 * r];
                                y1[t] = fma(bv, h1, y1[t]);
                                y0[t] = fma(bv, h0, y0[t]);
                            }
                        }
                    } else {
                        const double h = w2v.x * w3v.x * ca;
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) {
                            const int t = o0 + r;
                            if (t >= 0 && t < T3C) y0[t] = fma(bp[2 * r], h, y0[t]);
                        }
                    }
                };
                if (int3) {
                    // interior, unchunked: all loads hoisted, compile-time staircase (c3+1)/2
                    constexpr int NQ = 2 * P + 1;
                    double ca[NQ], cb[NQ], cc[NQ];
                    #pragma unroll
                    for (int c3 = 0; c3 < NQ; ++c3) {
                        ca[c3] = __ldg(pa);
                        if (STIFF) { cb[c3] = __ldg(pb); cc[c3] = __ldg(pc); }
                        pa += plane_stride;
                        pb += plane_stride;
                        pc += plane_stride;
                    }
                    unroll<NQ>([&](auto C3) {
                        constexpr int c3 = decltype(C3)::value;
                        point3(c3, ca[c3], STIFF ? cb[c3] : 0.0, STIFF ? cc[c3] : 0.0,
                               std::integral_constant<int, (c3 + 1) / 2>{});
                    });
                } else {
                    // boundary or chunked: rolled loop, next point's coefficients prefetched
                    double na = __ldg(pa), nb = STIFF ? __ldg(pb) : 0.0, nc = STIFF ? __ldg(pc) : 0.0;
                    #pragma unroll 1
                    for (int c3 = 0; c3 < nq3; ++c3) {
                        const double ca = na, cb = nb, cc = nc;
                        if (c3 + 1 < nq3) {
                            pa += plane_stride;
                            pb += plane_stride;
                            pc += plane_stride;
                            na = __ldg(pa);
                            if (STIFF) { nb = __ldg(pb); nc = __ldg(pc); }
                        }
                        const int off = v3.span[ql3 + c3] - jl3 - t3a;
                        if (CF::NCH == 1) dispatch<0, K - NP>(off, [&](auto O) { point3(c3, ca, cb, cc, O); });
                        else dispatch<-P, T3C - 1>(off, [&](auto O) { point3(c3, ca, cb, cc, O); });
                    }
                }
                double *Y1 = Ys + (((m * 2 + 1) * NQS + q1s) * QB + c2) * T3C;
                double *Y0 = Ys + (((m * 2 + 0) * NQS + q1s) * QB + c2) * T3C;
                #pragma unroll
                for (int t = 0; t < T3C; ++t) {
                    Y0[t] = y0[t];
                    if (STIFF) Y1[t] = y1[t];
                }
            }
            __syncthreads();
            // stage 2: fibres (t3l, a1, q1s), compile-time divisors only
            const int nfib2 = T3C * (STIFF ? 2 : 1) * nqs;
            for (int f = tid; f < nfib2; f += NT) {
                const int t3l = f % T3C;
                const int rest = f / T3C;
                const int a1 = STIFF ? rest & 1 : 0;
                const int q1s = STIFF ? rest >> 1 : rest;
                const int slot = (qs + q1s) % RING;
                double g0[K], g1[K];
                #pragma unroll
                for (int t = 0; t < K; ++t) { g0[t] = 0.0; g1[t] = 0.0; }
                const double *Yb0 = Ys + ((0 * 2 + a1) * NQS + q1s) * QB * T3C + t3l;  // m = 0 (or mass)
                const double *Yb1 = Ys + ((1 * 2 + a1) * NQS + q1s) * QB * T3C + t3l;  // m = 1
                const double *Yb2 = Ys + ((2 * 2 + a1) * NQS + q1s) * QB * T3C + t3l;  // m = 2
                auto point2 = [&](int c2, auto O) {
                    constexpr int o0 = decltype(O)::value;
                    const double2 *bp = B2s + c2 * NP;
                    if (STIFF) {
                        const double y0 = Yb0[c2 * T3C], y1 = Yb1[c2 * T3C], y2 = Yb2[c2 * T3C];
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) {
                            const double2 b = bp[r];
                            g1[o0 + r] = fma(b.x, y0, g1[o0 + r]);                // b1 = 1: m = 0
                            g0[o0 + r] = fma(b.y, y1, fma(b.x, y2, g0[o0 + r]));  // b1 = 0: m = 1, 2
                        }
                    } else {
                        const double y = Yb0[c2 * T3C];
                        #pragma unroll
                        for (int r = 0; r <= P; ++r) g0[o0 + r] = fma(bp[r].x, y, g0[o0 + r]);
                    }
                };
                if (t3l < nt3) {
                    if (int2) {
                        unroll<2 * P + 1>([&](auto C2) {
                            constexpr int c2 = decltype(C2)::value;
                            point2(c2, std::integral_constant<int, (c2 + 1) / 2>{});
                        });
                    } else {
                        for (int c2 = 0; c2 < nq2; ++c2) {
                            const int off = v2.span[ql2 + c2] - jl2;
                            dispatch<0, K - NP>(off, [&](auto O) { point2(c2, O); });
                        }
                    }
                }
                double *G0 = Gs + ((0 * 2 + a1) * RING + slot) * COLS + K * t3l;
                double *G1 = Gs + ((1 * 2 + a1) * RING + slot) * COLS + K * t3l;
                #pragma unroll
                for (int t = 0; t < K; ++t) {
                    G0[t] = g0[t];
                    if (STIFF) G1[t] = g1[t];
                }
            }
            __syncthreads();
        }
        q_done = q_hi;
        // ---------------- stage 1: row group grp, batch rows bl = grp*NR + k
        const int rg = r0 + grp * NR;
        double acc[NR][K];
        #pragma unroll
        for (int k = 0; k < NR; ++k)
            #pragma unroll
            for (int t = 0; t < K; ++t) acc[k][t] = 0.0;
        const bool interior = rg >= P + 1 && rg + NR - 1 <= n1 - P - 2;
        auto gload = [&](int slot, double &g00, double &g01, double &g10, double &g11) {
            g00 = Gs[((0 * 2 + 0) * RING + slot) * COLS + colx];
            if (STIFF) {
                g01 = Gs[((0 * 2 + 1) * RING + slot) * COLS + colx];
                g10 = Gs[((1 * 2 + 0) * RING + slot) * COLS + colx];
                g11 = Gs[((1 * 2 + 1) * RING + slot) * COLS + colx];
            }
        };
        if (fin && interior) {
            // rows of the group have the interior pattern: 2P+1 points, consecutive rows
            // shifted by 2 points, staircase offset (c+1)/2
            const int qb = qlo1[rg];
            const int slot0 = qb % RING;
            constexpr int UW = 2 * (NR - 1) + 2 * P + 1;
            #pragma unroll
            for (int u = 0; u < UW; ++u) {
                int slot = slot0 + u;
                if (slot >= RING) slot -= RING;
                double g00, g01 = 0.0, g10 = 0.0, g11 = 0.0;
                gload(slot, g00, g01, g10, g11);
                double2 bb[NP];
                #pragma unroll
                for (int r = 0; r <= P; ++r) bb[r] = B1w[slot * NP + r];
                #pragma unroll
                for (int k = 0; k < NR; ++k) {
                    if (u >= 2 * k && u <= 2 * k + 2 * P) {
                        const int c = u - 2 * k;
                        const int o0 = (c + 1) / 2;
                        const double2 *wr = W1b + ((grp * NR + k) * QB + c) * 2;
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
        }
        // write the group's rows (rows touching a boundary span are computed here one at a time)
        #pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int i1 = rg + k;
            const bool live = grp < NGRP && i1 < n1;
            int64_t goff = 0;
            int ni1 = 0;
            if (live) {
                ni1 = jlen1[i1];
                goff = line_off + (int64_t)(ni2 * ni3) * pref1[i1] + ni1 * ni2 * t3a;
            }
            if (fin && live) {
                if (!interior) {
                    double out[K];
                    #pragma unroll
                    for (int t = 0; t < K; ++t) out[t] = 0.0;
                    const int q0 = qlo1[i1], nq1 = qlen1[i1], jl1 = jlo1[i1];
                    for (int c = 0; c < nq1; ++c) {
                        const int q = q0 + c;
                        const int slot = q % RING;
                        const double2 *bp = B1w + slot * NP;
                        const double2 *wr = W1b + ((grp * NR + k) * QB + c) * 2;
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
                            #pragma unroll
                            for (int r = 0; r <= P; ++r) {
                                constexpr int o0 = decltype(O)::value;
                                const double2 b = bp[r];
                                out[o0 + r] = STIFF ? fma(b.x, u0, fma(b.y, u1, out[o0 + r])) : fma(b.x, u0, out[o0 + r]);
                            }
                        });
                    }
                    #pragma unroll
                    for (int t = 0; t < K; ++t) acc[k][t] = out[t];
                }
                // stage in CSR order of the row's chunk: t1 + ni1 * (t2 + ni2 * t3l), shifted so
                // that the 16-B aligned part of the global segment starts on a 16-B boundary
                const int colbase = jlo1[i1] + n1 * ((jl2 + t2c) + n2 * (jl3 + t3a + t3c));
                const int e0 = ni1 * (t2c + ni2 * t3c);
                double *sv = Sv + (sbuf * NGRP + grp) * STV + (int)(goff & 1);
                int32_t *sc = Sc + (sbuf * NGRP + grp) * 2 * STC + (int)(goff & 3);
                #pragma unroll
                for (int t = 0; t < K; ++t)
                    if (t < ni1) {
                        sv[e0 + t] = acc[k][t];
                        sc[e0 + t] = colbase + t;
                    }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            // one thread per group issues the TMA bulk copies of its row segment
            if (live && colx == 0) {
                const int len = ni1 * ni2 * nt3;
                const double *sv = Sv + (sbuf * NGRP + grp) * STV + (int)(goff & 1);
                const int32_t *sc = Sc + (sbuf * NGRP + grp) * 2 * STC + (int)(goff & 3);
                double *dv = a.val + goff;
                const int hv = (int)(goff & 1);              // unaligned head (values)
                const int nbv = (len - hv) & ~1;             // bulk elements
                if (hv && len > 0) dv[0] = sv[0];
                if (nbv > 0) bulk_s2g(dv + hv, sv + hv, (unsigned)nbv * 8u);
                for (int e = hv + nbv; e < len; ++e) dv[e] = sv[e];
                if (a.col) {
                    int32_t *dc = a.col + goff;
                    const int hc = (4 - (int)(goff & 3)) & 3;
                    const int hcn = hc < len ? hc : len;
                    const int nbc = (len - hcn) & ~3;
                    for (int e = 0; e < hcn; ++e) dc[e] = sc[e];
                    if (nbc > 0) bulk_s2g(dc + hcn, sc + hcn, (unsigned)nbc * 4u);
                    for (int e = hcn + nbc; e < len; ++e) dc[e] = sc[e];
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                // the other buffer is reused next: its copies (one group back) must have read smem
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
            sbuf ^= 1;
            __syncthreads();
        }
    }
    if (colx == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int P, bool STIFF>
wq_status launch_tile_p(wq_plan_s *Pl, double *val, int32_t *col, int64_t pl_lo, int64_t pl_hi, int64_t val_base,
                        cudaStream_t s, const int32_t *list = nullptr, int64_t n_list = 0) {
    using CF = Cfg<P, STIFF>;
    TileArgs a;
    a.g.init(Pl);
    for (int l = 0; l < 3; ++l) a.v[l] = Pl->dir[l];
    a.cv = STIFF && Pl->coef_std ? Pl->cview_std : Pl->cview;  // stiffness: standard-layout copy if the plan keeps one
    a.cq_b = Pl->cq_b;
    a.comp_mass = Pl->comp_mass;
    a.val = val;
    a.col = col;
    a.val_base = val_base;
    a.plane_lo = list ? 0 : pl_lo;
    a.lines = list;
    const int64_t lines = list ? n_list : Pl->dir[1].n * (pl_hi - pl_lo);
    const int64_t blocks = lines * CF::NCH;
    wq_smem_attr((const void *)k_tile<P, STIFF>, CF::SMEM);
    if (blocks > 0) {
        k_tile<P, STIFF><<<(unsigned)blocks, CF::NT, CF::SMEM, s>>>(a);
        wq_count_launches(1);
    }
    return wq_cuda_status(cudaGetLastError(), "tile assembly kernel");
}

template <bool STIFF>
wq_status dispatch_p(wq_plan_s *Pl, double *val, int32_t *col, int64_t lo, int64_t hi, int64_t vb, cudaStream_t s,
                     const int32_t *list = nullptr, int64_t n_list = 0) {
    switch (Pl->p) {
    case 1: return launch_tile_p<1, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 2: return launch_tile_p<2, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 3: return launch_tile_p<3, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 4: return launch_tile_p<4, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 5: return launch_tile_p<5, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 6: return launch_tile_p<6, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 7: return launch_tile_p<7, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 8: return launch_tile_p<8, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 9: return launch_tile_p<9, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    case 10: return launch_tile_p<10, STIFF>(Pl, val, col, lo, hi, vb, s, list, n_list);
    }
    wq_set_error("tile kernel: unsupported degree");
    return WQ_EINVAL;
}

}  // namespace

bool tile_supported(const wq_plan_s *P, int matrix) {
    if (P->d != 3 || P->p < 1 || P->p > 10) return false;
    for (int l = 0; l < 3; ++l)
        if (P->dir[l].maxq > 3 * P->p + 1) return false;  // a support holding both boundary spans
    return true;
}

wq_status launch_assemble_tile(wq_plan_s *P, int matrix, double *val, int32_t *col, int64_t plane_lo,
                               int64_t plane_hi, int64_t val_base, cudaStream_t s) {
    if (!tile_supported(P, matrix)) {
        wq_set_error("tile kernel not available for this plan");
        return WQ_EINVAL;
    }
    return matrix == WQ_MASS ? dispatch_p<false>(P, val, col, plane_lo, plane_hi, val_base, s)
                             : dispatch_p<true>(P, val, col, plane_lo, plane_hi, val_base, s);
}
