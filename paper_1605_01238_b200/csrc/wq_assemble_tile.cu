// wq_assemble_tile.cu -- step 7, sum-factorised row-tile kernel (WQ_KERNEL_TILE)
// for d = 3, compile-time degree P.  Eq. sumfactorization / Alg. 3
// (P:859-870), re-organised so that the rows of a tile share every stage but
// the last:
//
//   CTA = one line (i2, i3) of the row grid, a batch of RB consecutive rows
//         i1, and a chunk of T3C trial indices t3 (t3 is slowest in a CSR row).
//   stage 3 (+ pointwise test weights of directions 2, 3), per q1 of the
//         tile's q1-window and per c2:
//     stiffness, chains (m, a1), m = trial-derivative direction, a1 = [l = 1]:
//       Y_{m,a1}(q1,c2,t3) = sum_{c3} B3^{[m=3]}_{t3}(c3) *
//                            sum_{l: [l=1]=a1} w2^{([l=2],[m=2])}(c2) w3^{([l=3],[m=3])}(c3) C_lm(q1,c2,c3)
//     mass: Y(q1,c2,t3) = sum_{c3} B3_{t3}(c3) w2^(0,0)(c2) w3^(0,0)(c3) c(q1,c2,c3)
//   stage 2: G[b1][a1](q1,t2,t3) = sum_{c2} (B2^{[m=2]}_{t2} Y_{m,a1}) summed over the m
//         with [m=1] = b1   (mass: G = sum_{c2} B2_{t2} Y)
//   stage 1 (per row i1):  out(t1,t2,t3) = sum_{c1} B1^0_{t1}(c1) U^0(c1) + B1^1_{t1}(c1) U^1(c1)
//         U^0 = w1^(0,0) G[0][0] + w1^(1,0) G[0][1],  U^1 = w1^(0,1) G[1][0] + w1^(1,1) G[1][1]
//         (mass: out = sum_{c1} B1_{t1}(c1) w1^(0,0)(c1) G).
// (a, b) = (test, trial) derivative order (reading R3); directions 1..3 are
// indices 0..2 in the code.  Tables are dense (zero outside the B-spline
// support) so all inner loops have compile-time trip counts.
#include "wq_rows.cuh"

namespace {

struct TileArgs {
    RowGeo g;
    DirView v[3];
    const double *coef;
    int64_t nq1, nq2;     // coefficient strides
    int64_t cq_b;
    int64_t npts;
    int comp_mass;
    double *val;
    int32_t *col;
    int64_t val_base;
    int64_t plane_lo;     // first slab plane (relative) of this launch
    int n_batch;          // row batches per line
    int n_chunk;          // t3 chunks
};

template <int P, bool STIFF>
struct Cfg {
    static constexpr int K = 2 * P + 1;      // max #I
    static constexpr int QB = 3 * P + 1;     // max #Q (n_EL >= P + 2)
    static constexpr int NY = STIFF ? 6 : 1; // chains through stage 3
    static constexpr int NG = STIFF ? 4 : 1; // merged chains after stage 2
    static constexpr int NQS = 8;            // q1 sub-batch of stage 3
    static constexpr int NW1 = STIFF ? 4 : 1;
    __host__ __device__ static constexpr size_t ev(size_t x) { return (x + 1) & ~(size_t)1; }  // 16-B aligned regions
    __host__ __device__ static constexpr size_t bytes_for(int RB, int T3C) {
        size_t W = QB + 2 * RB + P;
        size_t d = ev((size_t)NY * NQS * QB * T3C)          // Y
                   + ev((size_t)NG * W * K * T3C)           // G
                   + (size_t)RB * K * QB * 2                // B1 pairs per row
                   + (size_t)RB * QB * 4                    // w1 per row
                   + 2 * ((size_t)K * QB * 2 + 4 * QB);     // B2, w2, B3, w3
        return d * sizeof(double);
    }
    static constexpr size_t LIMIT = 200 * 1024;
    // largest T3C (fewest t3 chunks), then largest RB in {8, 4, 2}, that fits
    __host__ __device__ static constexpr int pick(bool want_rb) {
        for (int nch = 1; nch <= K; ++nch) {
            int t3c = (K + nch - 1) / nch;
            for (int rb = 8; rb >= 2; rb /= 2)
                if (bytes_for(rb, t3c) <= LIMIT) return want_rb ? rb : t3c;
        }
        return want_rb ? 2 : 1;
    }
    static constexpr int RB = pick(true);
    static constexpr int T3C = pick(false);
    static constexpr int W = QB + 2 * RB + P;
    static constexpr size_t SMEM = bytes_for(RB, T3C);
    static_assert(SMEM <= 227 * 1024, "tile kernel shared memory");
};

__device__ __forceinline__ int comp_ix(int l, int m) {  // upper-triangle index, d = 3
    if (l > m) { int t = l; l = m; m = t; }
    return l * 3 - l * (l - 1) / 2 + (m - l);
}

// dense (value, derivative) pair of B_{j}(x_q) from the compact table
__device__ __forceinline__ double2 bpair(const DirView &v, int P, int64_t j, int64_t q) {
    int loc = (int)(j - v.span[q]);
    if (loc < 0 || loc > P) return make_double2(0.0, 0.0);
    const double *b = v.B + q * WQ_BROWS * (P + 1);
    return make_double2(b[loc], b[P + 1 + loc]);
}

template <int P, bool STIFF>
__global__ void __launch_bounds__(256) k_tile(TileArgs a) {
    using CF = Cfg<P, STIFF>;
    constexpr int K = CF::K, QB = CF::QB, NY = CF::NY, NG = CF::NG, NQS = CF::NQS;
    constexpr int RB = CF::RB, T3C = CF::T3C, W = CF::W;
    extern __shared__ __align__(16) double sm[];
    double *Ys = sm;                                        // [NY][NQS][QB][T3C]
    double *Gs = Ys + CF::ev(NY * NQS * QB * T3C);          // [NG][W][K][T3C]
    double2 *B1s = (double2 *)(Gs + CF::ev(NG * W * K * T3C)); // [RB][K][QB]
    double *w1s = (double *)(B1s + RB * K * QB);       // [RB][QB][4]
    double2 *B2s = (double2 *)(w1s + RB * QB * 4);     // [K][QB]
    double *w2s = (double *)(B2s + K * QB);            // [4][QB]
    double2 *B3s = (double2 *)(w2s + 4 * QB);          // [K][QB]
    double *w3s = (double *)(B3s + K * QB);            // [4][QB]

    const int tid = threadIdx.x;
    // ---- tile coordinates
    int64_t bid = blockIdx.x;
    const int chunk = (int)(bid % a.n_chunk);
    bid /= a.n_chunk;
    const int batch = (int)(bid % a.n_batch);
    const int64_t line = bid / a.n_batch;
    const int64_t n1 = a.g.n[0], n2 = a.g.n[1];
    const int64_t i2 = line % n2, i3 = a.g.slab_b + a.plane_lo + line / n2;
    const int64_t r0 = (int64_t)batch * RB;
    if (r0 >= n1) return;
    const int nrows = (int)(n1 - r0 < RB ? n1 - r0 : RB);
    const DirView &v1 = a.v[0], &v2 = a.v[1], &v3 = a.v[2];
    const int ni2 = v2.jlen[i2], nq2 = v2.qlen[i2];
    const int ni3 = v3.jlen[i3], nq3 = v3.qlen[i3];
    const int64_t jl2 = v2.jlo[i2], ql2 = v2.qlo[i2], jl3 = v3.jlo[i3], ql3 = v3.qlo[i3];
    const int t3a = chunk * T3C;
    if (t3a >= ni3) return;
    const int nt3 = ni3 - t3a < T3C ? ni3 - t3a : T3C;
    const int64_t qw0 = v1.qlo[r0];
    const int nw = (int)(v1.qlo[r0 + nrows - 1] + v1.qlen[r0 + nrows - 1] - qw0);

    // ---- tables
    for (int x = tid; x < K * QB; x += blockDim.x) {
        int t = x / QB, c = x % QB;
        B2s[x] = (t < ni2 && c < nq2) ? bpair(v2, P, jl2 + t, ql2 + c) : make_double2(0.0, 0.0);
        int t3 = t3a + t;
        B3s[x] = (t < nt3 && c < nq3) ? bpair(v3, P, jl3 + t3, ql3 + c) : make_double2(0.0, 0.0);
    }
    for (int x = tid; x < 4 * QB; x += blockDim.x) {
        int f = x / QB, c = x % QB;
        w2s[x] = c < nq2 ? v2.W[(i2 * 4 + f) * v2.maxq + c] : 0.0;
        w3s[x] = c < nq3 ? v3.W[(i3 * 4 + f) * v3.maxq + c] : 0.0;
    }
    for (int x = tid; x < RB * K * QB; x += blockDim.x) {
        int b = x / (K * QB), t = (x / QB) % K, c = x % QB;
        double2 val = make_double2(0.0, 0.0);
        if (b < nrows) {
            int64_t i1 = r0 + b;
            if (t < v1.jlen[i1] && c < v1.qlen[i1]) val = bpair(v1, P, v1.jlo[i1] + t, v1.qlo[i1] + c);
        }
        B1s[x] = val;
    }
    for (int x = tid; x < RB * QB * 4; x += blockDim.x) {
        int b = x / (QB * 4), c = (x / 4) % QB, f = x % 4;
        double val = 0.0;
        if (b < nrows) {
            int64_t i1 = r0 + b;
            if (c < v1.qlen[i1]) val = v1.W[(i1 * 4 + f) * v1.maxq + c];
        }
        w1s[x] = val;
    }
    __syncthreads();

    const double *__restrict__ C = a.coef;
    const int64_t plane_stride = a.nq1 * a.nq2;
    // ---- stages 3 and 2 over the q1 window, in sub-batches of NQS
    for (int qs0 = 0; qs0 < nw; qs0 += NQS) {
        const int nqs = nw - qs0 < NQS ? nw - qs0 : NQS;
        // stage 3: fibers (q1s, c2, m)
        const int nfib = nqs * nq2 * (STIFF ? 3 : 1);
        for (int f = tid; f < nfib; f += blockDim.x) {
            const int q1s = f % nqs;
            const int c2 = (f / nqs) % nq2;
            const int m = STIFF ? f / (nqs * nq2) : 0;
            const int64_t q1 = qw0 + qs0 + q1s;
            const int64_t pbase = q1 + a.nq1 * (ql2 + c2) + plane_stride * (ql3 - a.cq_b);
            double y0[T3C], y1[T3C];
            #pragma unroll
            for (int t = 0; t < T3C; ++t) { y0[t] = 0.0; y1[t] = 0.0; }
            if (STIFF) {
                const int b2 = (m == 1) ? 2 : 0, b3 = (m == 2) ? 2 : 0;  // 2*[trial derivative]
                const double wa2 = w2s[(0 + b2) * QB + c2];  // l = 0: w2^(0, [m==1])
                const double wb2 = w2s[(1 + b2) * QB + c2];  // l = 1: w2^(1, [m==1])
                const double wc2 = w2s[(0 + b2) * QB + c2];  // l = 2: w2^(0, [m==1])
                const double *Ca = C + (int64_t)comp_ix(0, m) * a.npts + pbase;
                const double *Cb = C + (int64_t)comp_ix(1, m) * a.npts + pbase;
                const double *Cc = C + (int64_t)comp_ix(2, m) * a.npts + pbase;
                for (int c3 = 0; c3 < nq3; ++c3) {
                    const int64_t o = plane_stride * c3;
                    const double ca = __ldg(Ca + o), cb = __ldg(Cb + o), cc = __ldg(Cc + o);
                    const double h1 = wa2 * w3s[(0 + b3) * QB + c3] * ca;
                    const double h0 = wb2 * w3s[(0 + b3) * QB + c3] * cb + wc2 * w3s[(1 + b3) * QB + c3] * cc;
                    #pragma unroll
                    for (int t = 0; t < T3C; ++t) {
                        const double2 bb = B3s[t * QB + c3];
                        const double B = m == 2 ? bb.y : bb.x;
                        y1[t] = fma(B, h1, y1[t]);
                        y0[t] = fma(B, h0, y0[t]);
                    }
                }
                #pragma unroll
                for (int t = 0; t < T3C; ++t) {
                    Ys[(((m * 2 + 1) * NQS + q1s) * QB + c2) * T3C + t] = y1[t];
                    Ys[(((m * 2 + 0) * NQS + q1s) * QB + c2) * T3C + t] = y0[t];
                }
            } else {
                const double w2v = w2s[c2];
                const double *Cm = C + (int64_t)a.comp_mass * a.npts + pbase;
                for (int c3 = 0; c3 < nq3; ++c3) {
                    const double h = w2v * w3s[c3] * __ldg(Cm + plane_stride * c3);
                    #pragma unroll
                    for (int t = 0; t < T3C; ++t) y0[t] = fma(B3s[t * QB + c3].x, h, y0[t]);
                }
                #pragma unroll
                for (int t = 0; t < T3C; ++t) Ys[(q1s * QB + c2) * T3C + t] = y0[t];
            }
        }
        __syncthreads();
        // stage 2: fibers (q1s, t3, a1) -> G[b1][a1]
        const int nfib2 = nqs * T3C * (STIFF ? 2 : 1);
        for (int f = tid; f < nfib2; f += blockDim.x) {
            const int q1s = f % nqs;
            const int t3 = (f / nqs) % T3C;
            const int a1 = STIFF ? f / (nqs * T3C) : 0;
            const int qw = qs0 + q1s;
            double g0[K], g1[K];
            #pragma unroll
            for (int t = 0; t < K; ++t) { g0[t] = 0.0; g1[t] = 0.0; }
            if (STIFF) {
                const double *Y0 = Ys + ((0 * 2 + a1) * NQS + q1s) * QB * T3C + t3;  // m = 1 (dir index 0)
                const double *Y1 = Ys + ((1 * 2 + a1) * NQS + q1s) * QB * T3C + t3;  // m = 2
                const double *Y2 = Ys + ((2 * 2 + a1) * NQS + q1s) * QB * T3C + t3;  // m = 3
                for (int c2 = 0; c2 < nq2; ++c2) {
                    const double y0 = Y0[c2 * T3C], y1 = Y1[c2 * T3C], y2 = Y2[c2 * T3C];
                    #pragma unroll
                    for (int t = 0; t < K; ++t) {
                        const double2 bb = B2s[t * QB + c2];
                        g1[t] = fma(bb.x, y0, g1[t]);                 // b1 = 1: m = 1, trial value in dir 2
                        g0[t] = fma(bb.y, y1, fma(bb.x, y2, g0[t]));  // b1 = 0: m = 2 (B2'), m = 3 (B2)
                    }
                }
                #pragma unroll
                for (int t = 0; t < K; ++t) {
                    Gs[(((0 * 2 + a1) * W + qw) * K + t) * T3C + t3] = g0[t];
                    Gs[(((1 * 2 + a1) * W + qw) * K + t) * T3C + t3] = g1[t];
                }
            } else {
                const double *Y0 = Ys + q1s * QB * T3C + t3;
                for (int c2 = 0; c2 < nq2; ++c2) {
                    const double y = Y0[c2 * T3C];
                    #pragma unroll
                    for (int t = 0; t < K; ++t) g0[t] = fma(B2s[t * QB + c2].x, y, g0[t]);
                }
                #pragma unroll
                for (int t = 0; t < K; ++t) Gs[(qw * K + t) * T3C + t3] = g0[t];
            }
        }
        __syncthreads();
    }
    // ---- stage 1 per row: items (row b, t2, t3)
    const int nitems = nrows * ni2 * nt3;
    for (int it = tid; it < nitems; it += blockDim.x) {
        const int t3 = it % nt3;
        const int t2 = (it / nt3) % ni2;
        const int b = it / (nt3 * ni2);
        const int64_t i1 = r0 + b;
        const int ni1 = v1.jlen[i1], nq1 = v1.qlen[i1];
        const int qoff = (int)(v1.qlo[i1] - qw0);
        double out[K];
        #pragma unroll
        for (int t = 0; t < K; ++t) out[t] = 0.0;
        const double2 *B1r = B1s + b * K * QB;
        const double *w1r = w1s + b * QB * 4;
        for (int c1 = 0; c1 < nq1; ++c1) {
            const int qw = qoff + c1;
            if (STIFF) {
                const double g00 = Gs[(((0 * 2 + 0) * W + qw) * K + t2) * T3C + t3];
                const double g01 = Gs[(((0 * 2 + 1) * W + qw) * K + t2) * T3C + t3];
                const double g10 = Gs[(((1 * 2 + 0) * W + qw) * K + t2) * T3C + t3];
                const double g11 = Gs[(((1 * 2 + 1) * W + qw) * K + t2) * T3C + t3];
                const double2 wA = *(const double2 *)(w1r + c1 * 4);      // w^(0,0), w^(1,0)
                const double2 wB = *(const double2 *)(w1r + c1 * 4 + 2);  // w^(0,1), w^(1,1)
                const double u0 = fma(wA.x, g00, wA.y * g01);
                const double u1 = fma(wB.x, g10, wB.y * g11);
                #pragma unroll
                for (int t = 0; t < K; ++t) {
                    const double2 bb = B1r[t * QB + c1];
                    out[t] = fma(bb.x, u0, fma(bb.y, u1, out[t]));
                }
            } else {
                const double g = Gs[(qw * K + t2) * T3C + t3];
                const double u = w1r[c1 * 4] * g;
                #pragma unroll
                for (int t = 0; t < K; ++t) out[t] = fma(B1r[t * QB + c1].x, u, out[t]);
            }
        }
        const int64_t off = a.g.offset(i1, i2, i3) - a.val_base;
        const int tt3 = t3a + t3;
        const int64_t base = off + (int64_t)ni1 * (t2 + (int64_t)ni2 * tt3);
        const int64_t jl1 = v1.jlo[i1];
        const int64_t colbase = n1 * ((jl2 + t2) + n2 * (jl3 + tt3));
        #pragma unroll
        for (int t = 0; t < K; ++t) {
            if (t < ni1) {
                a.val[base + t] = out[t];
                if (a.col) a.col[base + t] = (int32_t)(jl1 + t + colbase);
            }
        }
    }
}

template <int P, bool STIFF>
wq_status launch_tile_p(wq_plan_s *Pl, double *val, int32_t *col, int64_t pl_lo, int64_t pl_hi, int64_t val_base,
                        cudaStream_t s) {
    using CF = Cfg<P, STIFF>;
    TileArgs a;
    a.g.init(Pl);
    for (int l = 0; l < 3; ++l) a.v[l] = Pl->dir[l];
    a.coef = Pl->coef;
    a.nq1 = Pl->dir[0].nq;
    a.nq2 = Pl->dir[1].nq;
    a.cq_b = Pl->cq_b;
    a.npts = Pl->coef_points;
    a.comp_mass = Pl->need_stiff ? Pl->ncomp_s : 0;
    a.val = val;
    a.col = col;
    a.val_base = val_base;
    a.plane_lo = pl_lo;
    const int64_t n1 = Pl->dir[0].n;
    a.n_batch = (int)((n1 + CF::RB - 1) / CF::RB);
    a.n_chunk = (CF::K + CF::T3C - 1) / CF::T3C;
    const int64_t lines = Pl->dir[1].n * (pl_hi - pl_lo);
    const int64_t blocks = lines * a.n_batch * a.n_chunk;
    static bool set = false;
    if (!set) {
        cudaFuncSetAttribute(k_tile<P, STIFF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
        set = true;
    }
    if (blocks > 0) {
        k_tile<P, STIFF><<<(unsigned)blocks, 256, CF::SMEM, s>>>(a);
        wq_count_launches(1);
    }
    return wq_cuda_status(cudaGetLastError(), "tile assembly kernel");
}

template <bool STIFF>
wq_status dispatch(wq_plan_s *Pl, double *val, int32_t *col, int64_t lo, int64_t hi, int64_t vb, cudaStream_t s) {
    switch (Pl->p) {
    case 1: return launch_tile_p<1, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 2: return launch_tile_p<2, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 3: return launch_tile_p<3, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 4: return launch_tile_p<4, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 5: return launch_tile_p<5, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 6: return launch_tile_p<6, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 7: return launch_tile_p<7, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 8: return launch_tile_p<8, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 9: return launch_tile_p<9, STIFF>(Pl, val, col, lo, hi, vb, s);
    case 10: return launch_tile_p<10, STIFF>(Pl, val, col, lo, hi, vb, s);
    }
    wq_set_error("tile kernel: unsupported degree");
    return WQ_EINVAL;
}

}  // namespace

bool tile_supported(const wq_plan_s *P, int matrix) {
    (void)matrix;
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
    return matrix == WQ_MASS ? dispatch<false>(P, val, col, plane_lo, plane_hi, val_base, s)
                             : dispatch<true>(P, val, col, plane_lo, plane_hi, val_base, s);
}
