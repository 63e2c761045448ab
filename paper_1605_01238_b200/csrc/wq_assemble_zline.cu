// wq_assemble_zline.cu -- host side of the z-line kernel (WQ_KERNEL_ZLINE): applicability, the
// one-time check of the device rules (row staircase types, uniform-mesh rules, reading R16) and
// the launch dispatch to the per-degree translation units wq_zline_deg<p>.cu.  The kernel itself
// and its design notes are in wq_zline.cuh.
#include "wq_zline.cuh"

unsigned long long *g_zprof = nullptr;

bool zline_supported_p(int d, int p, const int64_t *n, const int32_t *maxq, int64_t n2l, int64_t nq2l) {
    if (d != 3 || !z_encode_fn()) return false;
    for (int l = 0; l < 3; ++l)
        if (maxq[l] > 3 * p + 1 || n[l] < 2) return false;  // a support holding both boundary spans
    return fits_z<false>(p, n2l, nq2l) && fits_z<true>(p, n2l, nq2l);
}

namespace {
// Uniform-mesh check of the device-computed rules (once per plan: the rules are a pure function of
// the plan's knots and degree): every interior row of every direction must carry the same weights
// on its points c = 0..2p and the same basis values at points of the same parity, to 1e-13 relative
// (uniform knots k/E agree to ~3e-14 because of the FP64 rounding of the knots, exactly when E is a
// power of two).  On success the representative row n/2 fills the kernel's uniform tables.
#define ZFAIL(...) do { if (getenv("WQ_DEBUG")) { fprintf(stderr, "[wq] uniform rules rejected: " __VA_ARGS__); fprintf(stderr, "\n"); } return false; } while (0)
template <int PP>
bool z_types_match(const std::vector<int32_t> &qlo, const std::vector<int32_t> &qlen, const std::vector<int32_t> &jlo,
                   const std::vector<int32_t> &span, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        const int t = ZTy<PP>::type(i, n);
        if (qlen[i] != ZTy<PP>::nq(t)) return false;
        for (int c = 0; c < qlen[i]; ++c)
            if (span[qlo[i] + c] - jlo[i] != ZTy<PP>::off(t, c)) return false;
    }
    return true;
}
bool z_fetch_uniform(wq_plan_s *P, ZUni &U, bool &types_ok, bool &cuda_ok) {
    const int p = P->p, K = 2 * p + 1, bs = wq_bstride(p);
    types_ok = false;
    cuda_ok = false;
    if (p > WQ_ZPMAX) ZFAIL("p");
    memset(&U, 0, sizeof(U));
    // staircase types of every row (the boundary-line kernel unrolls them at compile time)
    for (int l = 0; l < 3; ++l) {
        const DirView &v = P->dir[l];
        std::vector<int32_t> qlo(v.n), qlen(v.n), jlo(v.n), span(v.nq);
        if (cudaMemcpy(qlo.data(), v.qlo, v.n * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(qlen.data(), v.qlen, v.n * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(jlo.data(), v.jlo, v.n * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(span.data(), v.span, v.nq * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
            return false;
        const bool ok = p == 2 ? z_types_match<2>(qlo, qlen, jlo, span, v.n)
                      : p == 3 ? z_types_match<3>(qlo, qlen, jlo, span, v.n)
                      : p == 4 ? z_types_match<4>(qlo, qlen, jlo, span, v.n)
                      : p == 5 ? z_types_match<5>(qlo, qlen, jlo, span, v.n)
                               : z_types_match<6>(qlo, qlen, jlo, span, v.n);
        if (!ok) { cuda_ok = true; ZFAIL("dir %d: row staircase types do not match", l); }
    }
    types_ok = true;
    cuda_ok = true;
    for (int l = 0; l < 3; ++l) {
        const DirView &v = P->dir[l];
        const int64_t n = v.n, nq = v.nq;
        if (n - 1 - 2 * p < 2 * p) ZFAIL("dir %d: no row with uniform rules", l);
        std::vector<double> W((size_t)n * v.maxq * 4), B((size_t)nq * bs);
        std::vector<int32_t> qlo(n), qlen(n), jlo(n), span(nq);
        if (cudaMemcpy(W.data(), v.W, W.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(B.data(), v.B, B.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(qlo.data(), v.qlo, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(qlen.data(), v.qlen, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(jlo.data(), v.jlo, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(span.data(), v.span, nq * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
            cuda_ok = false;
            return false;
        }
        const int64_t ir = n / 2;  // in [2p, n-1-2p]
        const double *Wr = W.data() + (size_t)ir * v.maxq * 4;
        double wsc[4] = {0, 0, 0, 0}, bsc[2] = {0, 0};
        for (int c = 0; c < K; ++c)
            for (int f = 0; f < 4; ++f) wsc[f] = std::max(wsc[f], std::fabs(Wr[c * 4 + f]));
        for (int par = 0; par < 2; ++par)
            for (int r = 0; r <= p; ++r)
                for (int h = 0; h < 2; ++h) bsc[h] = std::max(bsc[h], std::fabs(B[(size_t)(qlo[ir] + par) * bs + 2 * r + h]));
        const double tol = 1e-13;
        for (int64_t i = 2 * p; i <= n - 1 - 2 * p; ++i) {
            if (qlen[i] != K) ZFAIL("dir %d row %lld: #Q %d", l, (long long)i, qlen[i]);
            const double *Wi = W.data() + (size_t)i * v.maxq * 4;
            for (int c = 0; c < K; ++c) {
                if (span[qlo[i] + c] - jlo[i] != (c + 1) / 2) ZFAIL("dir %d row %lld: staircase", l, (long long)i);
                for (int f = 0; f < 4; ++f)
                    if (std::fabs(Wi[c * 4 + f] - Wr[c * 4 + f]) > tol * wsc[f])
                        ZFAIL("dir %d row %lld c %d f %d: w %.17g vs %.17g", l, (long long)i, c, f, Wi[c * 4 + f], Wr[c * 4 + f]);
                for (int r = 0; r <= p; ++r)
                    for (int h = 0; h < 2; ++h)
                        if (std::fabs(B[(size_t)(qlo[i] + c) * bs + 2 * r + h] -
                                      B[(size_t)(qlo[ir] + (c & 1)) * bs + 2 * r + h]) > tol * bsc[h])
                            ZFAIL("dir %d row %lld c %d r %d h %d: B %.17g vs %.17g", l, (long long)i, c, r, h,
                                  B[(size_t)(qlo[i] + c) * bs + 2 * r + h], B[(size_t)(qlo[ir] + (c & 1)) * bs + 2 * r + h]);
            }
        }
        for (int c = 0; c < K; ++c)
            for (int f = 0; f < 4; ++f) U.w[l][c][f] = Wr[c * 4 + f];
        for (int par = 0; par < 2; ++par)
            for (int r = 0; r <= p; ++r)
                for (int h = 0; h < 2; ++h) U.b[l][par][r][h] = B[(size_t)(qlo[ir] + par) * bs + 2 * r + h];
    }
    return true;
}
}  // namespace

// Once per plan, after the rules have been built and synchronised (wq_plan_create): verify the row
// staircase types the kernel compiles in, and fetch the uniform-mesh rules (reading R16).  A type
// mismatch disables the z-line kernel for the plan (AUTO then runs another kernel); a CUDA failure
// is WQ_ECUDA.
wq_status zline_prepare(wq_plan_s *P) {
    static_assert(sizeof(ZUni) <= sizeof(P->zuni_buf), "uniform table buffer");
    ZUni U;
    bool types_ok = false, cuda_ok = false;
    bool ok = z_fetch_uniform(P, U, types_ok, cuda_ok);
    if (!cuda_ok) {
        wq_set_error("z-line preparation: device -> host copy of the rules failed");
        return WQ_ECUDA;
    }
    if (!types_ok) {
        P->zline_ok = 0;
        return WQ_OK;
    }
    if (getenv("WQ_ZLINE_NO_UNIFORM")) ok = false;
    P->zuni_state = ok ? 1 : -1;
    if (ok) memcpy(P->zuni_buf, &U, sizeof(U));
    return WQ_OK;
}

wq_status launch_assemble_zline(wq_plan_s *P, int cls, const int32_t *lines, int64_t n_lines, int64_t pl_lo,
                                int64_t pl_hi, double *val, int32_t *col, int64_t val_base, cudaStream_t s) {
    if (!P->zline_ok || P->zuni_state == 0) {
        wq_set_error("z-line kernel not prepared for this plan");
        return WQ_EINVAL;
    }
    if (n_lines <= 0) return WQ_OK;
    ZUni U;
    memcpy(&U, P->zuni_buf, sizeof(U));
    const bool cu = P->zuni_state == 1;
    // PU keeps each stage-A lane's tables in registers: one fibre per lane (a single stage-A pass)
    const bool one_pass = P->p <= 4;  // ZCfg<p, false>::NPASS == 1 (3 (2p+1) <= 32)
    static_assert(ZCfg<4, false>::NPASS == 1 && ZCfg<5, false>::NPASS > 1, "single-pass degrees");
    const bool bnd = cls == 2, pu = cls == 0 && cu && one_pass;
    switch (P->p) {
    case 2: return zline_launch_deg_2(P, bnd, pu, cu, lines, n_lines, pl_lo, pl_hi, val, col, val_base, &U, s);
    case 3: return zline_launch_deg_3(P, bnd, pu, cu, lines, n_lines, pl_lo, pl_hi, val, col, val_base, &U, s);
    case 4: return zline_launch_deg_4(P, bnd, pu, cu, lines, n_lines, pl_lo, pl_hi, val, col, val_base, &U, s);
    case 5: return zline_launch_deg_5(P, bnd, pu, cu, lines, n_lines, pl_lo, pl_hi, val, col, val_base, &U, s);
    case 6: return zline_launch_deg_6(P, bnd, pu, cu, lines, n_lines, pl_lo, pl_hi, val, col, val_base, &U, s);
    }
    wq_set_error("z-line kernel not available for this degree");
    return WQ_EINVAL;
}

// debug only (-DWQ_ZL_PROF, WQ_ZL_PROF=1): per-warp cycle accounting of the last z-line launches,
// [class uni/int/bnd][148 blocks][32 warps][total, wait1, wait2]
extern "C" int wq_debug_zprof(unsigned long long *host, int n) {
    if (!g_zprof) return -1;
    cudaDeviceSynchronize();
    return (int)cudaMemcpy(host, g_zprof, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
}
