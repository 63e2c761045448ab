// wq_api.cu -- the C-ABI of include/wq.h: validation, plan sizing and
// allocation, stream-ordered launches of the kernels, error reporting, and
// the host-buffer end-to-end call.  Host logic only; every arithmetic step of
// the WQ path runs in the CUDA kernels of this directory.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <atomic>
#include <vector>
#include <algorithm>
#include <mutex>
#include <set>
#include "wq_internal.cuh"

namespace {
thread_local std::string g_err;

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int64_t host_knot_pos(int64_t e, int64_t E, int p, int64_t nq) {
    if (e <= 0) return 0;
    if (e >= E) return nq - 1;
    return p + 2 * e;
}
int64_t host_nq(int64_t E, int p) { return E >= 2 ? 2 * E + 2 * p + 1 : p + 3; }
int64_t host_qlo(int64_t i, int64_t E, int p) { return host_knot_pos(i - p, E, p, host_nq(E, p)) + 1; }
int64_t host_qhi(int64_t i, int64_t E, int p) {
    return host_knot_pos(i + 1 < E ? i + 1 : E, E, p, host_nq(E, p)) - 1;
}
int64_t host_pref(int64_t i, int p, int64_t n) {
    int64_t s = 0;
    for (int64_t k = 0; k < i; ++k) s += wq_ni(k, p, n);
    return s;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

wq_status fail(wq_status st, const std::string &msg) {
    g_err = msg;
    return st;
}
}  // namespace

int64_t wq_host_qlo(int64_t i, int64_t E, int p) { return host_qlo(i, E, p); }
int64_t wq_host_qhi(int64_t i, int64_t E, int p) { return host_qhi(i, E, p); }

static std::atomic<uint64_t> g_launches{0};
void wq_count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
void wq_set_error(const std::string &msg) { g_err = msg; }

wq_status wq_cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return WQ_OK;
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return WQ_ECUDA;
}

cudaError_t wq_smem_attr(const void *func, size_t bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;  // (function, device) pairs already raised to 227 KB
    int dev = 0;
    cudaError_t ce = cudaGetDevice(&dev);
    if (ce != cudaSuccess) return ce;
    std::lock_guard<std::mutex> g(mu);
    if (done.count({func, dev})) return cudaSuccess;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    ce = cudaFuncGetAttributes(&fa, func);
    if (ce != cudaSuccess) return ce;
    const int avail = optin - (int)fa.sharedSizeBytes;
    if ((size_t)avail < bytes) return cudaErrorInvalidValue;
    ce = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, avail);
    if (ce == cudaSuccess) done.insert({func, dev});
    return ce;
}

extern "C" {

const char *wq_status_string(wq_status s) {
    switch (s) {
    case WQ_OK: return "WQ_OK";
    case WQ_EINVAL: return "WQ_EINVAL: invalid argument";
    case WQ_EKNOTS: return "WQ_EKNOTS: invalid knot vector";
    case WQ_ESINGULAR: return "WQ_ESINGULAR: WQ exactness system has no solution";
    case WQ_EGEOMETRY: return "WQ_EGEOMETRY: det J vanishes or changes sign";
    case WQ_ENOMEM: return "WQ_ENOMEM: device allocation failed";
    case WQ_ECUDA: return "WQ_ECUDA: CUDA error";
    case WQ_ERANGE: return "WQ_ERANGE: index out of range";
    }
    return "unknown status";
}

const char *wq_last_error(void) { return g_err.c_str(); }

const char *wq_version(void) { return "libwq sm_100a " __DATE__ " " __TIME__; }

uint64_t wq_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

static int64_t rows_per_plane(const wq_plan_s *P) {
    int64_t r = 1;
    for (int l = 0; l < P->d - 1; ++l) r *= P->dir[l].n;
    return r;
}

// Upload a host net of `count` doubles into *dst (allocated on first use).
static wq_status upload(double **dst, const double *src, size_t count) {
    if (!*dst && cudaMalloc((void **)dst, sizeof(double) * count) != cudaSuccess) {
        *dst = nullptr;
        return fail(WQ_ENOMEM, "control/coefficient net allocation failed");
    }
    return wq_cuda_status(cudaMemcpy(*dst, src, sizeof(double) * count, cudaMemcpyHostToDevice), "net upload");
}

// Verdict of the device-side latched flags after a synchronous build.
static wq_status flags_verdict(wq_plan_s *P) {
    Flags f;
    cudaError_t ce = cudaMemcpy(&f, P->flags, sizeof(Flags), cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "flag readback");
    if (f.weights_bad) {
        int code = f.weights_bad - 1;
        int row = code / 12, rem = code % 12, dir = rem / 4, fam = rem % 4;
        char buf[200];
        snprintf(buf, sizeof buf, "weight system failed (Eq. exact, residual > 1e-13): dir %d row %d family (%d,%d)", dir,
                 row, fam & 1, fam >> 1);
        return fail(WQ_ESINGULAR, buf);
    }
    if (f.det_zero || (f.det_pos && f.det_neg))
        return fail(WQ_EGEOMETRY, f.det_zero ? "det J = 0 at a grid point" : "det J changes sign on the grid");
    return WQ_OK;
}

// Synchronous part of plan creation: rules (ESINGULAR), coefficient field if a control net was
// given (EGEOMETRY), and the one-time z-line preparation (reading R16).
static wq_status create_build(wq_plan_s *P) {
    cudaStream_t s;
    cudaError_t ce = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "plan stream");
    wq_status st = launch_rules(P, s);
    if (!st) st = wq_cuda_status(cudaStreamSynchronize(s), "rules");
    if (!st) st = flags_verdict(P);
    if (!st && P->ctrl_dev) {
        st = launch_coef(P, P->ctrl_dev, P->kappa_dev, P->gamma_dev, s);
        if (!st) st = wq_cuda_status(cudaStreamSynchronize(s), "coefficient field");
        if (!st) st = flags_verdict(P);
        if (!st) P->has_coef = 1;
    }
    cudaStreamDestroy(s);
    if (!st && P->zline_ok) st = zline_prepare(P);
    return st;
}

wq_status wq_plan_create(const wq_plan_desc *desc, wq_plan *out) {
    if (!out) return fail(WQ_EINVAL, "out is NULL");
    *out = nullptr;
    if (!desc) return fail(WQ_EINVAL, "desc is NULL");
    const int d = desc->d, p = desc->p;
    if (d < 1 || d > 3) return fail(WQ_EINVAL, "d must be 1, 2 or 3");
    if (p < 1 || p > WQ_MAX_DEGREE) return fail(p < 1 ? WQ_EKNOTS : WQ_EINVAL, "p must be in [1, WQ_MAX_DEGREE]");
    if (!desc->n_knots || !desc->knots) return fail(WQ_EINVAL, "knots are NULL");
    if (!desc->need_mass && !desc->need_stiffness) return fail(WQ_EINVAL, "need_mass or need_stiffness required");
    if (desc->bpts != WQ_BPTS_INTERIOR && desc->bpts != WQ_BPTS_ENDPOINTS) return fail(WQ_EINVAL, "bad bpts");
    if ((desc->kappa || desc->gamma) && !desc->ctrl) return fail(WQ_EINVAL, "kappa/gamma given without a control net");
    // ---- validate knots
    int64_t nk_[3], E_[3];
    for (int l = 0; l < d; ++l) {
        int64_t nk = desc->n_knots[l];
        const double *xi = desc->knots[l];
        if (!xi) return fail(WQ_EINVAL, "knot vector is NULL");
        int64_t E = nk - 2 * (int64_t)p - 1;
        if (E < 1) return fail(WQ_EKNOTS, "dir " + std::to_string(l) + ": too few knots");
        for (int64_t k = 0; k < nk; ++k)
            if (!std::isfinite(xi[k])) return fail(WQ_EKNOTS, "dir " + std::to_string(l) + ": non-finite knot");
        for (int k = 1; k <= p; ++k)
            if (xi[k] != xi[0] || xi[nk - 1 - k] != xi[nk - 1])
                return fail(WQ_EKNOTS, "dir " + std::to_string(l) + ": knot vector is not open");
        for (int64_t k = p; k < nk - p - 1; ++k)
            if (!(xi[k] < xi[k + 1]))
                return fail(WQ_EKNOTS, "dir " + std::to_string(l) + ": repeated or decreasing interior knot at " +
                                           std::to_string(k));
        nk_[l] = nk;
        E_[l] = E;
    }
    if (desc->bpts == WQ_BPTS_ENDPOINTS) {
        // SPEC's reading of Remark 1: the p+1 boundary-span points include the span's knots, so only
        // p-1 new points lie strictly inside span 0; row 0 (supp B_0 = span 0, open) then has
        // #Q_0 = p-1 < #I_0 = p+1 (and row 1 #Q_1 = p+1 < p+2): Eq. numb_nodes fails.
        return fail(WQ_ESINGULAR, "WQ_BPTS_ENDPOINTS: dir 0 row 0 has #Q = " + std::to_string(p - 1) + " < #I = " +
                                      std::to_string(p + 1) + " (Eq. numb_nodes, P:640-642; reading R1)");
    }
    wq_plan_s *P = new wq_plan_s();
    // value-initialised: POD members zero, vectors empty
    P->d = d;
    P->p = p;
    P->device = desc->device;
    P->need_mass = desc->need_mass ? 1 : 0;
    P->need_stiff = desc->need_stiffness ? 1 : 0;
    for (int l = 0; l < d; ++l) {
        DirView &v = P->dir[l];
        v.nk = nk_[l];
        v.n = nk_[l] - p - 1;
        v.E = E_[l];
        v.nq = host_nq(v.E, p);
        int64_t mq = 0;
        for (int64_t i = 0; i < v.n; ++i) {
            int64_t q = host_qhi(i, v.E, p) - host_qlo(i, v.E, p) + 1;
            if (q < wq_ni(i, p, v.n)) { delete P; return fail(WQ_ESINGULAR, "#Q < #I (Eq. numb_nodes)"); }
            mq = q > mq ? q : mq;
        }
        v.maxq = (int32_t)mq;
        P->L[l] = host_pref(v.n, p, v.n);
    }
    for (int l = d; l < 3; ++l) {
        DirView &v = P->dir[l];
        v.nk = 0; v.n = 1; v.E = 1; v.nq = 1; v.maxq = 1;
        P->L[l] = 1;
    }
    int64_t N = 1, nnz = 1;
    for (int l = 0; l < d; ++l) { N *= P->dir[l].n; nnz *= P->L[l]; }
    if (N >= ((int64_t)1 << 31)) { delete P; return fail(WQ_ERANGE, "N_DOF >= 2^31 (int32 columns)"); }
    P->n_dof_total = N;
    P->nnz_total = nnz;
    // ---- slab of the slowest direction
    const int ld = d - 1;
    const int64_t nd = P->dir[ld].n;
    int64_t b = desc->slab_begin, e = desc->slab_end;
    if (b == 0 && e == -1) e = nd;
    if (b < 0 || e > nd || b >= e) { delete P; return fail(WQ_EINVAL, "bad slab range"); }
    P->slab_b = b;
    P->slab_e = e;
    int64_t L_per_plane = 1;
    for (int l = 0; l < ld; ++l) L_per_plane *= P->L[l];
    P->row_begin = b * rows_per_plane(P);
    P->n_rows_local = (e - b) * rows_per_plane(P);
    P->nnz_local = (host_pref(e, p, nd) - host_pref(b, p, nd)) * L_per_plane;
    // coefficient sub-grid along direction d (points of the owned rows' Q sets)
    P->cq_b = host_qlo(b, P->dir[ld].E, p);
    P->cq_e = host_qhi(e - 1, P->dir[ld].E, p) + 1;
    const int64_t nql = P->cq_e - P->cq_b;
    int64_t cp = nql;
    for (int l = 0; l < ld; ++l) cp *= P->dir[l].nq;
    P->coef_points = cp;
    P->ncomp_s = P->need_stiff ? d * (d + 1) / 2 : 0;
    P->ncomp = P->ncomp_s + P->need_mass;
    P->comp_mass = P->ncomp_s;
    // control planes k_d that the sub-grid's points see: spans of cq_b .. cq_e-1 (+p), and one
    // more below for the derivative differences
    P->k3b = 0;
    P->k3e = P->dir[ld].n;
    if (d == 3) {
        P->zld = (nql + 1) / 2 * 2;
        P->zcs = P->dir[0].nq * P->dir[1].nq * P->zld;
        P->cview.cs = P->zcs;
        P->cview.s1 = P->dir[1].nq * P->zld;
        P->cview.s2 = P->zld;
        P->cview.s3 = 1;
    } else {
        P->nld1 = d == 2 ? P->dir[0].nq : 1;
        P->zcs = cp;
        P->cview.cs = cp;
        P->cview.s1 = 1;
        P->cview.s2 = d == 2 ? P->nld1 : 0;
        P->cview.s3 = 0;
    }
    {
        int64_t nn[3];
        int32_t mq[3];
        for (int l = 0; l < 3; ++l) { nn[l] = P->dir[l].n; mq[l] = P->dir[l].maxq; }
        P->zline_ok = d == 3 && P->need_stiff && zline_supported_p(d, p, nn, mq, e - b, nql);
    }

    // ---- device allocations
    cudaError_t ce = cudaSetDevice(P->device);
    if (ce != cudaSuccess) { delete P; return wq_cuda_status(ce, "cudaSetDevice"); }
    size_t bytes = 0;
    auto take = [&](size_t n) { size_t o = bytes; bytes = align_up(bytes + n); return o; };
    struct Off { size_t knots, pts, span, qlo, qlen, jlo, jlen, pref, B, W; } O[3];
    // directions with bitwise-identical knot vectors share one set of rules tables (the rules are a
    // pure function of the knots and p): dir_src[l] = first such direction
    for (int l = 0; l < 3; ++l) P->dir_src[l] = l;
    for (int l = 1; l < d; ++l)
        for (int q = 0; q < l; ++q)
            if (P->dir_src[q] == q && desc->n_knots[q] == desc->n_knots[l] &&
                memcmp(desc->knots[q], desc->knots[l], sizeof(double) * (size_t)desc->n_knots[l]) == 0) {
                P->dir_src[l] = q;
                break;
            }
    for (int l = 0; l < d; ++l) {
        if (P->dir_src[l] != l) continue;
        DirView &v = P->dir[l];
        O[l].knots = take(sizeof(double) * v.nk);
        O[l].pts = take(sizeof(double) * v.nq);
        O[l].span = take(sizeof(int32_t) * v.nq);
        O[l].qlo = take(sizeof(int32_t) * v.n);
        O[l].qlen = take(sizeof(int32_t) * v.n);
        O[l].jlo = take(sizeof(int32_t) * v.n);
        O[l].jlen = take(sizeof(int32_t) * v.n);
        O[l].pref = take(sizeof(int64_t) * (v.n + 1));
        O[l].B = take(sizeof(double) * v.nq * wq_bstride(p));
        O[l].W = take(sizeof(double) * v.n * 4 * v.maxq);
    }
    size_t o_gl = take(sizeof(double) * 4 * (p + 1));
    size_t o_fl = take(sizeof(Flags));
    void *arena = nullptr;
    ce = cudaMalloc(&arena, bytes);
    if (ce != cudaSuccess) { delete P; return fail(WQ_ENOMEM, "arena allocation failed"); }
    cudaMemset(arena, 0, bytes);
    P->arena = arena;
    P->arena_bytes = bytes;
    char *A = (char *)arena;
    for (int l = 0; l < d; ++l) {
        DirView &v = P->dir[l];
        if (P->dir_src[l] != l) {  // alias: the source direction's tables
            const DirView &u = P->dir[P->dir_src[l]];
            v.knots = u.knots; v.pts = u.pts; v.span = u.span; v.qlo = u.qlo; v.qlen = u.qlen;
            v.jlo = u.jlo; v.jlen = u.jlen; v.pref = u.pref; v.B = u.B; v.W = u.W;
            continue;
        }
        v.knots = (const double *)(A + O[l].knots);
        v.pts = (double *)(A + O[l].pts);
        v.span = (int32_t *)(A + O[l].span);
        v.qlo = (int32_t *)(A + O[l].qlo);
        v.qlen = (int32_t *)(A + O[l].qlen);
        v.jlo = (int32_t *)(A + O[l].jlo);
        v.jlen = (int32_t *)(A + O[l].jlen);
        v.pref = (int64_t *)(A + O[l].pref);
        v.B = (double *)(A + O[l].B);
        v.W = (double *)(A + O[l].W);
        ce = cudaMemcpy((void *)v.knots, desc->knots[l], sizeof(double) * v.nk, cudaMemcpyHostToDevice);
        if (ce != cudaSuccess) { wq_plan_destroy(P); return wq_cuda_status(ce, "knot upload"); }
    }
    P->gl = (double *)(A + o_gl);
    P->flags = (Flags *)(A + o_fl);
    size_t cbytes = sizeof(double) * (size_t)P->ncomp * (size_t)P->zcs;
    ce = cudaMalloc((void **)&P->coef, cbytes);
    if (ce != cudaSuccess) {
        P->coef = nullptr;
        wq_plan_destroy(P);
        return fail(WQ_ENOMEM, "coefficient field allocation failed (" + std::to_string(cbytes) + " bytes)");
    }
    cudaMemset(P->coef, 0, cbytes);  // z-layout row padding stays zero
    P->cview.base = P->coef;
    if (P->zline_ok) {
        // lines (i1, i2) of the z-line kernel: uniform-rule lines, other interior lines, boundary lines
        const int64_t n0 = P->dir[0].n, n1 = P->dir[1].n;
        auto interz = [&](int l, int64_t i) {
            const int64_t E = P->dir[l].E, n = P->dir[l].n;
            return i >= p + 1 && i <= n - p - 2 && host_qhi(i, E, p) - host_qlo(i, E, p) + 1 == 2 * p + 1;
        };
        auto uniz = [&](int l, int64_t i) { return i >= 2 * p && i <= P->dir[l].n - 1 - 2 * p; };
        for (int64_t i1 = 0; i1 < n1; ++i1)
            for (int64_t i0 = 0; i0 < n0; ++i0) {
                const int32_t line = (int32_t)(i0 + n0 * i1);
                if (!(interz(0, i0) && interz(1, i1))) {
                    // measurement switch (debug only; wrong values): boundary lines of one kind only,
                    // 0 = boundary in direction 0 only, 1 = in direction 1 only, 2 = in both
                    static const char *flt = getenv("WQ_ZL_BND_FILTER");
                    if (flt) {
                        const int kind = interz(1, i1) ? 0 : (interz(0, i0) ? 1 : 2);
                        if (kind != atoi(flt)) continue;
                    }
                    P->zlines_bnd.push_back(line);
                }
                else (uniz(0, i0) && uniz(1, i1) ? P->zlines_uni : P->zlines_int).push_back(line);
            }
        // boundary lines: greedy longest-processing-time assignment to the CTAs of one launch (cost:
        // consumer work per line + producer stage-A fibre passes x #Q_0 + stage-B #Q_1), each CTA's
        // list sorted by row types (the kernel runs one unrolled staircase per type pair); the
        // lists are concatenated with bounds[c] = first item of CTA c
        auto ztype = [&](int l, int64_t i) -> int64_t {
            const int64_t n = P->dir[l].n;
            return i <= p ? i + 1 : (i >= n - 1 - p ? n - 1 - i + p + 2 : 0);
        };
        auto zq = [&](int l, int64_t i) {
            return (double)(host_qhi(i, P->dir[l].E, p) - host_qlo(i, P->dir[l].E, p) + 1);
        };
        int nsm = 0;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P->device);
        const int64_t G = std::min<int64_t>(nsm > 0 ? nsm : 148, (int64_t)P->zlines_bnd.size());
        std::vector<int32_t> bounds;
        if (G > 0) {
            std::vector<std::pair<double, int32_t>> items;
            for (int32_t line : P->zlines_bnd) {
                const int64_t i0 = line % n0, i1 = line / n0;
                const double q0 = zq(0, i0), q1 = zq(1, i1);
                items.push_back({2.0 * (2 * p + 1) + std::ceil(3.0 * q1 / 32.0) * q0 + q1, line});
            }
            std::stable_sort(items.begin(), items.end(), [](auto &x, auto &y) { return x.first > y.first; });
            std::vector<double> load(G, 0.0);
            std::vector<std::vector<int32_t>> per(G);
            for (auto &it : items) {
                const int64_t c = std::min_element(load.begin(), load.end()) - load.begin();
                load[c] += it.first;
                per[c].push_back(it.second);
            }
            P->zlines_bnd.clear();
            bounds.push_back(0);
            for (int64_t c = 0; c < G; ++c) {
                std::stable_sort(per[c].begin(), per[c].end(), [&](int32_t x, int32_t y) {
                    return ztype(0, x % n0) * 64 + ztype(1, x / n0) < ztype(0, y % n0) * 64 + ztype(1, y / n0);
                });
                P->zlines_bnd.insert(P->zlines_bnd.end(), per[c].begin(), per[c].end());
                bounds.push_back((int32_t)P->zlines_bnd.size());
            }
        }
        std::vector<int32_t> all(P->zlines_uni);
        all.insert(all.end(), P->zlines_int.begin(), P->zlines_int.end());
        all.insert(all.end(), P->zlines_bnd.begin(), P->zlines_bnd.end());
        P->zbounds_n = G;
        const size_t zl = sizeof(int32_t) * (all.size() + bounds.size() + 1);
        ce = cudaMalloc((void **)&P->zlines_dev, zl);
        if (ce != cudaSuccess) { P->zlines_dev = nullptr; wq_plan_destroy(P); return fail(WQ_ENOMEM, "z line lists"); }
        if (!all.empty()) cudaMemcpy(P->zlines_dev, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice);
        P->zbounds_dev = nullptr;
        if (!bounds.empty()) {
            P->zbounds_dev = P->zlines_dev + all.size();
            cudaMemcpy(P->zbounds_dev, bounds.data(), sizeof(int32_t) * bounds.size(), cudaMemcpyHostToDevice);
        }
        cbytes += zl;
    }
    if (d == 3) {
        // lines of the ZHP kernel: interior in directions 1 and 2 (boxes of 2p+1 points), then the rest
        const int64_t n0 = P->dir[0].n, n1 = P->dir[1].n;
        auto inter = [&](int l, int64_t i) {  // interior row type: touches no boundary span (R14)
            return i >= p + 1 && i <= P->dir[l].n - p - 2 &&
                   host_qhi(i, P->dir[l].E, p) - host_qlo(i, P->dir[l].E, p) + 1 == 2 * p + 1;
        };
        for (int64_t i1 = 0; i1 < n1; ++i1)
            for (int64_t i0 = 0; i0 < n0; ++i0)
                (inter(0, i0) && inter(1, i1) ? P->zh_int : P->zh_bnd).push_back((int32_t)(i0 + n0 * i1));
        std::vector<int32_t> all(P->zh_int);
        all.insert(all.end(), P->zh_bnd.begin(), P->zh_bnd.end());
        ce = cudaMalloc((void **)&P->zh_dev, sizeof(int32_t) * all.size());
        if (ce != cudaSuccess) { P->zh_dev = nullptr; wq_plan_destroy(P); return fail(WQ_ENOMEM, "line lists"); }
        cudaMemcpy(P->zh_dev, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice);
        cbytes += sizeof(int32_t) * all.size();
    }
    // ---- control net and coefficient nets (copied; the plan owns the device copies)
    wq_status st = WQ_OK;
    if (desc->ctrl) {
        st = upload(&P->ctrl_dev, desc->ctrl, (size_t)N * d);
        P->ctrl_bytes = sizeof(double) * (size_t)N * d;
        if (!st && desc->kappa) st = upload(&P->kappa_dev, desc->kappa, (size_t)N);
        if (!st && desc->gamma) st = upload(&P->gamma_dev, desc->gamma, (size_t)N);
        cbytes += sizeof(double) * (size_t)N * (d + (desc->kappa ? 1 : 0) + (desc->gamma ? 1 : 0));
    }
    // ---- which kernel WQ_KERNEL_AUTO runs
    if (!st) {
        // measured on C4 (100^3 elements, BASELINE configs[3]): mass by ZHP for p >= 4
        // and the row-tile kernel below, stiffness by the z-line kernel for p <= 6 except p = 5 (ZHP
        // 17.5 ms against 19.6: its boundary lines are faster), ZHP for p >= 7
        const bool zhp_m = zhp_supported(P, WQ_MASS) && p >= 4;
        P->kernel_auto[0] = !P->need_mass ? 0
                          : d < 3 ? (sf2_supported(P, WQ_MASS) ? WQ_KERNEL_SF2 : WQ_KERNEL_DIRECT)
                          : zhp_m ? WQ_KERNEL_ZHP
                          : tile_supported(P, WQ_MASS) ? WQ_KERNEL_TILE
                          : zhp_supported(P, WQ_MASS) ? WQ_KERNEL_ZHP : WQ_KERNEL_DIRECT;
        if (d == 3 && P->need_stiff && !P->zline_ok && !(zhp_supported(P, WQ_STIFFNESS) && p >= 7) &&
            tile_supported(P, WQ_STIFFNESS)) {
            // the row-tile stiffness (fallback when ZHP does not fit) reads a standard-layout copy
            // (made after every coefficient build; measured at C4 p = 10: 574 -> 407 ms; its mass
            // path is faster on the z layout)
            const size_t sb = sizeof(double) * (size_t)P->ncomp * (size_t)cp;
            ce = cudaMalloc((void **)&P->coef_std, sb);
            if (ce != cudaSuccess) { P->coef_std = nullptr; st = fail(WQ_ENOMEM, "standard-layout coefficient copy"); }
            else {
                cbytes += sb;
                P->cview_std.base = P->coef_std;
                P->cview_std.cs = cp;
                P->cview_std.s1 = 1;
                P->cview_std.s2 = P->dir[0].nq;
                P->cview_std.s3 = P->dir[0].nq * P->dir[1].nq;
            }
        }
        if (!st) st = create_build(P);
        // stiffness: ZHP for p >= 7 (C4 p = 10: 361 ms, row-tile on the standard-layout copy 407)
        P->kernel_auto[1] = !P->need_stiff ? 0
                          : d < 3 ? (sf2_supported(P, WQ_STIFFNESS) ? WQ_KERNEL_SF2 : WQ_KERNEL_DIRECT)
                          : p == 5 && zhp_supported(P, WQ_STIFFNESS) ? WQ_KERNEL_ZHP
                          : P->zline_ok ? WQ_KERNEL_ZLINE
                          : zhp_supported(P, WQ_STIFFNESS) && (p >= 7 || !tile_supported(P, WQ_STIFFNESS))
                              ? WQ_KERNEL_ZHP
                          : tile_supported(P, WQ_STIFFNESS) ? WQ_KERNEL_TILE : WQ_KERNEL_DIRECT;
    }
    if (st) {
        const std::string msg = g_err;
        wq_plan_destroy(P);
        g_err = msg;
        return st;
    }
    P->workspace_bytes = (int64_t)(bytes + cbytes);
    *out = P;
    return WQ_OK;
}

wq_status wq_plan_destroy(wq_plan P) {
    if (!P) return WQ_OK;
    cudaSetDevice(P->device);
    if (P->arena) cudaFree(P->arena);
    if (P->coef) cudaFree(P->coef);
    if (P->coef_std) cudaFree(P->coef_std);
    if (P->zlines_dev) cudaFree(P->zlines_dev);
    if (P->zh_dev) cudaFree(P->zh_dev);
    if (P->ctrl_dev) cudaFree(P->ctrl_dev);
    if (P->kappa_dev) cudaFree(P->kappa_dev);
    if (P->gamma_dev) cudaFree(P->gamma_dev);
    if (P->dnet) cudaFree(P->dnet);
    if (P->x2) cudaFree(P->x2);
    if (P->stage_val) cudaFree(P->stage_val);
    for (cudaStream_t z : P->zfork)
        if (z) cudaStreamDestroy(z);
    for (cudaEvent_t e : P->zev)
        if (e) cudaEventDestroy(e);
    delete P;
    return WQ_OK;
}

wq_status wq_plan_info(wq_plan P, wq_plan_info_t *info) {
    if (!P || !info) return fail(WQ_EINVAL, "NULL argument");
    info->n_dof_total = P->n_dof_total;
    info->nnz_total = P->nnz_total;
    info->row_begin = P->row_begin;
    info->n_rows_local = P->n_rows_local;
    info->nnz_local = P->nnz_local;
    for (int l = 0; l < 3; ++l) {
        info->n_dof[l] = P->dir[l].n;
        info->n_qp[l] = P->dir[l].nq;
        info->max_q[l] = P->dir[l].maxq;
    }
    info->coef_points = P->coef_points;
    info->workspace_bytes = P->workspace_bytes;
    info->kernel[0] = P->kernel_auto[0];
    info->kernel[1] = P->kernel_auto[1];
    info->uniform_rules = P->zuni_state == 1 ? 1 : 0;
    return WQ_OK;
}

wq_status wq_build_rules(wq_plan P, void *stream) {
    if (!P) return fail(WQ_EINVAL, "NULL plan");
    cudaSetDevice(P->device);
    cudaError_t ce = cudaMemsetAsync(&P->flags->weights_bad, 0, sizeof(int), S(stream));
    if (ce != cudaSuccess) return wq_cuda_status(ce, "flag reset");
    return launch_rules(P, S(stream));
}

wq_status wq_build_coef(wq_plan P, const double *d_ctrl, const double *d_kappa, const double *d_gamma, void *stream) {
    if (!P || !d_ctrl) return fail(WQ_EINVAL, "NULL argument");
    cudaSetDevice(P->device);
    cudaError_t ce = cudaMemsetAsync(&P->flags->det_pos, 0, 3 * sizeof(int), S(stream));
    if (ce != cudaSuccess) return wq_cuda_status(ce, "flag reset");
    wq_status st = launch_coef(P, d_ctrl, d_kappa, d_gamma, S(stream));
    if (!st) P->has_coef = 1;
    return st;
}

wq_status wq_pattern(wq_plan P, int64_t nnz_base, int64_t *d_row_ptr, int32_t *d_col, void *stream) {
    if (!P || !d_row_ptr) return fail(WQ_EINVAL, "NULL argument");
    if (nnz_base < 0) return fail(WQ_EINVAL, "negative nnz_base");
    cudaSetDevice(P->device);
    return launch_pattern(P, nnz_base, d_row_ptr, d_col, 0, P->n_rows_local, S(stream));
}

// z-line stiffness: boundary lines through the ZHP kernel's boundary class (the same line set:
// a support touching a boundary span in direction 1 or 2).  Measurement switch WQ_ZL_BND=zhp|zline.
static bool zl_bnd_zhp(const wq_plan_s *P) {
    if (!zhp_supported(P, WQ_STIFFNESS)) return false;
    static const char *env = getenv("WQ_ZL_BND");
    if (env) return strcmp(env, "zhp") == 0;
    return false;
}

static wq_status assemble_range(wq_plan_s *P, int matrix, wq_kernel kernel, double *val, int32_t *col,
                                int64_t pl_lo, int64_t pl_hi, int64_t val_base, cudaStream_t s) {
    if (matrix == WQ_MASS && !P->need_mass) return fail(WQ_EINVAL, "plan was created without need_mass");
    if (matrix == WQ_STIFFNESS && !P->need_stiff) return fail(WQ_EINVAL, "plan was created without need_stiffness");
    if (!P->has_coef) return fail(WQ_EINVAL, "no coefficient field: pass desc.ctrl or call wq_build_coef first");
    if (kernel == WQ_KERNEL_AUTO) kernel = (wq_kernel)P->kernel_auto[matrix];
    switch (kernel) {
    case WQ_KERNEL_ZLINE: {
        if (matrix != WQ_STIFFNESS || !P->zline_ok)
            return fail(WQ_EINVAL, "z-line kernel not available for this plan (stiffness, d = 3, 2 <= p <= 6)");
        const int64_t nu = (int64_t)P->zlines_uni.size(), ni = (int64_t)P->zlines_int.size(),
                      nb = (int64_t)P->zlines_bnd.size();
        // the three launches write disjoint rows: they run on forked streams so that the SMs a
        // launch drains are refilled by the next one (C4 p = 4: 5.37 -> 5.26 ms, DESIGN.md §6;
        // measurement switch WQ_ZL_FORK = 0 serial, 1 default, 2 boundary launch issued first)
        static const char *fk = getenv("WQ_ZL_FORK");
        const int fork = fk ? atoi(fk) : 1;
        cudaStream_t s1 = s, s2 = s;
        if (fork) {
            cudaError_t ce = cudaSuccess;
            for (int k = 0; k < 2 && ce == cudaSuccess; ++k)
                if (!P->zfork[k]) ce = cudaStreamCreateWithFlags(&P->zfork[k], cudaStreamNonBlocking);
            for (int k = 0; k < 3 && ce == cudaSuccess; ++k)
                if (!P->zev[k]) ce = cudaEventCreateWithFlags(&P->zev[k], cudaEventDisableTiming);
            if (ce == cudaSuccess) ce = cudaEventRecord(P->zev[0], s);
            for (int k = 0; k < 2 && ce == cudaSuccess; ++k) ce = cudaStreamWaitEvent(P->zfork[k], P->zev[0], 0);
            if (ce != cudaSuccess) return wq_cuda_status(ce, "z-line stream fork");
            s1 = P->zfork[0];
            s2 = P->zfork[1];
        }
        // order of issue: fork = 1 uniform, interior, boundary; fork = 2 boundary first
        wq_status st = WQ_OK;
        auto bnd = [&]() {
            // boundary lines: by the ZHP kernel's boundary class where that is measured faster
            // (zl_bnd_zhp), else the z-line kernel's boundary launch
            if (zl_bnd_zhp(P)) return launch_assemble_zhp(P, matrix, pl_lo, pl_hi, val, col, val_base, s2, 2);
            return launch_assemble_zline(P, 2, P->zlines_dev + nu + ni, nb, pl_lo, pl_hi, val, col, val_base, s2);
        };
        if (fork == 2) st = bnd();
        if (!st) st = launch_assemble_zline(P, 0, P->zlines_dev, nu, pl_lo, pl_hi, val, col, val_base, s);
        if (!st) st = launch_assemble_zline(P, 1, P->zlines_dev + nu, ni, pl_lo, pl_hi, val, col, val_base, s1);
        if (!st && fork != 2) st = bnd();
        if (fork) {
            cudaError_t ce = cudaEventRecord(P->zev[1], s1);
            if (ce == cudaSuccess) ce = cudaEventRecord(P->zev[2], s2);
            if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s, P->zev[1], 0);
            if (ce == cudaSuccess) ce = cudaStreamWaitEvent(s, P->zev[2], 0);
            if (!st && ce != cudaSuccess) st = wq_cuda_status(ce, "z-line stream join");
        }
        return st;
    }
    case WQ_KERNEL_ZHP:
        if (!zhp_supported(P, matrix)) return fail(WQ_EINVAL, "ZHP kernel not available for this plan (d = 3)");
        return launch_assemble_zhp(P, matrix, pl_lo, pl_hi, val, col, val_base, s);
    case WQ_KERNEL_TILE:
        if (!tile_supported(P, matrix)) return fail(WQ_EINVAL, "tile kernel not available for this (d, p)");
        return launch_assemble_tile(P, matrix, val, col, pl_lo, pl_hi, val_base, s);
    case WQ_KERNEL_SF2:
        if (!sf2_supported(P, matrix)) return fail(WQ_EINVAL, "sf2 kernel not available for this plan (d <= 2)");
        return launch_assemble_sf2(P, matrix, val, col, pl_lo, pl_hi, val_base, s);
    case WQ_KERNEL_DIRECT:
        return launch_assemble_direct(P, matrix, val, col, pl_lo, pl_hi, val_base, s);
    default:
        return fail(WQ_EINVAL, "unknown kernel");
    }
}

wq_status wq_assemble_ex(wq_plan P, wq_matrix matrix, wq_kernel kernel, double *d_val, int32_t *d_col, void *stream) {
    if (!P || !d_val) return fail(WQ_EINVAL, "NULL argument");
    if (matrix != WQ_MASS && matrix != WQ_STIFFNESS) return fail(WQ_EINVAL, "bad matrix");
    cudaSetDevice(P->device);
    return assemble_range(P, matrix, kernel, d_val, d_col, 0, P->slab_e - P->slab_b, 0, S(stream));
}

wq_status wq_assemble(wq_plan P, wq_matrix matrix, double *d_val, int32_t *d_col, void *stream) {
    return wq_assemble_ex(P, matrix, WQ_KERNEL_AUTO, d_val, d_col, stream);
}

wq_status wq_assemble_sgq(wq_plan P, wq_matrix matrix, const double *d_ctrl, const double *d_kappa,
                          const double *d_gamma, double *d_val, int32_t *d_col, void *stream) {
    if (!P || !d_val || !d_ctrl) return fail(WQ_EINVAL, "NULL argument");
    if (matrix != WQ_MASS && matrix != WQ_STIFFNESS) return fail(WQ_EINVAL, "bad matrix");
    cudaSetDevice(P->device);
    return launch_assemble_sgq(P, matrix, d_ctrl, d_kappa, d_gamma, d_val, d_col, S(stream));
}

wq_status wq_check(wq_plan P, void *stream) {
    if (!P) return fail(WQ_EINVAL, "NULL plan");
    cudaSetDevice(P->device);
    cudaError_t ce = cudaStreamSynchronize(S(stream));
    if (ce != cudaSuccess) return wq_cuda_status(ce, "stream synchronize");
    return flags_verdict(P);
}

wq_status wq_form_host(wq_plan P, wq_matrix matrix, const double *h_ctrl, const double *h_kappa, const double *h_gamma,
                       int64_t nnz_base, int64_t *h_row_ptr, int32_t *h_col, double *h_val, void *stream) {
    if (!P || !h_ctrl || !h_row_ptr || !h_col || !h_val) return fail(WQ_EINVAL, "NULL argument");
    if (matrix != WQ_MASS && matrix != WQ_STIFFNESS) return fail(WQ_EINVAL, "bad matrix");
    cudaSetDevice(P->device);
    cudaStream_t s = S(stream);
    const size_t nctrl = (size_t)P->n_dof_total * P->d;
    cudaError_t ce;
    if (P->ctrl_bytes < nctrl * sizeof(double)) {
        if (P->ctrl_dev) cudaFree(P->ctrl_dev);
        ce = cudaMalloc((void **)&P->ctrl_dev, nctrl * sizeof(double));
        if (ce != cudaSuccess) { P->ctrl_dev = nullptr; P->ctrl_bytes = 0; return fail(WQ_ENOMEM, "ctrl staging"); }
        P->ctrl_bytes = nctrl * sizeof(double);
    }
    for (double **dst : {&P->kappa_dev, &P->gamma_dev}) {
        const double *src = dst == &P->kappa_dev ? h_kappa : h_gamma;
        if (src && !*dst && cudaMalloc((void **)dst, sizeof(double) * (size_t)P->n_dof_total) != cudaSuccess) {
            *dst = nullptr;
            return fail(WQ_ENOMEM, "coefficient net staging");
        }
    }
    // chunking by slab planes, double-buffered staging for values + columns + row_ptr
    const int64_t nplanes = P->slab_e - P->slab_b;
    const int64_t rpp = rows_per_plane(P);
    const int64_t max_plane_nnz = [&] {
        int64_t m = 1;
        for (int l = 0; l < P->d - 1; ++l) m *= P->L[l];
        return m * (2 * P->p + 1);
    }();
    int64_t target = (int64_t)1 << 26;  // ~64M nnz per chunk (768 MB of CSR)
    if (const char *e = getenv("WQ_FORM_CHUNK_NNZ")) target = atoll(e) > 0 ? atoll(e) : target;  // tests
    int64_t ppc = target / max_plane_nnz;
    if (ppc < 1) ppc = 1;
    if (ppc > nplanes) ppc = nplanes;
    const int64_t chunk_nnz = ppc * max_plane_nnz;
    const int64_t chunk_rows = ppc * rpp + 1;
    const size_t per = align_up(sizeof(double) * chunk_nnz) + align_up(sizeof(int32_t) * chunk_nnz) +
                       align_up(sizeof(int64_t) * chunk_rows);
    if (P->stage_bytes < 2 * per) {
        if (P->stage_val) cudaFree(P->stage_val);
        ce = cudaMalloc((void **)&P->stage_val, 2 * per);
        if (ce != cudaSuccess) { P->stage_val = nullptr; P->stage_bytes = 0; return fail(WQ_ENOMEM, "staging"); }
        P->stage_bytes = 2 * per;
    }
    char *base = (char *)P->stage_val;
    double *sv[2];
    int32_t *sc[2];
    int64_t *sr[2];
    for (int k = 0; k < 2; ++k) {
        char *b = base + k * per;
        sv[k] = (double *)b;
        sc[k] = (int32_t *)(b + align_up(sizeof(double) * chunk_nnz));
        sr[k] = (int64_t *)(b + align_up(sizeof(double) * chunk_nnz) + align_up(sizeof(int32_t) * chunk_nnz));
    }
    cudaStream_t cs;
    ce = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (ce != cudaSuccess) return wq_cuda_status(ce, "copy stream");
    cudaEvent_t done[2], freed[2];
    for (int k = 0; k < 2; ++k) {
        cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&freed[k], cudaEventDisableTiming);
        cudaEventRecord(freed[k], cs);
    }
    wq_status st = WQ_OK;
    ce = cudaMemcpyAsync(P->ctrl_dev, h_ctrl, nctrl * sizeof(double), cudaMemcpyHostToDevice, s);
    if (!ce && h_kappa) ce = cudaMemcpyAsync(P->kappa_dev, h_kappa, sizeof(double) * P->n_dof_total, cudaMemcpyHostToDevice, s);
    if (!ce && h_gamma) ce = cudaMemcpyAsync(P->gamma_dev, h_gamma, sizeof(double) * P->n_dof_total, cudaMemcpyHostToDevice, s);
    if (ce != cudaSuccess) st = wq_cuda_status(ce, "ctrl upload");
    if (!st) st = wq_build_rules(P, s);
    if (!st) st = wq_build_coef(P, P->ctrl_dev, h_kappa ? P->kappa_dev : nullptr, h_gamma ? P->gamma_dev : nullptr, s);
    // host-side 1D prefix of the slowest direction for chunk offsets
    const int64_t nd = P->dir[P->d - 1].n;
    int64_t Lpp = 1;
    for (int l = 0; l < P->d - 1; ++l) Lpp *= P->L[l];
    const int64_t pref_b = host_pref(P->slab_b, P->p, nd);
    int k = 0;
    for (int64_t pl = 0; pl < nplanes && !st; pl += ppc, k ^= 1) {
        int64_t ph = pl + ppc < nplanes ? pl + ppc : nplanes;
        int64_t off_lo = (host_pref(P->slab_b + pl, P->p, nd) - pref_b) * Lpp;
        int64_t off_hi = (host_pref(P->slab_b + ph, P->p, nd) - pref_b) * Lpp;
        int64_t r_lo = pl * rpp, r_hi = ph * rpp;
        cudaStreamWaitEvent(s, freed[k], 0);
        st = assemble_range(P, matrix, WQ_KERNEL_AUTO, sv[k], sc[k], pl, ph, off_lo, s);
        if (st) break;
        st = launch_pattern(P, nnz_base, sr[k], nullptr, r_lo, r_hi - 1, s);
        if (st) break;
        cudaEventRecord(done[k], s);
        cudaStreamWaitEvent(cs, done[k], 0);
        size_t nz = (size_t)(off_hi - off_lo);
        cudaMemcpyAsync(h_val + off_lo, sv[k], nz * sizeof(double), cudaMemcpyDeviceToHost, cs);
        cudaMemcpyAsync(h_col + off_lo, sc[k], nz * sizeof(int32_t), cudaMemcpyDeviceToHost, cs);
        cudaMemcpyAsync(h_row_ptr + r_lo, sr[k], (size_t)(r_hi - r_lo) * sizeof(int64_t), cudaMemcpyDeviceToHost, cs);
        cudaEventRecord(freed[k], cs);
    }
    if (!st) {
        // final row_ptr entry
        h_row_ptr[P->n_rows_local] = nnz_base + P->nnz_local;
    }
    ce = cudaStreamSynchronize(cs);
    if (!st && ce != cudaSuccess) st = wq_cuda_status(ce, "copy stream");
    for (int kk = 0; kk < 2; ++kk) { cudaEventDestroy(done[kk]); cudaEventDestroy(freed[kk]); }
    cudaStreamDestroy(cs);
    if (!st) st = wq_check(P, stream);
    return st;
}

wq_status wq_export_rules(wq_plan P, int dir, double *h_points, int32_t *h_qlo, int32_t *h_qlen, double *h_w,
                          double *h_basis, int32_t *h_span) {
    if (!P) return fail(WQ_EINVAL, "NULL plan");
    if (dir < 0 || dir >= P->d) return fail(WQ_ERANGE, "dir out of range");
    cudaSetDevice(P->device);
    const DirView &v = P->dir[dir];
    const int P1 = P->p + 1;
    cudaError_t ce = cudaDeviceSynchronize();
    if (!ce && h_points) ce = cudaMemcpy(h_points, v.pts, sizeof(double) * v.nq, cudaMemcpyDeviceToHost);
    if (!ce && h_qlo) ce = cudaMemcpy(h_qlo, v.qlo, sizeof(int32_t) * v.n, cudaMemcpyDeviceToHost);
    if (!ce && h_qlen) ce = cudaMemcpy(h_qlen, v.qlen, sizeof(int32_t) * v.n, cudaMemcpyDeviceToHost);
    if (!ce && h_w) {  // device [n][maxq][4] -> documented [n][4][maxq]
        std::vector<double> t((size_t)v.n * 4 * v.maxq);
        ce = cudaMemcpy(t.data(), v.W, sizeof(double) * t.size(), cudaMemcpyDeviceToHost);
        for (int64_t i = 0; i < v.n; ++i)
            for (int c = 0; c < v.maxq; ++c)
                for (int f = 0; f < 4; ++f) h_w[(i * 4 + f) * v.maxq + c] = t[(i * v.maxq + c) * 4 + f];
    }
    if (!ce && h_basis) {  // device [nq][pairs..., low...] -> documented [nq][3][p+1]
        std::vector<double> t((size_t)v.nq * wq_bstride(P->p));
        ce = cudaMemcpy(t.data(), v.B, sizeof(double) * t.size(), cudaMemcpyDeviceToHost);
        for (int64_t q = 0; q < v.nq; ++q)
            for (int r = 0; r < P1; ++r) {
                const double *s = t.data() + q * wq_bstride(P->p);
                h_basis[(q * 3 + 0) * P1 + r] = s[2 * r];
                h_basis[(q * 3 + 1) * P1 + r] = s[2 * r + 1];
                h_basis[(q * 3 + 2) * P1 + r] = s[2 * P1 + r];
            }
    }
    if (!ce && h_span) ce = cudaMemcpy(h_span, v.span, sizeof(int32_t) * v.nq, cudaMemcpyDeviceToHost);
    return wq_cuda_status(ce, "export rules");
}

wq_status wq_export_coef(wq_plan P, double *h_out, int64_t *n_values, int32_t *ncomp, int64_t *q_d_begin) {
    if (!P) return fail(WQ_EINVAL, "NULL plan");
    if (n_values) *n_values = (int64_t)P->ncomp * P->coef_points;
    if (ncomp) *ncomp = P->ncomp;
    if (q_d_begin) *q_d_begin = P->cq_b;
    if (!h_out) return WQ_OK;
    cudaSetDevice(P->device);
    cudaError_t ce = cudaDeviceSynchronize();
    if (P->d == 3) {
        // z layout [comp][q_1][q_2][q_3 - cq_b] -> documented [comp][q_3][q_2][q_1]
        const int64_t nqa = P->dir[0].nq, nqb = P->dir[1].nq, nqc = P->cq_e - P->cq_b;
        std::vector<double> z((size_t)P->ncomp * P->zcs);
        if (!ce) ce = cudaMemcpy(z.data(), P->coef, sizeof(double) * z.size(), cudaMemcpyDeviceToHost);
        if (!ce)
            for (int k = 0; k < P->ncomp; ++k)
                for (int64_t qc = 0; qc < nqc; ++qc)
                    for (int64_t qb = 0; qb < nqb; ++qb)
                        for (int64_t qa = 0; qa < nqa; ++qa)
                            h_out[k * P->coef_points + (qc * nqb + qb) * nqa + qa] =
                                z[k * P->zcs + (qa * nqb + qb) * P->zld + qc];
    } else if (!ce) {
        ce = cudaMemcpy(h_out, P->coef, sizeof(double) * P->ncomp * P->coef_points, cudaMemcpyDeviceToHost);
    }
    return wq_cuda_status(ce, "export coef");
}

}  // extern "C"
