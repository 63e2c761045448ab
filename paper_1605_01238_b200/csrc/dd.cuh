// dd.cuh -- double-double arithmetic (~106-bit significand) for the weight
// construction (reading R5: extended precision from FP64 inputs, rounded
// once to FP64).  Every primitive uses explicit round-to-nearest intrinsics so
// the compiler cannot contract or reassociate the error-free transformations.
#pragma once
#include <cuda_runtime.h>

struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd dd_make(double a) { return dd{a, 0.0}; }

__device__ __forceinline__ dd two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return dd{s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double e = __dsub_rn(b, __dsub_rn(s, a));
    return dd{s, e};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
    double p = __dmul_rn(a, b);
    double e = __fma_rn(a, b, -p);
    return dd{p, e};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = quick_two_sum(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
__device__ __forceinline__ dd dd_add_d(dd a, double b) {
    dd s = two_sum(a.hi, b);
    s.lo = __dadd_rn(s.lo, a.lo);
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    p.lo = __fma_rn(a.hi, b.lo, p.lo);
    p.lo = __fma_rn(a.lo, b.hi, p.lo);
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
    dd p = two_prod(a.hi, b);
    p.lo = __fma_rn(a.lo, b, p.lo);
    return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
    double q1 = __ddiv_rn(a.hi, b.hi);
    dd r = dd_sub(a, dd_mul_d(b, q1));
    double q2 = __ddiv_rn(r.hi, b.hi);
    r = dd_sub(r, dd_mul_d(b, q2));
    double q3 = __ddiv_rn(r.hi, b.hi);
    dd q = quick_two_sum(q1, q2);
    return dd_add_d(q, q3);
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
    if (a.hi <= 0.0) return dd{0.0, 0.0};
    double x = __dsqrt_rn(a.hi);
    dd r = dd_sub(a, two_prod(x, x));
    double c = __ddiv_rn(r.hi, __dmul_rn(2.0, x));
    return quick_two_sum(x, c);
}
__device__ __forceinline__ double dd_to_d(dd a) { return __dadd_rn(a.hi, a.lo); }
__device__ __forceinline__ dd dd_abs(dd a) { return a.hi < 0.0 ? dd_neg(a) : a; }
__device__ __forceinline__ bool dd_lt(dd a, dd b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }
