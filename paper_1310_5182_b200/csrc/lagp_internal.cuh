// lagp_internal.cuh — device helpers shared by the sm_100a kernels of the
// product path. (The CPU oracle has its own, separate code: oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lagp.h"

namespace lagp {

constexpr double kSMin = 1e-12;    // exclusion threshold on s_c = m_j^{-1}(x') (R12)
constexpr double kTieGap = 1e-12;  // near-tie threshold on the top-2 relative gap (north_star)

// Squared distance accumulated with fma in the fixed order k = 0..p-1 from 0
// (R8). __dsub_rn / __fma_rn pin the rounding so the bits equal the oracle's.
__device__ __forceinline__ double sqdist_fma(const double *a, const double *b, int p) {
    double acc = 0.0;
    for (int k = 0; k < p; k++) {
        double diff = __dsub_rn(a[k], b[k]);
        acc = __fma_rn(diff, diff, acc);
    }
    return acc;
}

// Same with a strided second operand (SoA storage: b[k*stride]).
__device__ __forceinline__ double sqdist_fma_strided(const double *a, const double *b, int64_t stride,
                                                     int p) {
    double acc = 0.0;
    for (int k = 0; k < p; k++) {
        double diff = __dsub_rn(a[k], b[k * stride]);
        acc = __fma_rn(diff, diff, acc);
    }
    return acc;
}

// exp(x) for x <= 0, ~1 ulp: x = n ln2 + r with |r| <= ln2/2 (Cody–Waite split of
// ln2), e^r by a degree-13 Taylor polynomial (truncation < 1e-17 relative) in
// Horner form, then scaling by 2^n through the exponent field. x < -708 returns 0
// (the true value is below 1e-307). About 20 instructions against ~45 for the
// libdevice exp, whose overflow / NaN paths this argument range never needs.
__device__ __forceinline__ double exp_nonpos(double x) {
    if (x < -708.0) return 0.0;
    const double n = rint(x * 1.4426950408889634);
    // hi part first: x - n*ln2_hi is exact (Sterbenz), then the low part
    const double r = fma(n, -1.90821492927058770002e-10, fma(n, -6.93147180369123816490e-01, x));
    double q = 1.6059043836821613e-10;  // 1/13!
    q = fma(q, r, 2.0876756987868099e-09);  // 1/12!
    q = fma(q, r, 2.5052108385441720e-08);  // 1/11!
    q = fma(q, r, 2.7557319223985893e-07);  // 1/10!
    q = fma(q, r, 2.7557319223985888e-06);  // 1/9!
    q = fma(q, r, 2.4801587301587302e-05);  // 1/8!
    q = fma(q, r, 1.9841269841269841e-04);  // 1/7!
    q = fma(q, r, 1.3888888888888889e-03);  // 1/6!
    q = fma(q, r, 8.3333333333333332e-03);  // 1/5!
    q = fma(q, r, 4.1666666666666664e-02);  // 1/4!
    q = fma(q, r, 1.6666666666666666e-01);  // 1/3!
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    q = fma(q, r, 1.0);
    const int ni = (int)n;  // in [-1022, 0] here except the denormal tail handled below
    if (ni < -1021) return ldexp(q, ni);
    return __longlong_as_double(__double_as_longlong(q) + ((long long)ni << 52));
}

// exp(x) for x <= 0 from a 16-entry table, ~1 ulp, branch-free, no FP64<->int
// conversions (the hot-loop variant used by the incremental kernels):
//   N = round(16 x / ln2) by the 1.5*2^52 shifter (t = fma(x, 16/ln2, S), N in the
//   low bits of t), r = x - N ln2/16 (Cody-Waite, |r| <= ln2/32),
//   e^r - 1 by its degree-7 Taylor polynomial (truncation < 2e-18),
//   exp(x) = 2^m T[k] (1 + (e^r - 1)), N = 16 m + k, T[k] = 2^(k/16) (rounded).
// 16 entries = 16 distinct shared-memory bank pairs: a warp's table reads never
// conflict (equal indices broadcast). x is clamped at -708 (2^m stays normal) and
// the result selected to 0 below it; NaN propagates. `tab`: the 16 entries (shared).
__constant__ double c_exp2_16[16] = {
    1.0, 1.0442737824274138, 1.0905077326652577, 1.1387886347566916, 1.189207115002721, 1.241857812073484,
    1.2968395546510096, 1.3542555469368927, 1.4142135623730951, 1.4768261459394993, 1.5422108254079407,
    1.6104903319492543, 1.681792830507429, 1.7562521603732995, 1.8340080864093424, 1.9152065613971474};
__device__ __forceinline__ double exp_nonpos_tab(double x, const double *tab) {
    const double xc = fmax(x, -708.0);
    const double shifter = 6755399441055744.0;  // 1.5 * 2^52
    const double t = fma(xc, 23.083120654223414, shifter);  // 16 / ln2
    const double nd = t - shifter;
    const int N = (int)(unsigned)__double2loint(t);
    double r = fma(nd, -0.04332169877307024, xc);  // ln2_hi / 16 (32 significant bits)
    r = fma(nd, -1.1926343307941173e-11, r);       // ln2_lo / 16
    double p = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    const double pm1 = p * r;  // e^r - 1
    const double T = tab[N & 15];
    const double v0 = fma(T, pm1, T);
    const double v = __longlong_as_double(__double_as_longlong(v0) + ((long long)(N >> 4) << 52));
    return x < -708.0 ? 0.0 : (x == x ? v : x);
}
// The same for a finite x in [-708, 0] (the caller proves the range): no clamp, no
// NaN or underflow select, the 2^m scaling added to the high word only. Bitwise
// equal to exp_nonpos_tab on that domain.
__device__ __forceinline__ double exp_nonpos_tab_inrange(double x, const double *tab) {
    const double shifter = 6755399441055744.0;  // 1.5 * 2^52
    const double t = fma(x, 23.083120654223414, shifter);  // 16 / ln2
    const double nd = t - shifter;
    const int N = (int)(unsigned)__double2loint(t);
    double r = fma(nd, -0.04332169877307024, x);  // ln2_hi / 16
    r = fma(nd, -1.1926343307941173e-11, r);      // ln2_lo / 16
    double p = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    const double pm1 = p * r;  // e^r - 1
    const double T = tab[N & 15];
    const double v0 = fma(T, pm1, T);
    return __hiloint2double(__double2hiint(v0) + ((N >> 4) << 20), __double2loint(v0));
}

// s^{-1/2} for s > 0: reciprocal-square-root seed and two Newton steps
// (r <- r + r(1 - s r^2)/2); s <= 0 gives NaN (a non-PD append, flagged NONFINITE)
__device__ __forceinline__ double rsqrt_nr(double s) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
    double e = fma(-s * r, r, 1.0);
    r = fma(0.5 * r, e, r);
    e = fma(-s * r, r, 1.0);
    r = fma(0.5 * r, e, r);
    return s > 0.0 ? r : __longlong_as_double(0x7ff8000000000000LL);
}

// Isotropic Gaussian correlation exp(-d2/theta) with rtheta = 1/theta.
__device__ __forceinline__ double corr_from_d2(double d2, double rtheta) { return exp_nonpos(-d2 * rtheta); }

// (Delta, global index) order used by every argmax: larger Delta wins, equal
// Delta -> lower global row index (R7). Excluded candidates carry -inf.
__device__ __forceinline__ bool better(double da, int ia, double db, int ib) {
    return da > db || (da == db && (unsigned)ia < (unsigned)ib);
}

// Running top-2 for the argmax + gap: best (d1, i1) and second value d2.
struct Top2 {
    double d1, d2;
    int i1;
    int pos;  // pool position of the best
    __device__ __forceinline__ void init() {
        d1 = -INFINITY;
        d2 = -INFINITY;
        i1 = -1;
        pos = -1;
    }
    __device__ __forceinline__ void push(double d, int gi, int ps) {
        if (better(d, gi, d1, i1)) {
            d2 = d1;
            d1 = d;
            i1 = gi;
            pos = ps;
        } else if (d > d2) {
            d2 = d;
        }
    }
    // merge another Top2 (commutative & associative on the total order)
    __device__ __forceinline__ void merge(double od1, int oi1, int opos, double od2) {
        if (better(od1, oi1, d1, i1)) {
            d2 = fmax(d1, od2);
            d1 = od1;
            i1 = oi1;
            pos = opos;
        } else {
            d2 = fmax(d2, od1);
        }
    }
};

__device__ __forceinline__ void warp_merge_top2(Top2 &t) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double od1 = __shfl_xor_sync(0xffffffffu, t.d1, off);
        double od2 = __shfl_xor_sync(0xffffffffu, t.d2, off);
        int oi1 = __shfl_xor_sync(0xffffffffu, t.i1, off);
        int opos = __shfl_xor_sync(0xffffffffu, t.pos, off);
        t.merge(od1, oi1, opos, od2);
    }
}

// gap = (D1 - max(D2,0)) / D1, 0 when D1 <= 0 (same definition as the oracle).
__device__ __forceinline__ double top2_gap(double d1, double d2) {
    if (!(d1 > 0.0)) return 0.0;
    double d2c = d2 > 0.0 ? d2 : 0.0;
    return (d1 - d2c) / d1;
}

__device__ __forceinline__ double int_bits_to_double(int i) { return __longlong_as_double((long long)i); }
__device__ __forceinline__ int double_bits_to_int(double d) { return (int)__double_as_longlong(d); }

__device__ __forceinline__ uint64_t d2_key(double d2) { return (uint64_t)__double_as_longlong(d2); }

}  // namespace lagp
