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

// Isotropic Gaussian correlation exp(-d2/theta) with rtheta = 1/theta.
__device__ __forceinline__ double corr_from_d2(double d2, double rtheta) { return exp(-d2 * rtheta); }

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
