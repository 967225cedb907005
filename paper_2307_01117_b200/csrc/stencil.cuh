// stencil.cuh -- Eq. 2 of arxiv 2307.01117 as fp64 device code.
//
//   u(t+dt, x_i) = u_i + r * ((u_{i-1} - 2 u_i) + u_{i+1}),   r = k*dt/dx^2
//
// The expression order is the canonical one of DESIGN.md reading c3.  nvcc
// contracts a*b+c into DFMA by default, so every operation is spelled with an
// explicit round-to-nearest intrinsic:
//
//  OPS_MATCHED4 (any r): DFMA(-2,b,a)  DADD(+c)  DMUL(r*)  DADD(b+)
//     fma(-2,b,a) == a - 2.0*b bitwise because 2b is exact (no overflow for
//     |b| < 2^1023); the rest is the literal left-to-right sequence.
//  OPS_FMA3 (r a power of two, or fast mode): DFMA(-2,b,a)  DADD(+c)  DFMA(r,t,b)
//     for r = 2^-j, r*t is exact unless it is subnormal, so fma(r,t,b) ==
//     b + r*t bitwise (DESIGN.md §3 c3).  For other r this is the contracted
//     "fast" form (one rounding fewer), error <= 1e-12*max|u0|*nt.
#pragma once
#include <cuda_runtime.h>

namespace heat1d {

template <int OPS>
__device__ __forceinline__ double eq2(double a, double b, double c, double r) {
    double t = __fma_rn(-2.0, b, a);   // a - 2b   (exact product, one rounding)
    t = __dadd_rn(t, c);               // (a - 2b) + c
    if constexpr (OPS == 4) {
        t = __dmul_rn(r, t);           // r * (...)
        return __dadd_rn(b, t);        // b + r*(...)
    } else {
        return __fma_rn(r, t, b);      // b + r*(...) in one rounding
    }
}

// The same three (or four) operations split into phases so that a thread can
// issue one phase for all of its V cells before the next: consecutive
// dependent operations are then V instructions apart, which hides the fp64
// pipe latency without relying on other warps.  eq2 == p3(p2(p1(a,b),c),b,r).
__device__ __forceinline__ double eq2_p1(double a, double b) { return __fma_rn(-2.0, b, a); }
__device__ __forceinline__ double eq2_p2(double t, double c) { return __dadd_rn(t, c); }
template <int OPS>
__device__ __forceinline__ double eq2_p3(double t, double b, double r) {
    if constexpr (OPS == 4)
        return __dadd_rn(b, __dmul_rn(r, t));
    else
        return __fma_rn(r, t, b);
}

}  // namespace heat1d
