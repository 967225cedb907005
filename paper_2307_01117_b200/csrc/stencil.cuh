// stencil.cuh -- Eq. 2 of arxiv 2307.01117 as fp64 device code.
//
//   u(t+dt, x_i) = u_i + r * ((u_{i-1} - 2 u_i) + u_{i+1}),   r = k*dt/dx^2
//
// The expression order is the canonical one of DESIGN.md reading c3.  nvcc
// contracts a*b+c into DFMA by default, so every operation is spelled with an
// explicit round-to-nearest intrinsic.  `q` is the per-step coefficient the
// host passes for the variant (r for OPS 4/3, c = (1-2r)/r for OPS 2, unused
// for OPS 1):
//
//  OPS_MATCHED4 (any r): DFMA(-2,b,a)  DADD(+c)  DMUL(r*)  DADD(b+)
//     fma(-2,b,a) == a - 2.0*b bitwise because 2b is exact (no overflow for
//     |b| < 2^1023); the rest is the literal left-to-right sequence.
//  OPS_FMA3 (r a power of two, or fast mode): DFMA(-2,b,a)  DADD(+c)  DFMA(r,t,b)
//     for r = 2^-j, r*t is exact unless it is subnormal, so fma(r,t,b) ==
//     b + r*t bitwise (DESIGN.md §3 c3).  For other r this is the contracted
//     "fast" form (one rounding fewer), error <= 1e-12*max|u0|*nt.
//  OPS_SCALED2 (fast mode, 1/256 <= r < 1/2): Eq. 2 is u' = (1-2r) u_i + r (u_{i-1} + u_{i+1});
//     the scaled state v_t = u_t / r^t obeys  v' = c v_i + (v_{i-1} + v_{i+1}),
//     c = (1-2r)/r:  DADD, DFMA per update.  A pass of T' steps starts from
//     v = u and ends with u = v * r^T' (one DMUL per cell per pass).
//  OPS_SCALED1 (fast mode, r = 1/2 exactly, c = 0):  v' = v_{i-1} + v_{i+1}:
//     ONE DADD per update; the final scaling by 2^-T' is exact, so every step
//     equals fl(a + c) * 1/2 (DESIGN.md §3 c21).
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"  // ops_scaled, scale_of

namespace heat1d {

template <int OPS>
__device__ __forceinline__ double eq2(double a, double b, double c, double q) {
    if constexpr (OPS == 1) {
        return __dadd_rn(a, c);                // v_{i-1} + v_{i+1}
    } else if constexpr (OPS == 2) {
        return __fma_rn(q, b, __dadd_rn(a, c));  // c*v_i + (v_{i-1} + v_{i+1})
    } else {
        double t = __fma_rn(-2.0, b, a);   // a - 2b   (exact product, one rounding)
        t = __dadd_rn(t, c);               // (a - 2b) + c
        if constexpr (OPS == 4) {
            t = __dmul_rn(q, t);           // r * (...)
            return __dadd_rn(b, t);        // b + r*(...)
        } else {
            return __fma_rn(q, t, b);      // b + r*(...) in one rounding
        }
    }
}

// Cross-rank waits (peer-memory flags) must not hang a process forever if a neighbour
// rank died or diverged: after HEAT1D_WAIT_NS of polling the kernel traps (the CUDA
// error poisons the handle; the caller sees HEAT1D_ECUDA instead of a hang).
constexpr unsigned long long HEAT1D_WAIT_NS = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

}  // namespace heat1d
