// stencil.cuh -- Eq. 2 of arxiv 2307.01117 as fp64 device code.
//
//   u(t+dt, x_i) = u_i + r * ((u_{i-1} - 2 u_i) + u_{i+1}),   r = k*dt/dx^2
//
// The expression order is the canonical one of DESIGN.md reading c3.  nvcc
// contracts a*b+c into DFMA by default, so every operation is spelled with an
// explicit round-to-nearest intrinsic.  `q` is the per-step coefficient the
// host passes for the variant (r for OPS 5/4/3, c = (1-2r)/r for OPS 2, unused
// for OPS 1):
//
//  OPS_LITERAL5 (any r, any state): DMUL(2*b)  DADD(a-)  DADD(+c)  DMUL(r*)  DADD(b+)
//     the oracle's own sequence, operation for operation.  The exactness
//     fallback of the two contracted matched forms below (DESIGN.md c3).
//  OPS_MATCHED4 (any r): DFMA(-2,b,a)  DADD(+c)  DMUL(r*)  DADD(b+)
//     fma(-2,b,a) == a - 2.0*b bitwise while 2b is finite, i.e. |b| < 2^1023;
//     the rest is the literal left-to-right sequence.
//  OPS_FMA3 (r a power of two, or fast mode): DFMA(-2,b,a)  DADD(+c)  DFMA(r,t,b)
//     for r = 2^-j, fma(r,t,b) == b + r*t bitwise iff r*t is exact, i.e. unless
//     r*t lands in the subnormal range with bits below 2^-1074 (DESIGN.md c3).
//     For other r this is the contracted "fast" form (one rounding fewer),
//     error <= 1e-12*max|u0|*nt.
//  OPS_SCALED2 (fast mode, 1/256 <= r < 1/2): Eq. 2 is u' = (1-2r) u_i + r (u_{i-1} + u_{i+1});
//     the scaled state v_t = u_t / r^t obeys  v' = c v_i + (v_{i-1} + v_{i+1}),
//     c = (1-2r)/r:  DADD, DFMA per update.  A pass of T' steps starts from
//     v = u and ends with u = v * r^T' (one DMUL per cell per pass).
//  OPS_SCALED1 (fast mode, r = 1/2 exactly, c = 0):  v' = v_{i-1} + v_{i+1}:
//     ONE DADD per update; the final scaling by 2^-T' is exact, so every step
//     equals fl(a + c) * 1/2 (DESIGN.md §3 c21).
//
// Exactness guard of the contracted matched forms (OPS 4 and 3, DESIGN.md c3).
// Every kernel checks the cells its block of steps starts from (a K2 tile, a K3
// strip, a K6 span period) and runs that block with OPS_LITERAL5 unless every
// cell x passes (GuardAcc below; Guard and guard_of in kernels.h):
//   top:    |x| < 2^(E - 1023), E = 2045 - ceil(Tp log2 G), G = 1 for
//           r <= 1/2, 4r above.  Eq. 2 is a convex combination for r <= 1/2 and
//           grows max|u| by at most 4r per step otherwise, so (with the roundings'
//           (1+6 eps) per step) no value of the block reaches 2^1022: 2b never
//           overflows (OPS 4 and 3 exact) and neither does r*t.
//   bottom: x == 0 or |x| >= 2^(e - 1023), e = 1 + j*Tp for the 3-op
//           form with r = 2^-j (j >= 1), else 0.  Let q(x) be the largest power of
//           two dividing x.  Sums, differences and their roundings keep q >= the
//           operands' minimum and r*t divides it by 2^j, so after s steps every q is
//           >= 2^(j(Tp-s) - 1074); the step-s product r*t is a multiple of 2^-1074,
//           i.e. exactly representable, for every s < Tp (OPS 3 exact).
// The check is 5 integer instructions per cell per block, not per step.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"  // ops_scaled, scale_of

namespace heat1d {

template <int OPS>
__device__ __forceinline__ double eq2(double a, double b, double c, double q) {
    if constexpr (OPS == 1) {
        return __dadd_rn(a, c);                // v_{i-1} + v_{i+1}
    } else if constexpr (OPS == 2) {
        return __fma_rn(q, b, __dadd_rn(a, c));  // c*v_i + (v_{i-1} + v_{i+1})
    } else if constexpr (OPS == 5) {
        double t = __dmul_rn(2.0, b);          // 2.0*b
        t = __dsub_rn(a, t);                   // a - 2.0*b
        t = __dadd_rn(t, c);                   // (a - 2.0*b) + c
        t = __dmul_rn(q, t);                   // r * (...)
        return __dadd_rn(b, t);                // b + r*(...)
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

// Guarded variants: the contracted matched forms (and the 3-op fast fallback).
#ifdef HEAT1D_NO_GUARD  // measurement builds only (tools/ab_build.py): the guard's cost
__host__ __device__ constexpr bool ops_guarded(int) { return false; }
#else
__host__ __device__ constexpr bool ops_guarded(int ops) { return ops == 3 || ops == 4; }
#endif

// The guard's per-cell key: 2 * (high word without the sign) + (low word != 0).  It orders
// like |x|, is 0 only for x == 0, and a bound on the exponent field (e << 20 in the high
// word) becomes e << 21 in key space.  A block passes iff min(key - 1) >= g.kmin1 (every
// nonzero cell at or above the bottom bound; zero keys wrap to 0xffffffff) and
// max(key) <= g.kmax (every cell below the top bound).  5 integer instructions per cell.
struct GuardAcc {
    uint32_t mn = 0xffffffffu, mx = 0u;
    __device__ __forceinline__ void add(double x) {
        const uint32_t hi = (uint32_t)__double2hiint(x);
        const uint32_t lo = (uint32_t)__double2loint(x);
        const uint32_t key = hi + hi + min(lo, 1u);  // (the sign bit shifts out)
        mx = max(mx, key);
        mn = min(mn, key - 1u);
    }
    __device__ __forceinline__ bool ok(Guard g) const { return mn >= g.kmin1 && mx <= g.kmax; }
};

// FastRange (kernels.h): may the scaled fast form run?  (K5 wrote the word in an earlier launch.)
__device__ __forceinline__ bool scaled_in_range(const FastRange &f) { return !f.absmax || *f.absmax <= f.limit; }

// Bounds checks of a checked measurement build (tools/ab_build.py checked=HEAT1D_CHECKED; the
// pool's compute-sanitizer is closed): every shared/global index the kernels derive is
// asserted; a violation prints and traps (the handle reports ECUDA).  No code otherwise.
#ifdef HEAT1D_CHECKED
#include <cstdio>
#define HCHECK(cond)                                                                          \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("HCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                        \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define HCHECK(cond) \
    do {             \
    } while (0)
#endif

__device__ __forceinline__ uint32_t dynamic_smem_bytes() {
    uint32_t b;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(b));
    return b;
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
