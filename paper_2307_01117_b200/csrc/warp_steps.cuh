// warp_steps.cuh -- T Jacobi steps of Eq. 2 on a warp-row of 32*V
// cells held V per lane in registers: the inner loop of the pass kernel K2 (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include "stencil.cuh"

namespace heat1d {

// One Jacobi step of a warp-row of 32*V cells held V per lane: u -> v.
// The two inter-lane neighbours come by shuffle (issued first, consumed last);
// the cells of the warp's two outermost lanes go stale by one cell per step.
template <int V, int OPS>
__device__ __forceinline__ void warp_step(const double (&u)[V], double (&v)[V], double r) {
    const double L = __shfl_up_sync(0xffffffffu, u[V - 1], 1);
    const double R = __shfl_down_sync(0xffffffffu, u[0], 1);
#pragma unroll
    for (int j = 1; j < V - 1; ++j) v[j] = eq2<OPS>(u[j - 1], u[j], u[j + 1], r);
    v[0] = eq2<OPS>(L, u[0], u[1], r);
    v[V - 1] = eq2<OPS>(u[V - 2], u[V - 1], R, r);
}

// N (even, compile time) steps fully unrolled: the sub-periods of the 1-op form, with
// no loop control between steps; the result is left in u.
template <int V, int OPS, int N>
__device__ __forceinline__ void warp_steps_fixed(double (&u)[V], double r) {
    static_assert(N % 2 == 0, "even step count keeps the result in u");
    double v[V];
#pragma unroll
    for (int s = 0; s < N; s += 2) {
        warp_step<V, OPS>(u, v, r);
        warp_step<V, OPS>(v, u, r);
    }
}

// T steps in registers, ping-pong between u and a scratch array (no moves
// inside the loop); the result is left in u.
template <int V, int OPS>
__device__ __forceinline__ void warp_steps(double (&u)[V], int T, double r) {
    double v[V];
    int s = 0;
    for (; s + 2 <= T; s += 2) {
        warp_step<V, OPS>(u, v, r);
        warp_step<V, OPS>(v, u, r);
    }
    if (s < T) {
        warp_step<V, OPS>(u, v, r);
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = v[j];
    }
}

}  // namespace heat1d
