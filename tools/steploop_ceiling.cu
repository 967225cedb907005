// Ceiling of K2's step loop alone (measurement aid, not product): every warp runs the same
// warp_steps<V, OPS> instruction stream as k2p_pass on registers, with no tiles, TMA,
// inter-warp exchanges or barriers, at K2's launch shape (2 CTAs of 4+1 warps per SM, the
// 5th warp idle like the producer).  Reports fp64 instructions per second vs the pipe peak.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2307_01117_b200/csrc -I include \
//        tools/steploop_ceiling.cu -o steploop && ./steploop
#include <cstdio>
#include <cuda_runtime.h>

#include "warp_steps.cuh"

using namespace heat1d;

template <int V, int OPS>
__global__ void __launch_bounds__(160, 2) steploop(double *out, int steps, double r) {
    if ((threadIdx.x >> 5) == 4) return;  // the idle "producer" warp
    double u[V];
#pragma unroll
    for (int j = 0; j < V; ++j) u[j] = 0.25 + 1e-3 * (threadIdx.x + j);
    warp_steps<V, OPS>(u, steps, r);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < V; ++j) acc += u[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V, int OPS>
void run(const char *name, int ops_per_update) {
    const int sms = 148, grid = 2 * sms, steps = 4096;
    double *out;
    cudaMalloc(&out, grid * 160 * sizeof(double));
    steploop<V, OPS><<<grid, 160>>>(out, 64, 0.5);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        steploop<V, OPS><<<grid, 160>>>(out, steps, 0.5);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double lanes = (double)grid * 4 * 32 * V;  // cells updated per step
    const double inst = lanes * steps * ops_per_update / 32.0;  // warp-level fp64 instructions
    const double tinst = inst * 32.0 / (best / 1e3) / 1e12;   // lane-instructions / s (T)
    printf("{\"loop\": \"%s\", \"V\": %d, \"ops\": %d, \"ms\": %.3f, \"fp64_tinst_s\": %.3f, \"glups\": %.1f}\n", name, V,
           ops_per_update, best, tinst, lanes * steps / (best / 1e3) / 1e9);
    cudaFree(out);
}

int main() {
    run<51, 3>("warp_steps 3-op (matched r=2^-j)", 3);
    run<51, 4>("warp_steps 4-op (matched)", 4);
    run<51, 1>("warp_steps 1-op (fast r=1/2)", 1);
    run<51, 2>("warp_steps 2-op (fast)", 2);
    return 0;
}
