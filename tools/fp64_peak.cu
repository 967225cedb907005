// fp64_peak.cu -- measured fp64 pipe throughput of this B200 (DADD and DFMA), the
// denominator of the kernels' "alu" roofline ("must be re-measured with a
// DFMA microbenchmark, since MEASURED_PEAKS.json has no fp64 entry").
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_peak.cu -o /tmp/fp64_peak
//   /tmp/fp64_peak > profiles/fp64_peak.json
//
// Every thread runs CH independent dependency chains (enough ILP to cover the pipe
// latency at any occupancy), ITERS times; grid = 148 SMs x BLOCKS_PER_SM CTAs of 256
// threads.  Reported: lane-instructions per second (one DADD or DFMA on one lane = 1;
// a DFMA is 2 flops), best of 5 after a warm-up, and the SM clock during the run.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 16;
constexpr int ITERS = 4096;

template <bool FMA>
__global__ void __launch_bounds__(256) burn(double *out, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = FMA ? __fma_rn(x[c], a, b) : __dadd_rn(x[c], b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[threadIdx.x] = s;  // keeps the chains alive, never taken
}

// The stencil's operand pattern: every DADD reads TWO different registers of a 1D array
// and writes a third (ping-pong, like K2's v[j] = u[j-1] + u[j+1]); the plain chains above
// read one register and a constant.  A gap between the two is register-file bandwidth.
__global__ void __launch_bounds__(256) burn_stencil(double *out, double b) {
    constexpr int NV = 34;
    double u[NV], v[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) u[c] = threadIdx.x * 1e-9 + c * b;
    for (int i = 0; i < ITERS / 2; ++i) {
#pragma unroll
        for (int c = 1; c < NV - 1; ++c) v[c] = __dadd_rn(u[c - 1], u[c + 1]);
        v[0] = u[1];
        v[NV - 1] = u[NV - 2];
#pragma unroll
        for (int c = 1; c < NV - 1; ++c) u[c] = __dadd_rn(v[c - 1], v[c + 1]);
        u[0] = v[1];
        u[NV - 1] = v[NV - 2];
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < NV; ++c) s += u[c];
    if (s == 12345.678) out[threadIdx.x] = s;
}

double run_stencil(int sms, int bps, double *out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * bps;
    burn_stencil<<<grid, 256>>>(out, 1e-7);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        burn_stencil<<<grid, 256>>>(out, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double inst = (double)grid * 256 * ITERS * 32;  // 32 DADD per half-iteration pair x 2
    return inst / (best * 1e-3) / 1e12;
}

template <bool FMA>
double run(int sms, int bps, double *out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * bps;
    burn<FMA><<<grid, 256>>>(out, 0.999999, 1e-7);  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        burn<FMA><<<grid, 256>>>(out, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double inst = (double)grid * 256 * ITERS * CH;
    return inst / (best * 1e-3) / 1e12;  // T lane-instructions / s
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    double *out;
    cudaMalloc(&out, 256 * sizeof(double));
    printf("{\"sms\": %d, \"sm_clock_max_mhz\": %.0f, \"chains_per_thread\": %d, \"results\": [", sms, clk_khz / 1e3, CH);
    bool first = true;
    for (int bps : {1, 2, 4, 8}) {
        const double dadd = run<false>(sms, bps, out), dfma = run<true>(sms, bps, out);
        const double sten = run_stencil(sms, bps, out);
        printf("%s{\"blocks_per_sm\": %d, \"dadd_tinst_s\": %.3f, \"dfma_tinst_s\": %.3f, \"dfma_tflops\": %.3f, "
               "\"stencil_dadd_tinst_s\": %.3f}",
               first ? "" : ", ", bps, dadd, dfma, 2 * dfma, sten);
        first = false;
    }
    printf("], \"derived_tinst_s\": %.3f}\n", sms * 64.0 * clk_khz * 1e3 / 1e12);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
