// kernels.h -- internal launcher interface between the runtime (heat1d.cpp)
// and the sm_100a kernels (kernels.cu).  Not part of the public C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace heat1d {

// Arithmetic variants of Eq. 2 (see stencil.cuh).
enum Ops { OPS_MATCHED4 = 4, OPS_FMA3 = 3, OPS_SCALED2 = 2, OPS_SCALED1 = 1 };

// Scaled variants work on v = u / r^t: true iff a pass must end with u = v * r^T'.
__host__ __device__ constexpr bool ops_scaled(int ops) { return ops <= 2; }

// r^T' as the left-to-right product ((1*r)*r)*...  -- host and device evaluate
// the same sequence of IEEE products, so every kernel rescales by the same bits.
__host__ __device__ inline double scale_of(double r, int Tp) {
    double s = 1.0;
    for (int i = 0; i < Tp; ++i) s = s * r;
    return s;
}


// Ghost depth (= steps between exchanges) of the inter-warp exchange of pass-kernel
// kinds 3 (8) and 4 (16); 0 for the other kinds.
constexpr int kx_of(int kind) { return kind == 3 ? 8 : kind == 4 ? 16 : 0; }

// Geometry of the temporal-blocked pass kernel (K2) for one launch config.
struct PassGeom {
    int V;            // cells per thread (odd: conflict-free 64-bit LDS/STS)
    int NW;           // compute warps per CTA
    int S;            // TMA pipeline stages (per CTA for kind 0, per warp for kind 1)
    int ctas_per_sm;  // resident CTAs per SM the config is sized for (capped by occupancy)
    int kind = 1;     // 0: CTA tiles (one TMA copy per CTA tile, 2 CTA barriers per tile)
                      // 1: warp-autonomous spans (each warp its own TMA ring; no CTA barriers)
                      // 2: CTA tiles + a dedicated TMA producer warp (NW+1 warps per CTA)
                      // 3, 4: kind 2 + compute warps trade kx_of(kind)-deep ghosts through
                      //    shared memory every kx_of(kind) steps (only the CTA edges keep the
                      //    T trapezoid)
    size_t smem_bytes(int T) const;
    // output cells per scheduling unit (a CTA tile for kind 0, a warp span for kind 1)
    int64_t tile_out(int T) const {
        if (kx_of(kind)) return (int64_t)NW * 32 * V - 2 * (int64_t)kx_of(kind) * (NW - 1) - 2 * T;
        return (kind != 1 ? (int64_t)NW : 1) * (32 * V - 2 * T);
    }
};

// True iff the pass kernel is instantiated for this geometry and arithmetic variant.
bool pass_supported(const PassGeom &g, int ops);

// Pick the pass-kernel configuration for (n, T).
PassGeom choose_geom(int64_t n_out, int T, int num_sms, int ops);

// K2: T fused Jacobi steps over outputs [out_lo, out_hi) of a slab.
// A, B point at cell 0 of padded slab buffers (ghost cells at negative
// offsets and at [n, n+pad)).  Reads A[out_lo-T, out_hi+T), writes B[out_lo, out_hi).
// wrapT > 0 (single-slab ring): cells [0,wrapT) are also written to
// B[n, n+wrapT) and cells [n-wrapT, n) to B[-wrapT, 0)  (periodic self-halo).
// q = the variant's per-step coefficient, scale = r^T (scaled variants only; stencil.cuh).
cudaError_t launch_pass(const PassGeom &g, int ops, const double *A, double *B, int64_t n,
                        int T, int64_t out_lo, int64_t out_hi, int wrapT, double q, double scale,
                        int num_sms, cudaStream_t st, int *grid_out);

// K1: one step over the whole ring with modular indexing (no pads used).
cudaError_t launch_naive(int ops, const double *A, double *B, int64_t n, double r, cudaStream_t st);

// K3: the two edge strips [0,T) and [n-T,n) of a slab after its ghosts arrived.
cudaError_t launch_edges(int ops, const double *A, double *B, int64_t n, int T, double q, double scale,
                         cudaStream_t st);

// K3p: K3 fused with a peer-memory halo put (kernels.cu).  my_flags: this slab's two
// exchange-index words (side 0 at +0, side 1 at +32); put_left/right: where the new
// left/right strips go in the neighbours' B (their right/left pads); flag_left/right:
// the neighbours' words for those pads.  Waits for index g, releases g+1.
cudaError_t launch_edges_put(int ops, const double *A, double *B, int64_t n, int T, double q, double scale,
                             const unsigned *my_flags, unsigned g, double *put_left, double *put_right,
                             unsigned *flag_left, unsigned *flag_right, cudaStream_t st);
// Push A[0,T) / A[n-T,n) into the neighbours' pads and release their flags with g+1.
cudaError_t launch_push_edges(const double *A, int64_t n, int T, unsigned g, double *put_left, double *put_right,
                              unsigned *flag_left, unsigned *flag_right, cudaStream_t st);

// Test-only fault injection: a kernel that spins `us` microseconds on `st`.
cudaError_t launch_delay(unsigned us, cudaStream_t st);

// K4: fill `pad` ghost cells on each side of a single-slab ring, modularly.
cudaError_t launch_wrap_fill(double *A, int64_t n, int64_t pad, cudaStream_t st);

// K5: *out = max(*out, bits of max |u[i]|)  (caller zeroes *out first).
cudaError_t launch_absmax(const double *u, int64_t count, unsigned long long *out, cudaStream_t st);

// K0: u[i] = lo + (hi-lo) * U(seed, first+i), splitmix64 counter form.
cudaError_t launch_init_uniform(double *u, int64_t count, int64_t first, uint64_t seed,
                                double lo, double hi, cudaStream_t st);

// K6 across ranks: each rank's mailbox = double[2 sides][2 slots][MBOX_TMAX] + two flag
// words on their own 128-byte lines at MBOX_FLAG_OFF (side 0: from the left rank, side 1:
// from the right rank).  left/right point at the neighbour ranks' mailboxes (CUDA IPC peer
// mappings over NVLink; == self for one rank, which routes the ring's wrap through them).
constexpr int MBOX_TMAX = 128;
constexpr size_t MBOX_FLAG_OFF = 2 * 2 * MBOX_TMAX * sizeof(double);
constexpr size_t MBOX_BYTES = MBOX_FLAG_OFF + 256;
struct MboxArgs {
    double *self = nullptr, *left = nullptr, *right = nullptr;
    unsigned base = 0;  // first global exchange index of this launch
    int on = 0;
};

// Initialise a mailbox: data slots to the data-as-flag EMPTY pattern, flag words to 0.
cudaError_t launch_mbox_init(double *mbox, cudaStream_t st);

// K6: whole nt-step solve of a single-slab ring held in registers (resident.cu).
int64_t resident_capacity(int T, int num_sms);
bool resident_fits(int ops, int64_t n, int T, int num_sms, bool mbox = false);  // plan + co-residency
size_t resident_scratch_bytes(int T, int num_sms);
cudaError_t resident_scratch_init(void *scratch, int T, int num_sms, cudaStream_t st);
cudaError_t launch_resident(int ops, const double *A, double *B, int64_t n, int T, int64_t nt, double q,
                            double r, void *scratch, int num_sms, cudaStream_t st, int *warps_out,
                            const MboxArgs &mb = MboxArgs{});

}  // namespace heat1d
