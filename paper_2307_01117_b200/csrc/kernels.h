// kernels.h -- internal launcher interface between the runtime (heat1d.cpp)
// and the sm_100a kernels (kernels.cu).  Not part of the public C ABI.
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace heat1d {

// Arithmetic variants of Eq. 2 (see stencil.cuh).
enum Ops { OPS_LITERAL5 = 5, OPS_MATCHED4 = 4, OPS_FMA3 = 3, OPS_SCALED2 = 2, OPS_SCALED1 = 1 };

// Scaled variants work on v = u / r^t: true iff a pass must end with u = v * r^T'.
__host__ __device__ constexpr bool ops_scaled(int ops) { return ops <= 2; }

// r^T' as the left-to-right product ((1*r)*r)*...  -- host and device evaluate
// the same sequence of IEEE products, so every kernel rescales by the same bits.
__host__ __device__ inline double scale_of(double r, int Tp) {
    double s = 1.0;
    for (int i = 0; i < Tp; ++i) s = s * r;
    return s;
}


// Exactness guard of the contracted matched forms (stencil.cuh): a block of steps runs
// its OPS only if its cells' keys (GuardAcc) satisfy min(key - 1) >= kmin1 and
// max(key) <= kmax, else the literal 5-op sequence.  {0, 0xffffffff} = no guard.
struct Guard {
    uint32_t kmin1 = 0u, kmax = 0xffffffffu;
};

// The guard of a block of Tp steps of Eq. 2 with coefficient r in arithmetic `ops`
// (matched: the result must equal the literal sequence bitwise; fast: no guard).
inline Guard guard_of(bool matched, int ops, double r, int Tp) {
    Guard g;
    if (!matched || (ops != 3 && ops != 4)) return g;
    // top: max|u| grows by at most G = max(1, 4r) per step (DESIGN.md c3): |x| < 2^(E-1023)
    const double G = r > 0.5 ? 4.0 * r : 1.0;
    const double E = 2045.0 - std::ceil((double)Tp * std::log2(G));  // biased exponent bound
    g.kmax = E < 1.0 ? 0u : (uint32_t)E * (1u << 21) - 1u;
    // bottom: r = 2^-j, j >= 1, 3-op form: x == 0 or |x| >= 2^(e-1023), e = 1 + j*Tp
    if (ops == 3 && r > 0.0 && r < 1.0) {
        int ex = 0;
        (void)std::frexp(r, &ex);  // r = 0.5 * 2^ex = 2^-j
        const double e = 1.0 + (double)(1 - ex) * (double)Tp;
        g.kmin1 = e >= 2047.0 ? 0xffffffffu : (uint32_t)e * (1u << 21) - 1u;
    }
    return g;
}

// Fast mode's scaled forms (OPS 2, 1; stencil.cuh, DESIGN.md c21) reach max|u0| * r^-T within
// a pass and must stay below 2^1000: the kernels compare K5's max|u| word (the bit pattern of a
// non-negative double) with `limit` and, if it is larger, run the contracted 3-op form with the
// coefficient r instead -- decided on the device, CTA-uniformly, so set_initial needs no host
// round trip.  absmax == nullptr: always the scaled form.
struct FastRange {
    const unsigned long long *absmax = nullptr;
    unsigned long long limit = ~0ull;
    double r = 0.0;
};

// Ghost depth (= steps between exchanges) of the inter-warp exchange of pass-kernel
// kinds 3 (8) and 4 (16).
constexpr int kx_of(int kind) { return kind == 3 ? 8 : kind == 4 ? 16 : 0; }

// Geometry of the temporal-blocked pass kernel (K2) for one launch config.
struct PassGeom {
    int V;            // cells per thread (odd: conflict-free 64-bit LDS/STS)
    int NW;           // compute warps per CTA (plus one TMA producer warp)
    int S;            // TMA pipeline stages per CTA
    int ctas_per_sm;  // resident CTAs per SM the config is sized for (capped by occupancy)
    int kind = 4;     // 3, 4: compute warps trade kx_of(kind)-deep ghosts through shared memory
                      // every kx_of(kind) steps (only the CTA edges keep the T trapezoid)
    size_t smem_bytes(int T) const;
    // output cells per CTA tile
    int64_t tile_out(int T) const {
        return (int64_t)NW * 32 * V - 2 * (int64_t)kx_of(kind) * (NW - 1) - 2 * T;
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
// q = the variant's per-step coefficient, scale = r^T (scaled variants only; stencil.cuh),
// guard = the exactness guard (guard_of; guarded variants only).
// whether launch_pass runs a full pass of depth T as feed tiles (k2f_pass)
bool pass_uses_feed(const PassGeom &g, int ops, int T);

cudaError_t launch_pass(const PassGeom &g, int ops, const double *A, double *B, int64_t n,
                        int T, int64_t out_lo, int64_t out_hi, int wrapT, double q, double scale,
                        Guard guard, const FastRange &fr, int num_sms, cudaStream_t st, int *grid_out);

// K1: one step over the whole ring with modular indexing (no pads used); ops 5 (literal,
// matched mode) or 3 (fast mode).
cudaError_t launch_naive(int ops, const double *A, double *B, int64_t n, double r, cudaStream_t st);

// K3: the two edge strips [0,T) and [n-T,n) of a slab after its ghosts arrived.
cudaError_t launch_edges(int ops, const double *A, double *B, int64_t n, int T, double q, double scale,
                         Guard guard, const FastRange &fr, cudaStream_t st);

// K3p: K3 fused with a peer-memory halo put (kernels.cu).  my_flags: this slab's two
// exchange-index words (side 0 at +0, side 1 at +32); put_left/right: where the new
// left/right strips go in the neighbours' B (their right/left pads); flag_left/right:
// the neighbours' words for those pads.  Waits for index g, releases g+1.
cudaError_t launch_edges_put(int ops, const double *A, double *B, int64_t n, int T, double q, double scale,
                             Guard guard, const FastRange &fr, const unsigned *my_flags, unsigned g, double *put_left, double *put_right,
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

// K6 across ranks: each rank's mailbox = [2 sides][2 slots][MBOX_TMAX] cells of 16 bytes (two
// tagged words, resident.cu; the V = 17 flag protocol uses them as plain doubles) + two flag
// words on their own 128-byte lines at MBOX_FLAG_OFF (side 0: from the left rank, side 1:
// from the right rank).  left/right point at the neighbour ranks' mailboxes (CUDA IPC peer
// mappings over NVLink; == self for one rank, which routes the ring's wrap through them).
constexpr int MBOX_TMAX = 128;
constexpr size_t MBOX_FLAG_OFF = 2 * 2 * MBOX_TMAX * 16;
constexpr size_t MBOX_BYTES = MBOX_FLAG_OFF + 256;
struct MboxArgs {
    double *self = nullptr, *left = nullptr, *right = nullptr;
    unsigned base = 0;  // first global exchange index of this launch
    int on = 0;
};

// Initialise a mailbox: every data word tag 0 (never a live tag), flag words 0.
cudaError_t launch_mbox_init(double *mbox, cudaStream_t st);

// K6: whole nt-step solve of a single-slab ring held in registers (resident.cu).
int64_t resident_capacity(int T, int num_sms);
bool resident_fits(int ops, int64_t n, int T, int num_sms, bool mbox = false);  // plan + co-residency
int resident_plan_v(int ops, int64_t n, int T, int num_sms, bool mbox);  // cells per lane of the plan, 0: no fit
size_t resident_scratch_bytes(int T, int num_sms);
cudaError_t resident_scratch_init(void *scratch, int T, int num_sms, cudaStream_t st);
cudaError_t launch_resident(int ops, const double *A, double *B, int64_t n, int T, int64_t nt, double q,
                            double r, Guard guard, const FastRange &fr, void *scratch, int num_sms, cudaStream_t st,
                            int *warps_out, int *v_out, const MboxArgs &mb,
                            unsigned tbase);  // tag of this launch's first period (>= 1, new per launch)

}  // namespace heat1d
