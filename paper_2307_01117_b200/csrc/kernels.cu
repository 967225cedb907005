// kernels.cu -- sm_100a kernels of libheat1d.
//
//   K2 k2f_pass     T fused Jacobi steps of Eq. 2 per HBM pass (the hot kernel): TMA
//                   producer warp, register-resident warp spans trading 16-deep ghost zones
//                   between warps, CTAs walking strips of left-fed tiles (full passes at
//                   T = 64/96/128 on the default geometry)
//      k2p_pass     the same with round-robin tiles and both T-deep margins (other T, tail
//                   passes; kind 3 = 8-deep exchanges for small slabs)
//   K1 k1_naive     one step per launch, modular indexing (T = 1 baseline)
//   K3 k3_edges     the two T-wide edge strips of a slab once its ghosts arrived
//   K3p k3_edges_put  K3 fused with the halo put into the neighbours' pads (P2P
//                   transport), with k_push_edges for the start of a run
//   K4 k4_wrap_fill periodic self-halo of a single-slab ring
//   K5 k5_absmax    max |u| of an initial state (fast mode's scaled-state range check)
//   K0 k0_uniform   splitmix64 initial condition (same counter generator as synth/)
//   (K6, the whole-solve resident kernel, is resident.cu)
//
// Eq. 2 on the periodic ring, segmented with
// ghost zones.  The arithmetic is stencil.cuh; DESIGN.md §6
// describes the data layout and the roofline of each kernel.
#include <cstdio>
#include <cstdint>
#include <mutex>

#include "kernels.h"
#include "stencil.cuh"
#include "warp_steps.cuh"

namespace heat1d {

// ------------------------------------------------------------------ PTX helpers
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Producer-side wait: the tile it waits for takes ~10 us of compute, so poll with a
// ~0.25 us back-off sleep -- a spinning (or hardware-suspend-retrying) producer warp
// otherwise takes ~7 % of the issue slots of the SM sub-partition it shares with
// compute warps (ncu: NANOSLEEP.SYNCS retry loop, profiles/r01_ncu_k2p_c4_fast_T96.txt).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) __nanosleep(256);
}

// Same, but the waiting thread is suspended in hardware until the phase completes (or the
// time hint, in ns, runs out) instead of re-issuing try_wait: a waiting warp then takes no
// issue slots from the compute warps sharing its SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!ok);
}

// TMA 1D bulk copy global -> shared, completion counted on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// TMA 1D bulk copy shared -> global, tracked by bulk async-groups.
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Order this thread's generic-proxy shared-memory accesses before later async-proxy (TMA) ones.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}



}  // namespace

// Named barrier 1 among the compute warps, AND-reducing a predicate (bar.red.and).
template <int NTHREADS>
__device__ __forceinline__ bool bar1_and(bool ok) {
    uint32_t res;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 q, %1, 0;\n\t"
        "bar.red.and.pred p, 1, %2, q;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(res)
        : "r"((uint32_t)ok), "n"(NTHREADS)
        : "memory");
    return res != 0;
}

// ------------------------------------------------------------------ K2
//
// k2p_pass: persistent CTAs of NW compute warps plus one TMA producer warp walk
// output tiles, round robin.  Tile [x0, x1) needs inputs [x0-T, x1+T): the
// producer's 1D bulk copy (aligned down/up to 16 B; SASS UBLKCP) lands them in an
// S-stage shared-memory ring (mbarrier complete_tx); once the compute warps
// signal done[s] it bulk-stores the results and refills the stage.
//
// Compute warp w holds tile-input cells [w(32V-2KX), w(32V-2KX)+32V), V per lane
// in registers; every step fetches the two inter-lane neighbours with shuffles.
// Every KX steps the warps trade KX-deep ghost zones through shared memory
// (kind 3: KX = 8, kind 4: KX = 16) -- PAPER.md:73's ghost exchange between
// neighbouring segments, at depth KX, between warps: after KX steps a warp's KX
// outermost cells on an inner side are stale and are refreshed from the
// neighbour warp's first/last KX owned cells (lane 0 / lane 31 registers; one
// named barrier per exchange, slots double-buffered by parity).  Only the CTA's
// two outer sides keep the T-deep trapezoid, so the redundant work is
// (2T + 2KX(NW-1))/(NW 32V).  V odd makes the 64-bit shared accesses of a
// half-warp hit 16 distinct bank pairs.
//
// Guarded variants (OPS 4, 3; stencil.cuh): every compute warp checks the input
// cells of its span (GuardAcc, 5 integer instructions per cell and tile) and the
// verdicts are AND-reduced in the first barrier the compute warps pass anyway; a tile
// that fails is redone -- by every warp, the decision is CTA-uniform -- with the
// literal 5-op sequence.  (Scanning the stages in the idle producer warp instead cost
// 5 % at C4: it loads one SM sub-partition unevenly.)

// The steps of a tile.  The first barrier among the compute warps (the first ghost
// exchange, or for T <= KX a barrier after the steps) orders every warp's span load
// before any warp's in-place write-back; with GUARD it also AND-reduces `ok` and the
// function returns false on every warp if some cell failed (nothing was written back:
// the stage still holds the tile's input).
template <int V, int NW, int KX, int OPS, bool GUARD>
__device__ __forceinline__ bool tile_steps(double (&u)[V], int T, double r, double scale, double *xbuf,
                                           int warp, int lane, bool ok) {
    int dn = 0;
    for (int e = 0;; ++e) {
        const int Ks = (T - dn) < KX ? (T - dn) : KX;
        // (full unrolling pays for the 1-op form only: the 3/4-op sub-period
        // code would outgrow the instruction cache)
        if (OPS == 1 && Ks == KX)
            warp_steps_fixed<V, OPS, KX>(u, r);
        else
            warp_steps<V, OPS>(u, Ks, r);  // (scaled forms: rescale below, once per pass)
        dn += Ks;
        if (dn >= T) {
            if (e == 0) {  // no exchange happened: the load-before-write-back barrier
                if constexpr (GUARD) {
                    if (!__shfl_sync(0xffffffffu, (int)bar1_and<NW * 32>(ok), 0)) return false;
                } else {
                    asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
                }
            }
            break;
        }
        double *X = xbuf + (size_t)(e & 1) * (NW * 2 * KX);
        if (lane == 0 && warp > 0) {
#pragma unroll
            for (int i = 0; i < KX; ++i) X[(warp * 2 + 0) * KX + i] = u[KX + i];
        }
        if (lane == 31 && warp < NW - 1) {
#pragma unroll
            for (int i = 0; i < KX; ++i) X[(warp * 2 + 1) * KX + i] = u[V - 2 * KX + i];
        }
        if (GUARD && e == 0) {
            // (the reduction is CTA-uniform; the broadcast lets ptxas prove it warp-uniform,
            // or the shuffles of the step loops become WARPSYNC-collective sequences)
            if (!__shfl_sync(0xffffffffu, (int)bar1_and<NW * 32>(ok), 0)) return false;
        } else {
            asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        }
        if (lane == 0 && warp > 0) {
#pragma unroll
            for (int i = 0; i < KX; ++i) u[i] = X[((warp - 1) * 2 + 1) * KX + i];
        }
        if (lane == 31 && warp < NW - 1) {
#pragma unroll
            for (int i = 0; i < KX; ++i) u[V - KX + i] = X[((warp + 1) * 2 + 0) * KX + i];
        }
    }
    if constexpr (ops_scaled(OPS)) {
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = __dmul_rn(u[j], scale);
    }
    return true;
}

// In-place write-back of a warp's owned cells (inner sides exclude the KX ghost zone,
// the CTA's outer sides the T-deep one).
template <int V, int NW, int KX>
__device__ __forceinline__ void write_back(const double (&u)[V], double *st, int base, int T, int warp, int lane) {
    const int lo = warp == 0 ? T : KX;
    const int hi = warp == NW - 1 ? 32 * V - T : 32 * V - KX;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int p = lane * V + j;
        if (p >= lo && p < hi) st[base + j] = u[j];
    }
}

// The guard's fallback (rare): a tile with the literal 5-op sequence.  Out of line, so
// its registers do not add to the hot path's.  (Measured: an inline copy of the tile loop
// for the rest of the pass after a failing tile instead cost 2.5 % -- the code size.)
template <int V, int NW, int KX>
__device__ __noinline__ void tile_literal(double *st, int base, int T, double r, double *xbuf, int warp, int lane) {
    double u[V];
#pragma unroll
    for (int j = 0; j < V; ++j) u[j] = st[base + j];
    tile_steps<V, NW, KX, 5, false>(u, T, r, 1.0, xbuf, warp, lane, true);
    write_back<V, NW, KX>(u, st, base, T, warp, lane);
}

// The compute warps' tile loop (OPS, coefficient r; fast mode's fallback for a pass whose scaled
// state could overflow runs it with OPS 3 and r).  Inlined at both call sites as disjoint
// branches: a call (out of line) would constrain the hot loop's registers (-2 %).
template <int V, int NW, int S, int KX, int OPS, bool GUARD>
__device__ __forceinline__ void compute_loop_rr(uint64_t *full, uint64_t *done, double *stages,
                                                uint32_t stage_doubles, int64_t out_lo, int64_t W, int T, double r,
                                                double scale, Guard guard, int64_t ntiles, double *xbuf, int warp,
                                                int lane) {
    const int SW = 32 * V - 2 * KX;
    int k = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int s = k % S;
        double *st = stages + (size_t)s * stage_doubles;
        const int64_t x0 = out_lo + tile * W;
        mbar_wait_sleep(&full[s], (uint32_t)((k / S) & 1));
        const int base = (int)((x0 - T) & 1) + warp * SW + lane * V;
        HCHECK(base >= 0 && base + V <= (int)stage_doubles);
        double u[V];
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = st[base + j];
        bool ok = true;
        if constexpr (GUARD) {
            GuardAcc acc;
#pragma unroll
            for (int j = 0; j < V; ++j) acc.add(u[j]);
            ok = acc.ok(guard);
        }
        if (tile_steps<V, NW, KX, OPS, GUARD>(u, T, r, scale, xbuf, warp, lane, ok))
            write_back<V, NW, KX>(u, st, base, T, warp, lane);
        else
            tile_literal<V, NW, KX>(st, base, T, r, xbuf, warp, lane);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[s]);
    }
}

// The producer warp of a pass kernel: for the CTA's tiles i = 0 .. geo.count()-1 (geo.span(i):
// output [x0, x1), 16-byte-aligned load window [ld_lo, ld_hi)), keep S TMA loads in flight,
// and once the compute warps release a stage store its output (bulk, plus the scalar
// leftovers: an odd first/last cell and the periodic self-halo of a single-slab ring).
template <int S, int NW, int KX, class Geo>
__device__ __forceinline__ void producer_loop(const Geo &geo, uint64_t *full, uint64_t *done, double *stages,
                                              uint32_t stage_doubles, const double *__restrict__ A,
                                              double *__restrict__ B, int64_t n, int wrapT, int halo, int feed_doubles,
                                              int lane) {
    const uint64_t pol_in = policy_evict_first();
    const int64_t count = geo.count();
    auto issue_load = [&](int64_t i, int s) {
        int64_t x0, x1, ld_lo, ld_hi;
        geo.span(i, &x0, &x1, &ld_lo, &ld_hi);
        const uint32_t bytes = (uint32_t)((ld_hi - ld_lo) * 8);
        HCHECK(bytes <= stage_doubles * 8u);                             // the stage holds the tile input
        HCHECK(ld_lo >= -(int64_t)halo - 1 && ld_hi <= n + halo + 1);  // within the padded slab
        HCHECK((128 + (size_t)S * stage_doubles * 8 + (size_t)2 * NW * 2 * KX * 8 + (size_t)feed_doubles * 8) <=
               dynamic_smem_bytes());
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(stages + (size_t)s * stage_doubles, A + ld_lo, bytes, &full[s], pol_in);
    };
    HCHECK(wrapT <= n && wrapT <= 128);  // (wrapT: the pad fill, <= T_MAX)
    if (lane == 0)
        for (int i = 0; i < S && i < count; ++i) issue_load(i, i);
    for (int64_t i = 0; i < count; ++i) {
        const int s = (int)(i % S);
        double *st = stages + (size_t)s * stage_doubles;
        int64_t x0, x1, ld_lo, ld_hi;
        geo.span(i, &x0, &x1, &ld_lo, &ld_hi);
        mbar_wait_backoff(&done[s], (uint32_t)((i / S) & 1));
        if (lane == 0 && (x0 & 1)) B[x0] = st[x0 - ld_lo];
        if (lane == 1 && (x1 & 1) && x1 - 1 >= x0) B[x1 - 1] = st[x1 - 1 - ld_lo];
        for (int j = lane; j < wrapT; j += 32) {
            if (j >= x0 && j < x1) B[n + j] = st[j - ld_lo];
            const int64_t c = n - wrapT + j;
            if (c >= x0 && c < x1) B[j - wrapT] = st[c - ld_lo];
        }
        __syncwarp();
        if (lane == 0) {
            const int64_t a = x0 + (x0 & 1);
            const int64_t b = x1 - (x1 & 1);
            if (b > a) bulk_s2g(B + a, st + (a - ld_lo), (uint32_t)((b - a) * 8));
            bulk_commit();
            if (i + S < count) {
                bulk_wait_read<0>();  // the tile's bytes have left the stage
                fence_proxy_async();
                issue_load(i + S, s);
            }
        }
        __syncwarp();
    }
    if (lane == 0) bulk_wait<0>();
}

// k2p_pass's tiles: round robin over the CTAs, both T-deep margins loaded
struct RoundRobinTiles {
    int64_t out_lo, out_hi, W, ntiles;
    int T;
    __device__ int64_t count() const {
        return ntiles > (int64_t)blockIdx.x ? (ntiles - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
    }
    __device__ void span(int64_t i, int64_t *x0, int64_t *x1, int64_t *ld_lo, int64_t *ld_hi) const {
        const int64_t tile = (int64_t)blockIdx.x + i * gridDim.x;
        *x0 = out_lo + tile * W;
        *x1 = min(*x0 + W, out_hi);
        const int64_t lo = *x0 - T;
        *ld_lo = lo - (lo & 1);
        *ld_hi = *x1 + T + ((*x1 + T) & 1);
    }
};

// Register target: the occupancy choose_geom plans for (2 CTAs/SM; 4 for V <= 17 tiles).
// Without it ptxas sizes the kernel for the guard's out-of-line fallback as well.
template <int V, int NW, int S, int OPS, int KX>
__global__ void __launch_bounds__((NW + 1) * 32, V <= 17 ? 4 : 2)
k2p_pass(const double *__restrict__ A, double *__restrict__ B, int64_t n, int T, int64_t out_lo,
         int64_t out_hi, int wrapT, double r, double scale, int64_t ntiles, uint32_t stage_doubles,
         Guard guard, FastRange fr) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);  // TMA landed
    uint64_t *done = full + S;                                 // compute warps finished
    double *stages = reinterpret_cast<double *>(smem_raw + 128);
    constexpr bool GUARD = ops_guarded(OPS);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
    const int64_t W = (int64_t)NW * 32 * V - 2 * KX * (NW - 1) - 2 * T;  // output cells per tile
    double *xbuf = stages + (size_t)S * stage_doubles;  // [2 parities][NW][2 sides][KX]

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NW) {  // ---------------- producer warp
        HCHECK(out_lo >= 0 && out_hi <= n);
        const RoundRobinTiles geo{out_lo, out_hi, W, ntiles, T};
        producer_loop<S, NW, KX>(geo, full, done, stages, stage_doubles, A, B, n, wrapT, T, 0, lane);
        return;
    }

    // ---------------- compute warps
    // scaled fast forms whose state could overflow run the whole pass in the 3-op form (no
    // branch inside the hot loop); the decision is CTA-uniform, broadcast so that ptxas sees
    // it warp-uniform
    if constexpr (ops_scaled(OPS)) {
        if (!__shfl_sync(0xffffffffu, (int)scaled_in_range(fr), 0)) {
            compute_loop_rr<V, NW, S, KX, 3, false>(full, done, stages, stage_doubles, out_lo, W, T, fr.r, 1.0, guard,
                                                    ntiles, xbuf, warp, lane);
            return;
        }
    }
    compute_loop_rr<V, NW, S, KX, OPS, GUARD>(full, done, stages, stage_doubles, out_lo, W, T, r, scale, guard, ntiles,
                                              xbuf, warp, lane);
}

// ------------------------------------------------------------------ K2f: feed tiles
//
// k2f_pass: K2 with each CTA walking a contiguous STRIP of the output, tile after tile,
// where every tile but the strip's first is fed its left boundary: the previous tile's last
// warp records, at every step t, the time-t value of the cell just left of the next tile
// (one column, shared memory), and the next tile's warp 0 lane 0 takes its left neighbour
// at step t from that record instead of computing a T-deep left halo.  So only the right
// side keeps a shrinking margin: T^2/2 wasted cell-steps per tile instead of 2 T^2 (K2's
// two trapezoids), and a tile's output grows from SPAN - 2T to SPAN - T cells.  (A parallel-
// ogram tiling: each tile's output is its window shifted left by T at the end of the pass.)
// T is a template parameter (the recorded column's lane and register are compile-time);
// other T, tail passes and other geometries run k2p_pass.
//
// Exactness guard: the fed values of a tile depend on time-0 cells of the previous tile's
// window (the cone of the recorded column, < T cells back), so a tile takes the contracted
// form only if its own cells AND the previous tile's cells passed the guard.
template <int V, int OPS, int LS, int JS>
__device__ __forceinline__ void warp_step_fd(const double (&u)[V], double (&v)[V], double r, int t, const double *fin,
                                             double *fout, bool rd, bool wr, int lane) {
    if (wr && lane == LS) fout[t] = u[JS];  // the time-t value of the next tile's left neighbour
    double L = __shfl_up_sync(0xffffffffu, u[V - 1], 1);
    const double R = __shfl_down_sync(0xffffffffu, u[0], 1);
    if (rd && lane == 0) L = fin[t];
#pragma unroll
    for (int j = 1; j < V - 1; ++j) v[j] = eq2<OPS>(u[j - 1], u[j], u[j + 1], r);
    v[0] = eq2<OPS>(L, u[0], u[1], r);
    v[V - 1] = eq2<OPS>(u[V - 2], u[V - 1], R, r);
}

template <int V, int OPS, int LS, int JS, int N>
__device__ __forceinline__ void warp_steps_fd_fixed(double (&u)[V], double r, int t0, const double *fin,
                                                    double *fout, bool rd, bool wr, int lane) {
    double v[V];
#pragma unroll
    for (int s = 0; s < N; s += 2) {
        warp_step_fd<V, OPS, LS, JS>(u, v, r, t0 + s, fin, fout, rd, wr, lane);
        warp_step_fd<V, OPS, LS, JS>(v, u, r, t0 + s + 1, fin, fout, rd, wr, lane);
    }
}

template <int V, int OPS, int LS, int JS>
__device__ __forceinline__ void warp_steps_fd(double (&u)[V], int K, double r, int t0, const double *fin,
                                              double *fout, bool rd, bool wr, int lane) {
    double v[V];
    int s = 0;
    for (; s + 2 <= K; s += 2) {
        warp_step_fd<V, OPS, LS, JS>(u, v, r, t0 + s, fin, fout, rd, wr, lane);
        warp_step_fd<V, OPS, LS, JS>(v, u, r, t0 + s + 1, fin, fout, rd, wr, lane);
    }
    if (s < K) {
        warp_step_fd<V, OPS, LS, JS>(u, v, r, t0 + s, fin, fout, rd, wr, lane);
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = v[j];
    }
}

// The TT steps of a tile (tile_steps with the feed hooks).  prev_ok: the previous tile's
// guard verdict (CTA-uniform); own_ok returns this tile's (for the next).
template <int V, int NW, int KX, int OPS, bool GUARD, int TT>
__device__ __forceinline__ bool tile_steps_fd(double (&u)[V], double r, double scale, double *xbuf,
                                              const double *fin, double *fout, bool rd, int warp, int lane,
                                              bool ok, bool prev_ok, bool &own_ok) {
    constexpr int POS = 32 * V - TT - 1;  // the recorded column in the last warp's span
    constexpr int LS = POS / V, JS = POS % V;
    static_assert(TT > KX && TT >= 2 * KX, "feed records must be ordered by the exchange barriers");
    const bool wr = warp == NW - 1;
    own_ok = true;
    int dn = 0;
    for (int e = 0;; ++e) {
        const int Ks = (TT - dn) < KX ? (TT - dn) : KX;
        if (OPS == 1 && Ks == KX)
            warp_steps_fd_fixed<V, OPS, LS, JS, KX>(u, r, dn, fin, fout, rd, wr, lane);
        else
            warp_steps_fd<V, OPS, LS, JS>(u, Ks, r, dn, fin, fout, rd, wr, lane);
        dn += Ks;
        if (dn >= TT) break;  // (TT > KX: the barrier of exchange 0 ordered every span load before)
        double *X = xbuf + (size_t)(e & 1) * (NW * 2 * KX);
        if (lane == 0 && warp > 0) {
#pragma unroll
            for (int i = 0; i < KX; ++i) X[(warp * 2 + 0) * KX + i] = u[KX + i];
        }
        if (lane == 31 && warp < NW - 1) {
#pragma unroll
            for (int i = 0; i < KX; ++i) X[(warp * 2 + 1) * KX + i] = u[V - 2 * KX + i];
        }
        if (GUARD && e == 0) {
            own_ok = __shfl_sync(0xffffffffu, (int)bar1_and<NW * 32>(ok), 0) != 0;
            if (!(own_ok && prev_ok)) return false;
        } else {
            asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
        }
        if (lane == 0 && warp > 0) {
#pragma unroll
            for (int i = 0; i < KX; ++i) u[i] = X[((warp - 1) * 2 + 1) * KX + i];
        }
        if (lane == 31 && warp < NW - 1) {
#pragma unroll
            for (int i = 0; i < KX; ++i) u[V - KX + i] = X[((warp + 1) * 2 + 0) * KX + i];
        }
    }
    if constexpr (ops_scaled(OPS)) {
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = __dmul_rn(u[j], scale);
    }
    return true;
}

// write-back of a feed tile: warp 0 owns from position 0 when fed (else T), the last warp up
// to 32V - TT (the right margin), inner sides exclude the KX ghost zones
template <int V, int NW, int KX, int TT>
__device__ __forceinline__ void write_back_fd(const double (&u)[V], double *st, int base, bool fed, int warp,
                                              int lane) {
    const int lo = warp == 0 ? (fed ? 0 : TT) : KX;
    const int hi = warp == NW - 1 ? 32 * V - TT : 32 * V - KX;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int p = lane * V + j;
        if (p >= lo && p < hi) st[base + j] = u[j];
    }
}

template <int V, int NW, int KX, int TT>
__device__ __noinline__ void tile_literal_fd(double *st, int base, double r, double *xbuf, const double *fin,
                                             double *fout, bool fed, int warp, int lane) {
    double u[V];
#pragma unroll
    for (int j = 0; j < V; ++j) u[j] = st[base + j];
    bool dummy;
    tile_steps_fd<V, NW, KX, 5, false, TT>(u, r, 1.0, xbuf, fin, fout, fed, warp, lane, true, true, dummy);
    write_back_fd<V, NW, KX, TT>(u, st, base, fed, warp, lane);
}

// A CTA's strip [S0, S1) of the output and its tiles: the first with both T-deep margins
// (window [x0 - TT, x1 + TT)), the rest fed on the left (window [x0, x1 + TT)).
struct FdStrip {
    int64_t S0 = 0, S1 = 0, W = 0, Ws = 0;
    int64_t ntile = 0;
    __device__ void tile(int64_t i, int64_t *x0, int64_t *x1, int64_t *win_lo) const {
        *x0 = i == 0 ? S0 : S0 + W + (i - 1) * Ws;
        const int64_t e = *x0 + (i == 0 ? W : Ws);
        *x1 = e < S1 ? e : S1;
        *win_lo = i == 0 ? *x0 - (Ws - W) : *x0;  // the first tile has a T-deep left margin (Ws - W = T)
    }
};

template <int V, int NW, int KX, int TT>
__device__ __forceinline__ FdStrip fd_strip(int64_t out_lo, int64_t out_hi) {
    constexpr int64_t SPAN = (int64_t)NW * 32 * V - 2 * KX * (NW - 1);
    FdStrip f;
    f.W = SPAN - 2 * TT;
    f.Ws = SPAN - TT;
    const int64_t total = out_hi - out_lo;
    const int64_t L = (total + gridDim.x - 1) / gridDim.x;
    f.S0 = out_lo + (int64_t)blockIdx.x * L;
    f.S1 = f.S0 + L < out_hi ? f.S0 + L : out_hi;
    if (f.S0 >= f.S1) return f;
    const int64_t len = f.S1 - f.S0;
    f.ntile = len <= f.W ? 1 : 1 + (len - f.W + f.Ws - 1) / f.Ws;
    return f;
}

// k2f_pass's tiles for the producer: the strip's, with their 16-byte-aligned load windows
template <int TT>
struct FdTilesT {
    FdStrip f;
    __device__ int64_t count() const { return f.ntile; }
    __device__ void span(int64_t i, int64_t *x0, int64_t *x1, int64_t *ld_lo, int64_t *ld_hi) const {
        int64_t wl;
        f.tile(i, x0, x1, &wl);
        *ld_lo = wl - (wl & 1);
        *ld_hi = *x1 + TT + ((*x1 + TT) & 1);
    }
};

// The compute warps' strip loop (OPS, coefficient r); also fast mode's 3-op fallback.
template <int V, int NW, int S, int KX, int OPS, bool GUARD, int TT>
__device__ __forceinline__ void compute_loop_fd(uint64_t *full, uint64_t *done, double *stages,
                                                uint32_t stage_doubles, const FdStrip &f, double r, double scale,
                                                Guard guard, double *xbuf, double *feed, int warp, int lane) {
    const int SW = 32 * V - 2 * KX;
    bool prev_ok = true;
    for (int64_t i = 0; i < f.ntile; ++i) {
        const int s = (int)(i % S);
        double *st = stages + (size_t)s * stage_doubles;
        int64_t x0, x1, wl;
        f.tile(i, &x0, &x1, &wl);
        const bool fed = i > 0;
        mbar_wait_sleep(&full[s], (uint32_t)((i / S) & 1));
        const int base = (int)(wl & 1) + warp * SW + lane * V;
        HCHECK(base >= 0 && base + V <= (int)stage_doubles);
        double u[V];
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = st[base + j];
        bool ok = true;
        if constexpr (GUARD) {
            GuardAcc acc;
#pragma unroll
            for (int j = 0; j < V; ++j) acc.add(u[j]);
            ok = acc.ok(guard);
        }
        const double *fin = feed + (size_t)((i + 1) & 1) * TT;  // written by tile i - 1
        double *fout = feed + (size_t)(i & 1) * TT;
        bool own_ok = true;
        if (tile_steps_fd<V, NW, KX, OPS, GUARD, TT>(u, r, scale, xbuf, fin, fout, fed, warp, lane, ok, prev_ok,
                                                     own_ok))
            write_back_fd<V, NW, KX, TT>(u, st, base, fed, warp, lane);
        else
            tile_literal_fd<V, NW, KX, TT>(st, base, r, xbuf, fin, fout, fed, warp, lane);
        prev_ok = own_ok;
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[s]);
    }
}

template <int V, int NW, int S, int OPS, int KX, int TT>
__global__ void __launch_bounds__((NW + 1) * 32, 2)
k2f_pass(const double *__restrict__ A, double *__restrict__ B, int64_t n, int T, int64_t out_lo, int64_t out_hi,
         int wrapT, double r, double scale, int64_t ntiles, uint32_t stage_doubles, Guard guard, FastRange fr) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem_raw);
    uint64_t *done = full + S;
    double *stages = reinterpret_cast<double *>(smem_raw + 128);
    constexpr bool GUARD = ops_guarded(OPS);
    (void)T;
    (void)ntiles;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
    double *xbuf = stages + (size_t)S * stage_doubles;  // [2 parities][NW][2 sides][KX]
    double *feed = xbuf + (size_t)2 * NW * 2 * KX;      // [2 tile parities][TT]
    const FdStrip f = fd_strip<V, NW, KX, TT>(out_lo, out_hi);

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NW) {  // ---------------- producer warp: the strip's tiles in order
        HCHECK(out_lo >= 0 && out_hi <= n);
        producer_loop<S, NW, KX>(FdTilesT<TT>{f}, full, done, stages, stage_doubles, A, B, n, wrapT, TT, 2 * TT, lane);
        return;
    }

    // ---------------- compute warps
    if constexpr (ops_scaled(OPS)) {
        if (!__shfl_sync(0xffffffffu, (int)scaled_in_range(fr), 0)) {
            compute_loop_fd<V, NW, S, KX, 3, false, TT>(full, done, stages, stage_doubles, f, fr.r, 1.0, guard, xbuf,
                                                        feed, warp, lane);
            return;
        }
    }
    compute_loop_fd<V, NW, S, KX, OPS, GUARD, TT>(full, done, stages, stage_doubles, f, r, scale, guard, xbuf, feed,
                                                  warp, lane);
}

size_t PassGeom::smem_bytes(int T) const {
    const int64_t in_cells = tile_out(T) + 2 * T + 2;
    const int64_t stage = (in_cells + 15) / 16 * 16;
    const size_t xch = (size_t)2 * NW * 2 * kx_of(kind) * sizeof(double);
    const size_t feed = (size_t)2 * 128 * sizeof(double);  // k2f_pass's boundary records (T <= 128)
    return 128 + (size_t)S * (size_t)stage * sizeof(double) + xch + feed;
}

namespace {

using PassFn = void (*)(const double *, double *, int64_t, int, int64_t, int64_t, int, double, double,
                        int64_t, uint32_t, Guard, FastRange);

// (V, NW, S) instantiated for kinds 3 and 4 and all four arithmetic variants: the
// two defaults of choose_geom (51,4,2) and (17,4,3) plus the tuning points of the
// V sweeps.
#define HEAT1D_GEOMS_X(X) X(17, 4, 3) X(25, 4, 3) X(33, 4, 2) X(49, 4, 2) X(51, 4, 2)

template <int V, int NW, int S, int KX>
PassFn pass_fn_x(int ops) {
    if constexpr (V < 2 * KX) {  // the exchanged KX-cell edges must lie inside one lane
        (void)ops;
        return nullptr;
    } else {
        switch (ops) {
            case 4: return &k2p_pass<V, NW, S, 4, KX>;
            case 3: return &k2p_pass<V, NW, S, 3, KX>;
            case 2: return &k2p_pass<V, NW, S, 2, KX>;
            case 1: return &k2p_pass<V, NW, S, 1, KX>;
            default: return nullptr;
        }
    }
}

// feed tiles (k2f_pass): the default geometry at T = 64 / 96 / 128 (-DHEAT1D_NOFEED: never; A/B builds)
PassFn lookup_feed(const PassGeom &g, int ops, int T) {
#ifdef HEAT1D_NOFEED
    (void)g; (void)ops; (void)T;
    return nullptr;
#else
    if (!(g.V == 51 && g.NW == 4 && g.S == 2 && g.kind == 4)) return nullptr;
#define F(tt)                                                   \
    if (T == tt) switch (ops) {                                 \
            case 4: return &k2f_pass<51, 4, 2, 4, 16, tt>;      \
            case 3: return &k2f_pass<51, 4, 2, 3, 16, tt>;      \
            case 2: return &k2f_pass<51, 4, 2, 2, 16, tt>;      \
            case 1: return &k2f_pass<51, 4, 2, 1, 16, tt>;      \
            default: return nullptr;                            \
        }
    F(64) F(96) F(128)
#undef F
    return nullptr;
#endif
}

PassFn lookup_pass(int V, int NW, int S, int ops, int kind) {
    if (kind != 3 && kind != 4) return nullptr;
#define X(v, nw, s) \
    if (V == v && NW == nw && S == s) return kind == 3 ? pass_fn_x<v, nw, s, 8>(ops) : pass_fn_x<v, nw, s, 16>(ops);
    HEAT1D_GEOMS_X(X)
#undef X
    return nullptr;
}

}  // namespace

bool pass_supported(const PassGeom &g, int ops) { return lookup_pass(g.V, g.NW, g.S, ops, g.kind) != nullptr; }

bool pass_uses_feed(const PassGeom &g, int ops, int T) { return lookup_feed(g, ops, T) != nullptr; }

PassGeom choose_geom(int64_t n_out, int T, int num_sms, int ops) {
    // Default (profiles/r01_sweep_kx.jsonl): CTA tiles of 4 compute warps x
    // V = 51 cells per lane trading 16-deep ghosts every 16 steps (kind 4), plus a TMA
    // producer warp, 2 stages, 2 CTAs per SM.  V = 45..55 swept for all four arithmetic
    // forms: 51 is best or within 0.3 % of best for each (V >= 53 spills the 1-/3-op forms
    // to one CTA per SM).  Rings too small to give every CTA a tile use 4-warp V=17 tiles
    // exchanging every 8 steps.
    (void)ops;
    PassGeom g{51, 4, 2, 2, 4};
    if (n_out < (int64_t)num_sms * g.ctas_per_sm * g.tile_out(T)) g = PassGeom{17, 4, 3, 4, 3};
    return g;
}

cudaError_t launch_pass(const PassGeom &g, int ops, const double *A, double *B, int64_t n, int T,
                        int64_t out_lo, int64_t out_hi, int wrapT, double q, double scale, Guard guard,
                        const FastRange &fr, int num_sms, cudaStream_t st, int *grid_out) {
    PassFn fn = lookup_pass(g.V, g.NW, g.S, ops, g.kind);
    if (!fn) return cudaErrorInvalidConfiguration;
    if (PassFn ffn = lookup_feed(g, ops, T)) fn = ffn;
    if (out_hi <= out_lo) {
        if (grid_out) *grid_out = 0;
        return cudaSuccess;
    }
    const int64_t W = g.tile_out(T);
    const int kx = kx_of(g.kind);
    // the outer warps' T-deep trapezoid must stay inside their span, and the exchanged
    // KX-cell edges inside one lane
    if (W <= 0 || T > 32 * g.V - kx || g.V < 2 * kx) return cudaErrorInvalidValue;
    const int64_t units = (out_hi - out_lo + W - 1) / W;
    const size_t smem = g.smem_bytes(T);
    const int64_t in_cells = W + 2 * T + 2;
    const uint32_t stage_doubles = (uint32_t)((in_cells + 15) / 16 * 16);
    // Raise the dynamic shared-memory limit once per instantiation (max over T).
    {
        static std::mutex mu;
        static PassFn done_fn[256] = {nullptr};
        std::lock_guard<std::mutex> lk(mu);
        bool done = false;
        int slot = -1;
        for (int i = 0; i < 256; ++i) {
            if (done_fn[i] == fn) { done = true; break; }
            if (done_fn[i] == nullptr) { slot = i; break; }
        }
        if (!done) {
            const size_t want = g.smem_bytes(1);  // the largest tile (T=1)
            cudaError_t e = cudaFuncSetAttribute((const void *)fn,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
            if (e != cudaSuccess) return e;
            if (slot >= 0) done_fn[slot] = fn;
        }
    }
    // Persistent grid: never more CTAs than can be co-resident (static round-robin
    // assignment assumes a single wave).
    int occ = 0;
    const int threads = (g.NW + 1) * 32;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)fn, threads, smem) != cudaSuccess ||
        occ < 1)
        occ = 1;
    const int per_sm = g.ctas_per_sm < occ ? g.ctas_per_sm : occ;
    int64_t grid = (int64_t)num_sms * per_sm;
    if (grid > units) grid = units;  // (k2f_pass: strips of at least one first-tile width)
    if (grid_out) *grid_out = (int)grid;
    fn<<<(unsigned)grid, threads, smem, st>>>(A, B, n, T, out_lo, out_hi, wrapT, q, scale, units, stage_doubles,
                                             guard, fr);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K1
template <int OPS>
__global__ void __launch_bounds__(256) k1_naive(const double *__restrict__ A, double *__restrict__ B, int64_t n,
                                                double r) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t il = (i == 0) ? n - 1 : i - 1;  // periodic
        const int64_t ir = (i == n - 1) ? 0 : i + 1;
        B[i] = eq2<OPS>(A[il], A[i], A[ir], r);
    }
}

cudaError_t launch_naive(int ops, const double *A, double *B, int64_t n, double r, cudaStream_t st) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (ops == 5)
        k1_naive<5><<<(unsigned)blocks, 256, 0, st>>>(A, B, n, r);
    else if (ops == 3)
        k1_naive<3><<<(unsigned)blocks, 256, 0, st>>>(A, B, n, r);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K3
// Block 0: outputs [0,T) from A[-T, 2T); block 1: outputs [n-T, n) from A[n-2T, n+T).
// The 3T-cell window shrinks by one cell per side per step (light cone).
// Guarded variants (stencil.cuh) run the literal sequence if any window cell fails.
template <int OPS>
__device__ __forceinline__ int strip_steps(double (*w)[3 * 128], int T, double r) {
    const int len = 3 * T;
    int cur = 0;
    for (int s = 0; s < T; ++s) {
        const int lo = s + 1, hi = len - 1 - s;  // cells valid after step s+1
        for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
            w[cur ^ 1][i] = eq2<OPS>(w[cur][i - 1], w[cur][i], w[cur][i + 1], r);
        cur ^= 1;
        __syncthreads();
    }
    return cur;
}

// Returns the buffer holding the result; *scaled = whether it is in the scaled state.
template <int OPS>
__device__ __forceinline__ int strip_steps_guarded(double (*w)[3 * 128], int T, double r, Guard guard,
                                                   const FastRange &fr, bool *scaled) {
    *scaled = ops_scaled(OPS);
    if constexpr (ops_guarded(OPS)) {
        GuardAcc acc;
        for (int i = threadIdx.x; i < 3 * T; i += blockDim.x) acc.add(w[0][i]);
        if (!__syncthreads_and(acc.ok(guard))) return strip_steps<5>(w, T, r);
    }
    if constexpr (ops_scaled(OPS)) {
        if (!scaled_in_range(fr)) {
            *scaled = false;
            return strip_steps<3>(w, T, fr.r);
        }
    }
    return strip_steps<OPS>(w, T, r);
}

template <int OPS>
__global__ void __launch_bounds__(96) k3_edges(const double *__restrict__ A, double *__restrict__ B, int64_t n,
                                               int T, double r, double scale, Guard guard, FastRange fr) {
    __shared__ double w[2][3 * 128];
    const int64_t base = (blockIdx.x == 0) ? -(int64_t)T : n - 2 * (int64_t)T;
    const int len = 3 * T;
    HCHECK(T >= 1 && T <= 128 && n >= (int64_t)T);  // windows [-T, 2T), [n-2T, n+T) inside the pads
    for (int i = threadIdx.x; i < len; i += blockDim.x) w[0][i] = A[base + i];
    __syncthreads();
    bool scaled;
    const int cur = strip_steps_guarded<OPS>(w, T, r, guard, fr, &scaled);
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
        double x = w[cur][T + i];
        if (scaled) x = __dmul_rn(x, scale);
        B[base + T + i] = x;
    }
}

cudaError_t launch_edges(int ops, const double *A, double *B, int64_t n, int T, double q, double scale,
                         Guard guard, const FastRange &fr, cudaStream_t st) {
    if (T < 1 || T > 128) return cudaErrorInvalidValue;
    switch (ops) {
        case 4: k3_edges<4><<<2, 96, 0, st>>>(A, B, n, T, q, scale, guard, fr); break;
        case 3: k3_edges<3><<<2, 96, 0, st>>>(A, B, n, T, q, scale, guard, fr); break;
        case 2: k3_edges<2><<<2, 96, 0, st>>>(A, B, n, T, q, scale, guard, fr); break;
        case 1: k3_edges<1><<<2, 96, 0, st>>>(A, B, n, T, q, scale, guard, fr); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K3p
// K3 fused with the halo exchange over peer memory (transport HEAT1D_TRANSPORT_P2P):
// block 0 waits until its left ghost pad of A holds exchange index g (system-scope
// acquire on the flag its left neighbour releases), advances the strip [0,T) T steps,
// writes it to B AND straight into the left neighbour's right pad of B (remote stores
// over NVLink, or plain stores for a slab on the same GPU), then releases the
// neighbour's flag with g+1; block 1 mirrors this for [n-T,n) and the right
// neighbour.  No NCCL call, host round trip or extra kernel sits between the edge
// update and the data's arrival at the neighbour (PAPER.md:73's ghost exchange).
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int OPS>
__global__ void __launch_bounds__(96) k3_edges_put(const double *__restrict__ A, double *__restrict__ B, int64_t n,
                                                   int T, double r, double scale, Guard guard, FastRange fr,
                                                   const unsigned *my_flags, unsigned g, double *put_left,
                                                   double *put_right, unsigned *flag_left, unsigned *flag_right) {
    __shared__ double w[2][3 * 128];
    const int side = blockIdx.x;  // 0: [0,T) <- left pad; 1: [n-T,n) <- right pad
    if (threadIdx.x == 0) {
        const unsigned *f = my_flags + side * 32;
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys_u32(f) < g + 1) {
            if (globaltimer_ns() - t0 > HEAT1D_WAIT_NS) __trap();
        }
    }
    __syncthreads();
    const int64_t base = (side == 0) ? -(int64_t)T : n - 2 * (int64_t)T;
    const int len = 3 * T;
    HCHECK(T >= 1 && T <= 128 && n >= 2 * (int64_t)T);
    for (int i = threadIdx.x; i < len; i += blockDim.x) w[0][i] = __ldcv(A + base + i);  // pads: peer-written
    __syncthreads();
    bool scaled;
    const int cur = strip_steps_guarded<OPS>(w, T, r, guard, fr, &scaled);
    double *put = side == 0 ? put_left : put_right;
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
        double x = w[cur][T + i];
        if (scaled) x = __dmul_rn(x, scale);
        B[base + T + i] = x;
        put[i] = x;
    }
    __syncthreads();  // every thread's put precedes thread 0's (cumulative) release
    if (threadIdx.x == 0) st_release_sys_u32(side == 0 ? flag_left : flag_right, g + 2);
}

cudaError_t launch_edges_put(int ops, const double *A, double *B, int64_t n, int T, double q, double scale,
                             Guard guard, const FastRange &fr, const unsigned *my_flags, unsigned g,
                             double *put_left, double *put_right, unsigned *flag_left, unsigned *flag_right,
                             cudaStream_t st) {
    if (T < 1 || T > 128 || n < 2 * (int64_t)T) return cudaErrorInvalidValue;
#define K3P(o) k3_edges_put<o><<<2, 96, 0, st>>>(A, B, n, T, q, scale, guard, fr, my_flags, g, put_left, put_right, flag_left, flag_right)
    switch (ops) {
        case 4: K3P(4); break;
        case 3: K3P(3); break;
        case 2: K3P(2); break;
        case 1: K3P(1); break;
        default: return cudaErrorInvalidValue;
    }
#undef K3P
    return cudaGetLastError();
}

// Start of a run (transport P2P): push this slab's current edge cells [0,T) and [n-T,n)
// into the neighbours' pads of the same buffer and release their flags with g+1 (the
// index the run's first pass waits for).  Also covers a new initial state and a run
// whose first pass is deeper than the previous run's tail pass.
__global__ void __launch_bounds__(128) k_push_edges(const double *__restrict__ A, int64_t n, int T, unsigned g,
                                                   double *put_left, double *put_right, unsigned *flag_left,
                                                   unsigned *flag_right) {
    const int side = blockIdx.x;
    const double *src = side == 0 ? A : A + n - T;
    double *dst = side == 0 ? put_left : put_right;
    for (int i = threadIdx.x; i < T; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    if (threadIdx.x == 0) st_release_sys_u32(side == 0 ? flag_left : flag_right, g + 1);
}

cudaError_t launch_push_edges(const double *A, int64_t n, int T, unsigned g, double *put_left, double *put_right,
                              unsigned *flag_left, unsigned *flag_right, cudaStream_t st) {
    if (T < 1 || n < T) return cudaErrorInvalidValue;
    k_push_edges<<<2, 128, 0, st>>>(A, n, T, g, put_left, put_right, flag_left, flag_right);
    return cudaGetLastError();
}

// Fault injection (tests): occupy the comm stream for `us` microseconds before the halo
// exchange of a pass (HEAT1D_COMM_DELAY_US); results must not change.
__global__ void k_delay(unsigned us) {
    const unsigned long long t0 = globaltimer_ns();
    while (globaltimer_ns() - t0 < 1000ull * us) __nanosleep(1000);
}

cudaError_t launch_delay(unsigned us, cudaStream_t st) {
    k_delay<<<1, 32, 0, st>>>(us);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K4
__global__ void k4_wrap_fill(double *A, int64_t n, int64_t pad) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < pad; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = j % n;
        A[n + j] = A[m];           // right pad: cells 0, 1, ...
        A[-1 - j] = A[n - 1 - m];  // left pad:  cells n-1, n-2, ...
    }
}

cudaError_t launch_wrap_fill(double *A, int64_t n, int64_t pad, cudaStream_t st) {
    k4_wrap_fill<<<1, 128, 0, st>>>(A, n, pad);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K5
// max |u| over a slab, as the bit pattern of a non-negative double (those order
// like unsigned integers; inf and NaN sort above every finite value).  Used once
// per initial state to check the fast mode's scaled-state range.
__global__ void __launch_bounds__(256) k5_absmax(const double *__restrict__ u, int64_t count,
                                                 unsigned long long *out) {
    unsigned long long m = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(u[i]) & 0x7fffffffffffffffull;
        m = b > m ? b : m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
        m = x > m ? x : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

cudaError_t launch_absmax(const double *u, int64_t count, unsigned long long *out, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k5_absmax<<<(unsigned)blocks, 256, 0, st>>>(u, count, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K0
__global__ void k0_uniform(double *u, int64_t count, int64_t first, uint64_t seed, double lo, double hi) {
    const double d = __dsub_rn(hi, lo);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        uint64_t z = seed + (uint64_t)(first + i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const double U = __dmul_rn((double)(z >> 11), 0x1.0p-53);
        u[i] = __dadd_rn(lo, __dmul_rn(d, U));
    }
}

cudaError_t launch_init_uniform(double *u, int64_t count, int64_t first, uint64_t seed, double lo, double hi,
                                cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    k0_uniform<<<(unsigned)blocks, 256, 0, st>>>(u, count, first, seed, lo, hi);
    return cudaGetLastError();
}

}  // namespace heat1d
