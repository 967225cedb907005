// resident.cu -- K6: register-resident ring for slabs that fit on chip.
//
// A ring of up to ~2 M cells (C1, C2, C5 of BASELINE.json) is latency-bound
// on B200 if every T steps costs a kernel launch.  K6 runs the WHOLE nt-step
// solve in one cooperative launch.  The slab is cut into Ns equal "spans";
// each span keeps its owned cells plus a T-deep halo on each side in
// registers (V cells per lane, the per-warp trapezoid of K2), advances T
// steps, publishes its first and last T owned cells to a global edge buffer
// and refreshes its halos from its two neighbour spans' edges -- the paper's
// ghost-zone exchange between segments at depth T, between warps.
//
// Synchronisation is pairwise, no grid-wide barrier: spans of V = 17 cells per
// lane (periods T <= 32) publish their edges with a release of a per-span flag;
// spans of V >= 25 (periods 32 < T <= 128) publish tagged words (below): no
// flag, no fence.  Edge buffers are double-buffered by period parity: a span
// writes period p+2 edges only after its neighbours published p+1, i.e. after
// they finished reading period p.
//
// Guarded variants (OPS 4, 3; stencil.cuh): at the start of every period a warp
// checks the cells of its span (owned + halos) and, if any fails, advances that
// period with the literal 5-op sequence (a warp-uniform branch).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "kernels.h"
#include "stencil.cuh"

namespace heat1d {

namespace {

__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// system scope: flags written by a peer GPU over NVLink (K6 across ranks)
__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// One step on the V cells of each lane; the neighbour cells L, R of the lane's
// outermost cells were fetched by the previous step (shuffles issued early, right
// after the two outer cells are computed, so their latency hides behind the rest).
template <int V, int OPS>
__device__ __forceinline__ void step_regs(const double (&u)[V], double (&v)[V], double &L, double &R, double r) {
    v[0] = eq2<OPS>(L, u[0], u[1], r);
    v[V - 1] = eq2<OPS>(u[V - 2], u[V - 1], R, r);
    L = __shfl_up_sync(0xffffffffu, v[V - 1], 1);
    R = __shfl_down_sync(0xffffffffu, v[0], 1);
#pragma unroll
    for (int j = 1; j < V - 1; ++j) v[j] = eq2<OPS>(u[j - 1], u[j], u[j + 1], r);
}

// Tp steps on u (v is scratch), result in u; scaled variants end with u *= r^Tp.
template <int V, int OPS>
__device__ __forceinline__ void steps_regs(double (&u)[V], double (&v)[V], int Tp, double r, double scale) {
    double L = __shfl_up_sync(0xffffffffu, u[V - 1], 1);
    double R = __shfl_down_sync(0xffffffffu, u[0], 1);
    int s = 0;
    for (; s + 2 <= Tp; s += 2) {
        step_regs<V, OPS>(u, v, L, R, r);
        step_regs<V, OPS>(v, u, L, R, r);
    }
    if (s < Tp) {
        step_regs<V, OPS>(u, v, L, R, r);
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = v[j];
    }
    if constexpr (ops_scaled(OPS)) {
#pragma unroll
        for (int j = 0; j < V; ++j) u[j] = __dmul_rn(u[j], scale);
    }
}

// The guard's fallback (rare): a period with the literal 5-op sequence on the span's
// row (which holds the period's input), out of line so that its registers do not add
// to the hot path's.
// (OPS = 3: fast mode's fallback when the scaled state could overflow, FastRange)
template <int V, int OPS = 5>
__device__ __noinline__ void period_literal(double *row, int Tp, double r, int lane) {
    double u[V], v[V];
#pragma unroll
    for (int j = 0; j < V; ++j) u[j] = row[lane * V + j];
    steps_regs<V, OPS>(u, v, Tp, r, 1.0);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < V; ++j) row[lane * V + j] = u[j];
    __syncwarp();
}

// A period of Tp steps of one span, guarded (stencil.cuh): `live` = the span's row
// positions holding ring cells (own + 2T; the rest of the 32V registers is slack).
// The row holds the same cells as u on entry.
template <int V, int OPS>
__device__ __forceinline__ void period_steps(double (&u)[V], double (&v)[V], double *row, int Tp, double r,
                                             double scale, Guard guard, int live, int lane, bool scaled,
                                             double r3) {
    if constexpr (ops_scaled(OPS)) {
        if (!scaled) {  // the scaled state could overflow: the contracted 3-op form (coefficient r3)
            period_literal<V, 3>(row, Tp, r3, lane);
#pragma unroll
            for (int j = 0; j < V; ++j) u[j] = row[lane * V + j];
            return;
        }
    }
    if constexpr (ops_guarded(OPS)) {
        GuardAcc acc;
#pragma unroll
        for (int j = 0; j < V; ++j)
            if (lane * V + j < live) acc.add(u[j]);
        if (!__all_sync(0xffffffffu, acc.ok(guard))) {
            period_literal<V>(row, Tp, r, lane);
#pragma unroll
            for (int j = 0; j < V; ++j) u[j] = row[lane * V + j];
            return;
        }
    }
    steps_regs<V, OPS>(u, v, Tp, r, scale);
}

// One span: its cells [start, start+own) of the ring, staged in `row`
// (positions 0..T-1 left halo, T..T+own-1 owned, then right halo).
struct Span {
    int64_t start;
    int own, id, left, right;
    double *row;
};

__device__ __forceinline__ Span make_span(int id, int Ns, int64_t n, double *row) {
    const int64_t base = n / Ns, rem = n % Ns;
    Span s;
    s.id = id;
    s.own = (int)(base + (id < rem ? 1 : 0));
    s.start = (int64_t)id * base + (id < rem ? id : rem);
    s.left = (id + Ns - 1) % Ns;
    s.right = (id + 1) % Ns;
    s.row = row;
    return s;
}

template <int V>
__device__ __forceinline__ void load_span(const Span &s, const double *__restrict__ A, int64_t n, int T,
                                          int lane) {
    const int span = s.own + 2 * T;
#pragma unroll
    for (int k = 0; k < V; ++k) {  // uniform trip count (no divergent loop before the shuffles)
        const int p = lane + 32 * k;
        double x = 0.0;
        if (p < span) {
            int64_t g = (s.start - T + p) % n;  // rings shorter than a halo wrap more than once
            if (g < 0) g += n;
            x = A[g];
        }
        s.row[p] = x;
    }
    __syncwarp();
}

template <int V>
__device__ __forceinline__ void row_to_regs(const double *row, double (&u)[V], int lane) {
#pragma unroll
    for (int j = 0; j < V; ++j) u[j] = row[lane * V + j];
}

template <int V>
__device__ __forceinline__ void regs_to_row(const double (&u)[V], double *row, int lane) {
    __syncwarp();
#pragma unroll
    for (int j = 0; j < V; ++j) row[lane * V + j] = u[j];
    __syncwarp();
}

// Tagged words (V >= 25: the spans' edges inside one GPU, and the mailboxes between ranks):
// an edge value travels as two 8-byte words (tag << 32) | half, stored by one st.v2.b64.
// Each naturally aligned 8-byte element of a vector access is single-copy atomic (PTX
// memory model; over NVLink as well -- NCCL's LL protocol rests on the same property), so a
// reader that finds the expected tag in both words holds both halves of that one write.
// Tags are unique per launch and period (spans: tbase + p, the host advances tbase past every
// launch; mailboxes: the global exchange index + 1), so a slot's stale content never matches;
// the reader writes nothing back and nobody fences: a slot is overwritten (two periods later)
// only after its writer computed from the reader's next edges, which the reader computed from
// the values it read (a data dependency orders its read before its next publish).
// SYS: system scope (a neighbour rank's mailbox over NVLink), else GPU scope.
template <bool SYS = false>
__device__ __forceinline__ void st_tagged(unsigned long long *p, double v, unsigned tag) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long t = (unsigned long long)tag << 32;
    if constexpr (SYS)
        asm volatile("st.relaxed.sys.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(t | (b & 0xffffffffull)),
                     "l"(t | (b >> 32))
                     : "memory");
    else
        asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(t | (b & 0xffffffffull)),
                     "l"(t | (b >> 32))
                     : "memory");
}
template <bool SYS = false>
__device__ __forceinline__ bool ld_tagged(const unsigned long long *p, unsigned tag, double *v) {
    unsigned long long w0, w1;
    if constexpr (SYS)
        asm volatile("ld.relaxed.sys.global.v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    *v = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
    return (unsigned)(w0 >> 32) == tag && (unsigned)(w1 >> 32) == tag;
}
// the tagged edge slots of span `id`, period parity `par`, side `side` (2 words per cell)
__device__ __forceinline__ unsigned long long *tagged_slot(double *edges, int id, unsigned par, int side, int T) {
    return reinterpret_cast<unsigned long long *>(edges) + (((size_t)id * 4 + par * 2 + side) * T) * 2;
}

// edges: [Ns][2 parities][2 sides][T]; publish this span's period-p edges
// (DF: tagged words, compiled into its own kernel instantiation; else a release flag per span)
template <bool DF = false>
__device__ __forceinline__ void publish(const Span &s, int T, unsigned p, double *edges, unsigned *flags,
                                        unsigned tbase, int lane) {
    if constexpr (DF) {
        unsigned long long *E0 = tagged_slot(edges, s.id, p & 1, 0, T), *E1 = tagged_slot(edges, s.id, p & 1, 1, T);
        for (int i = lane; i < T; i += 32) {
            st_tagged(E0 + 2 * i, s.row[T + i], tbase + p);
            st_tagged(E1 + 2 * i, s.row[s.own + i], tbase + p);
        }
    } else {
        double *E = edges + ((size_t)s.id * 4 + (p & 1) * 2) * T;
        for (int i = lane; i < T; i += 32) {
            E[i] = s.row[T + i];          // side 0: first T owned cells
            E[T + i] = s.row[s.own + i];  // side 1: last T owned cells
        }
        __syncwarp();  // orders the lanes' writes before lane 0's (cumulative) release
        if (lane == 0) st_release(flags + s.id, p + 1);
    }
}

// The slab's boundary spans trade halos with the neighbour RANKS through mailboxes
// (MboxArgs, kernels.h): span 0 writes its first T owned cells into the left rank's
// mailbox side 1, the last span its last T owned cells into the right rank's side 0,
// with remote (NVLink) stores and a system-scope release of the slot's flag; each rank
// reads its own mailbox.  Slots alternate with the global exchange index g (see
// launch_resident: indices never repeat across runs, and skip one at run boundaries).
__device__ __forceinline__ double *mbox_data(double *mb, int side, unsigned g) {  // 2 doubles per cell
    return mb + ((size_t)side * 2 + (g & 1)) * MBOX_TMAX * 2;
}
__device__ __forceinline__ unsigned long long *mbox_tagged(double *mb, int side, unsigned g) {
    return reinterpret_cast<unsigned long long *>(mbox_data(mb, side, g));
}
__device__ __forceinline__ unsigned *mbox_flag(double *mb, int side) {
    return reinterpret_cast<unsigned *>(reinterpret_cast<char *>(mb) + MBOX_FLAG_OFF) + side * 32;
}

// DF: tagged words straight into the neighbour rank's mailbox slot (tag g + 1), no flag, no
// fence; else the slot's values plus a system-scope release of its flag.
template <bool DF = false>
__device__ __forceinline__ void mbox_publish(const Span &s, int Ns, int T, unsigned g, const MboxArgs &mb, int lane) {
    if constexpr (DF) {
        if (s.id == 0) {
            unsigned long long *D = mbox_tagged(mb.left, 1, g);
            for (int i = lane; i < T; i += 32) st_tagged<true>(D + 2 * i, s.row[T + i], g + 1);
        }
        if (s.id == Ns - 1) {
            unsigned long long *D = mbox_tagged(mb.right, 0, g);
            for (int i = lane; i < T; i += 32) st_tagged<true>(D + 2 * i, s.row[s.own + i], g + 1);
        }
        return;
    }
    if (s.id == 0) {
        double *D = mbox_data(mb.left, 1, g);
        for (int i = lane; i < T; i += 32) D[i] = s.row[T + i];
        __syncwarp();
        if (lane == 0) st_release_sys(mbox_flag(mb.left, 1), g + 1);
    }
    if (s.id == Ns - 1) {
        double *D = mbox_data(mb.right, 0, g);
        for (int i = lane; i < T; i += 32) D[i] = s.row[s.own + i];
        __syncwarp();
        if (lane == 0) st_release_sys(mbox_flag(mb.right, 0), g + 1);
    }
}

// wait for the neighbours' period-p edges and write them into the halos; with mailboxes
// on, the slab's outer halos come from the neighbour ranks (exchange index g)
// initial: the exchange of the initial state (only the remote sides; the local halos
// were loaded from the slab).
// Halo refresh of a V >= 25 span, kept out of line: inlined into the period loop its 64-bit
// polls and pointers raised the matched kernels from 115 to 154 registers (and -25 %).
// Each side is a neighbour span's tagged edge on this GPU (gpu scope, tag tl / tr) or, with
// SYS, this rank's mailbox slot filled by a neighbour rank (system scope); null = that side's
// halo is already valid (the initial exchange of local sides).
template <bool SYS>
__device__ __noinline__ void refresh_df(double *row, int own, int T, const unsigned long long *L,
                                        const unsigned long long *R, bool lsys, bool rsys, unsigned tl, unsigned tr,
                                        int lane) {
    const unsigned long long t0 = SYS ? globaltimer_ns() : 0;
    for (int i0 = 0; i0 < T; i0 += 32) {
        const int i = i0 + lane;
        double lv = 0.0, rv = 0.0;
        bool ok;
        do {
            bool lok = true, rok = true;
            if (i < T) {
                if (L) lok = (SYS && lsys) ? ld_tagged<true>(L + 2 * i, tl, &lv) : ld_tagged<false>(L + 2 * i, tl, &lv);
                if (R) rok = (SYS && rsys) ? ld_tagged<true>(R + 2 * i, tr, &rv) : ld_tagged<false>(R + 2 * i, tr, &rv);
            }
            ok = lok && rok;
            if (SYS && globaltimer_ns() - t0 > HEAT1D_WAIT_NS) __trap();  // a neighbour rank is gone
        } while (!__all_sync(0xffffffffu, ok));
        if (i < T) {
            if (L) row[i] = lv;
            if (R) row[own + T + i] = rv;
        }
    }
    __syncwarp();
}

template <bool DF = false, bool SYS = false>
__device__ __forceinline__ void refresh(const Span &s, int T, unsigned p, double *edges,
                                        const unsigned *flags, int lane, int Ns, const MboxArgs &mb,
                                        unsigned g, unsigned tbase, bool initial = false) {
    const bool lrem = mb.on && s.id == 0, rrem = mb.on && s.id == Ns - 1;
    if constexpr (DF) {
        // left neighbour's side 1 and right neighbour's side 0, or this rank's mailbox
        const unsigned long long *L = lrem ? mbox_tagged(mb.self, 0, g) : tagged_slot(edges, s.left, p & 1, 1, T);
        const unsigned long long *R = rrem ? mbox_tagged(mb.self, 1, g) : tagged_slot(edges, s.right, p & 1, 0, T);
        refresh_df<SYS>(s.row, s.own, T, (lrem || !initial) ? L : nullptr, (rrem || !initial) ? R : nullptr, lrem,
                        rrem, lrem ? g + 1 : tbase + p, rrem ? g + 1 : tbase + p, lane);
        return;
    }
    if (lrem || rrem) {
        const bool doL = lrem || !initial, doR = rrem || !initial;
        const unsigned *Lf = lrem ? mbox_flag(mb.self, 0) : flags + s.left;
        const unsigned *Rf = rrem ? mbox_flag(mb.self, 1) : flags + s.right;
        const unsigned Lt = !doL ? 0u : lrem ? g + 1 : p + 1, Rt = !doR ? 0u : rrem ? g + 1 : p + 1;
        const unsigned long long t0 = globaltimer_ns();
        while (!__all_sync(0xffffffffu, ld_relaxed_sys(Lf) >= Lt && ld_relaxed_sys(Rf) >= Rt)) {
            if (globaltimer_ns() - t0 > HEAT1D_WAIT_NS) __trap();  // a neighbour rank is gone
        }
        if (doL) (void)ld_acquire_sys(Lf);
        if (doR) (void)ld_acquire_sys(Rf);
        __syncwarp();
        const double *LE = lrem ? mbox_data(mb.self, 0, g) : edges + ((size_t)s.left * 4 + (p & 1) * 2) * T + T;
        const double *RE = rrem ? mbox_data(mb.self, 1, g) : edges + ((size_t)s.right * 4 + (p & 1) * 2) * T;
        for (int i = lane; i < T; i += 32) {
            if (doL) s.row[i] = __ldcg(LE + i);
            if (doR) s.row[s.own + T + i] = __ldcg(RE + i);
        }
        __syncwarp();
        return;
    }
    // every lane polls (one coalesced request per poll); the vote makes the exit
    // warp-uniform, so ptxas keeps the step loop's shuffles non-collective.
    // Relaxed polls: an acquire at gpu scope invalidates L1 (CCTL.IVALL) each
    // time; one acquire per flag after the wait orders the edge reads.
    while (!__all_sync(0xffffffffu, ld_relaxed(flags + s.left) >= p + 1 && ld_relaxed(flags + s.right) >= p + 1)) {
    }
    (void)ld_acquire(flags + s.left);
    (void)ld_acquire(flags + s.right);
    __syncwarp();
    const double *LE = edges + ((size_t)s.left * 4 + (p & 1) * 2) * T + T;  // left's side 1
    const double *RE = edges + ((size_t)s.right * 4 + (p & 1) * 2) * T;     // right's side 0
    for (int i = lane; i < T; i += 32) {
        s.row[i] = __ldcg(LE + i);
        s.row[s.own + T + i] = __ldcg(RE + i);
    }
    __syncwarp();
}

}  // namespace

// MB: the cross-rank mailbox code is compiled in (only then: it costs ~30 registers).
// DF: tagged-word halos between spans (V >= 25), data-as-flag mailboxes between ranks.
template <int V, int OPS, bool MB, bool DF>
__global__ void __launch_bounds__(256, (DF && V <= 33 && !(MB && OPS == 1)) ? 2 : 0)
k6_resident(const double *__restrict__ A, double *__restrict__ B, int64_t n, int T, int64_t nt, double r,
            double rr, double *__restrict__ edges, unsigned *__restrict__ flags, int Wt, Guard guard,
            FastRange fr, MboxArgs mb_in, unsigned tbase) {
    const MboxArgs mb = MB ? mb_in : MboxArgs{};
    extern __shared__ __align__(16) double srow[];
    const int lane = threadIdx.x & 31;
    const int wib = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);  // warp-uniform for the compiler
    const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
    if (gw >= Wt) return;  // whole warps only; no CTA-wide barrier is used below
    const int Ns = Wt;
    double *rows = srow + (size_t)wib * (32 * V + 1);
    const Span a = make_span(gw, Ns, n, rows);
    const int live = a.own + 2 * T;
    HCHECK(live <= 32 * V && a.own >= T && a.start + a.own <= n);  // the span and its halos fit
    HCHECK((size_t)(blockDim.x >> 5) * (32 * V + 1) * 8 <= dynamic_smem_bytes());
    HCHECK(T <= MBOX_TMAX);
    const bool scaled = !ops_scaled(OPS) || __shfl_sync(0xffffffffu, (int)scaled_in_range(fr), 0) != 0;
    double ua[V], v[V];
    // scaled variants: r is their coefficient c, rr the true r; r^T per full period
    const double scaleT = ops_scaled(OPS) ? scale_of(rr, T) : 1.0;
    load_span<V>(a, A, n, T, lane);
    row_to_regs<V>(a.row, ua, lane);

    if (mb.on && (a.id == 0 || a.id == Ns - 1)) {  // outer halos of the initial state: neighbour ranks
        mbox_publish<DF>(a, Ns, T, mb.base, mb, lane);
        refresh<DF, MB>(a, T, 0, edges, flags, lane, Ns, mb, mb.base, tbase, true);
        row_to_regs<V>(a.row, ua, lane);
    }
    int64_t done = 0;
    for (unsigned p = 0;; ++p) {
        const int Tp = (int)((nt - done) < T ? (nt - done) : T);
        const double sc = (ops_scaled(OPS) && Tp != T) ? scale_of(rr, Tp) : scaleT;
        period_steps<V, OPS>(ua, v, a.row, Tp, r, sc, guard, live, lane, scaled, fr.r);
        regs_to_row<V>(ua, a.row, lane);
        done += Tp;
        if (done >= nt) break;
        // system scope only for the slab's two boundary spans (their halos cross GPUs):
        // a .sys fence in every warp every period cost more than half of C5's speed
        if (MB && mb.on && (a.id == 0 || a.id == Ns - 1)) {
            publish<DF>(a, T, p, edges, flags, tbase, lane);
            mbox_publish<DF>(a, Ns, T, mb.base + 1 + p, mb, lane);
            refresh<DF, true>(a, T, p, edges, flags, lane, Ns, mb, mb.base + 1 + p, tbase);
        } else {
            publish<DF>(a, T, p, edges, flags, tbase, lane);
            refresh<DF, false>(a, T, p, edges, flags, lane, Ns, mb, mb.base + 1 + p, tbase);
        }
        row_to_regs<V>(a.row, ua, lane);
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const int q = T + lane + 32 * k;
        if (q < T + a.own) B[a.start + (q - T)] = a.row[q];
    }
}

namespace {
// cells per lane: at most 17 for periods T <= 32, 33 for 32 < T <= 64, 49 up to 128 (span
// 32V >= own + 2T); the plan then takes the smallest instantiated V that holds its spans
// (every step computes all 32V register cells, live or slack: C2's 845-cell spans + 128 halo
// cells fit V = 31, 6 % less work than V = 33)
int rv_of(int T) { return T > 64 ? 49 : T > 32 ? 33 : 17; }
constexpr int kResV[] = {17, 25, 29, 31, 33, 49};  // instantiated (res_fn)
// warps per SM the register budget allows: V=17: ~100 regs; V=25..33: <= 128 regs; V=49: ~220 regs
int max_wps(int rv) { return rv == 49 ? 9 : rv >= 25 ? 15 : 20; }
constexpr int MAX_WPS_ANY = 20;
constexpr int MAX_NW = 8;     // warps per CTA (__launch_bounds__(256))

struct ResPlan {
    int64_t wt = 0, nw = 0, grid = 0;
    int rv = 17;
    size_t smem = 0;
};

// Tagged-word halos for V >= 25 spans (every arithmetic form; the matched kernels are
// compiled with a 2-blocks/SM register target: left alone ptxas gave them ~155 registers
// and -25 %; profiles/r01_k6_sync3.jsonl).  V = 17 spans (periods T <= 32) keep the flag
// protocol, whose build keeps three CTAs per SM co-resident for the largest on-chip rings.
bool res_df(int rv) { return rv >= 25; }

template <int V>
const void *res_fn_v(int ops, bool mbox) {
    constexpr bool DF = V >= 25;
    if (mbox) {
        switch (ops) {
            case 4: return (const void *)&k6_resident<V, 4, true, DF>;
            case 3: return (const void *)&k6_resident<V, 3, true, DF>;
            case 2: return (const void *)&k6_resident<V, 2, true, DF>;
            default: return (const void *)&k6_resident<V, 1, true, DF>;
        }
    }
    switch (ops) {
        case 4: return (const void *)&k6_resident<V, 4, false, DF>;
        case 3: return (const void *)&k6_resident<V, 3, false, DF>;
        case 2: return (const void *)&k6_resident<V, 2, false, DF>;
        default: return (const void *)&k6_resident<V, 1, false, DF>;
    }
}

const void *res_fn(int ops, int rv, bool mbox) {
    switch (rv) {
        case 49: return res_fn_v<49>(ops, mbox);
        case 33: return res_fn_v<33>(ops, mbox);
        case 31: return res_fn_v<31>(ops, mbox);
        case 29: return res_fn_v<29>(ops, mbox);
        case 25: return res_fn_v<25>(ops, mbox);
        default: return res_fn_v<17>(ops, mbox);
    }
}

cudaError_t res_attr(const void *fn) {  // raise the dynamic shared-memory limit once per kernel
    static std::mutex mu;
    static std::vector<const void *> done;
    std::lock_guard<std::mutex> lk(mu);
    for (const void *d : done)
        if (d == fn) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         MAX_NW * (32 * 49 + 1) * 8);
    if (e == cudaSuccess) done.push_back(fn);
    return e;
}

// Split the ring into Ns = Wt equal spans (each owning >= T cells, span own + 2T <= 32*RV)
// with warps balanced across SMs, one span per warp.
bool res_plan(int ops, int64_t n, int T, int num_sms, ResPlan *p, bool mbox = false) {
    const int RV = rv_of(T);
    p->rv = RV;
    const int cap = 32 * RV - 2 * T;
    if (T < 1 || cap <= 0 || n < T) return false;
    const int64_t wt_min = (n + cap - 1) / cap;
    if (wt_min <= num_sms) {
        p->wt = wt_min;  // one warp per CTA, each on its own SM
        p->nw = 1;
        p->grid = p->wt;
    } else {
        const int64_t wps = (wt_min + num_sms - 1) / num_sms;
        if (wps > max_wps(RV)) return false;
        const int64_t cps = (wps + MAX_NW - 1) / MAX_NW;  // CTAs per SM (blocks <= 8 warps)
        p->nw = (wps + cps - 1) / cps;
        p->grid = (int64_t)num_sms * cps;
        p->wt = p->grid * p->nw;
    }
    while (p->wt > 1 && n / p->wt < T) {
        p->wt = (p->wt + 1) / 2;
        p->nw = 1;
        p->grid = p->wt;
    }
    const int64_t ns = p->wt;
    const int64_t need = n / ns + (n % ns ? 1 : 0) + 2 * T;  // the largest span with its halos
    if (n / ns < T || need > 32 * RV) return false;
#ifndef HEAT1D_K6_VFIXED
    // the smallest V of the same protocol family (flags: 17; tagged words: 25..49) that holds it
    for (int v : kResV)
        if (v <= RV && res_df(v) == res_df(RV) && 32 * v >= need) {
            p->rv = v;
            break;
        }
#endif
    p->smem = (size_t)p->nw * (32 * p->rv + 1) * sizeof(double);
    const void *fn = res_fn(ops, p->rv, mbox);
    if (res_attr(fn) != cudaSuccess) return false;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, (int)(p->nw * 32), p->smem) != cudaSuccess)
        return false;
    if (getenv("HEAT1D_DEBUG"))
        fprintf(stderr, "[heat1d] K6 plan n=%lld T=%d V=%d ops=%d wt=%lld nw=%lld grid=%lld occ=%d smem=%zu\n",
                (long long)n, T, p->rv, ops, (long long)p->wt, (long long)p->nw, (long long)p->grid, occ, p->smem);
    return (int64_t)occ * num_sms >= p->grid;  // cooperative launch: all CTAs co-resident
}

}  // namespace

int64_t resident_capacity(int T, int num_sms) {
    const int rv = rv_of(T);
    return (int64_t)num_sms * max_wps(rv) * (32 * rv - 2 * T);
}

bool resident_fits(int ops, int64_t n, int T, int num_sms, bool mbox) {
    ResPlan p;
    return res_plan(ops, n, T, num_sms, &p, mbox);
}

int resident_plan_v(int ops, int64_t n, int T, int num_sms, bool mbox) {
    ResPlan p;
    return res_plan(ops, n, T, num_sms, &p, mbox) ? p.rv : 0;
}

// edges: [Ns][2 parities][2 sides][T] cells, 16 B each (tagged words; the V = 17 flag
// protocol uses the first half as plain doubles), then the per-span flags
size_t resident_scratch_bytes(int T, int num_sms) {
    const int64_t ns = (int64_t)num_sms * (MAX_WPS_ANY + MAX_NW);  // >= any plan's wt
    return (size_t)ns * 4 * T * 16 + (size_t)ns * sizeof(unsigned) + 256;
}

cudaError_t resident_scratch_init(void *scratch, int T, int num_sms, cudaStream_t st) {
    // tag 0 everywhere: launches use tags >= 1 (launch_resident's tbase)
    return cudaMemsetAsync(scratch, 0, resident_scratch_bytes(T, num_sms), st);
}


cudaError_t launch_mbox_init(double *mbox, cudaStream_t st) {  // every tag 0, flags 0
    return cudaMemsetAsync(mbox, 0, MBOX_BYTES, st);
}

cudaError_t launch_resident(int ops, const double *A, double *B, int64_t n, int T, int64_t nt, double q,
                            double r, Guard guard, const FastRange &fr, void *scratch, int num_sms, cudaStream_t st,
                            int *warps_out, int *v_out, const MboxArgs &mb, unsigned tbase) {
    ResPlan p;
    if (!res_plan(ops, n, T, num_sms, &p, mb.on != 0)) return cudaErrorInvalidValue;
    const int64_t ns = p.wt;
    double *edges = static_cast<double *>(scratch);
    unsigned *flags = reinterpret_cast<unsigned *>(edges + (size_t)ns * 4 * T * 2);
    cudaError_t e = cudaMemsetAsync(flags, 0, (size_t)ns * sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    int Wt = (int)p.wt;
    // (tagged edges need no reset between launches: tbase is new for every launch)
    void *args[] = {(void *)&A, (void *)&B, (void *)&n, (void *)&T, (void *)&nt, (void *)&q, (void *)&r,
                    (void *)&edges, (void *)&flags, (void *)&Wt, (void *)&guard, (void *)&fr, (void *)&mb,
                    (void *)&tbase};
    if (warps_out) *warps_out = Wt;
    if (v_out) *v_out = p.rv;
    return cudaLaunchCooperativeKernel(res_fn(ops, p.rv, mb.on != 0), dim3((unsigned)p.grid),
                                       dim3((unsigned)(p.nw * 32)), args, p.smem, st);
}

}  // namespace heat1d
