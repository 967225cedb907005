// heat1d.cpp -- host runtime behind include/heat1d.h.
//
// One handle per rank.  A handle owns S slabs (S = virtual_slabs on one GPU,
// else 1) of the periodic ring, each stored as two padded fp64 buffers
//     [pad ghost cells | count cells | pad ghost cells]
// (ping-pong, Jacobi: PAPER.md:68 reads time-t values only).
// A "pass" advances T steps:
//   single slab, single rank : K2 over [0,n) reading its own periodic pads,
//                              which K2 rewrites for the next pass (self-halo)
//   several slabs / ranks    : exchange depth-T halos with the ring neighbours
//                              on the comm stream (NCCL send/recv, or device
//                              copies between virtual slabs) while K2 updates
//                              the interior [T, n-T); then K3 does the edges.
// This is the paper's segmented ghost-zone algorithm with the
// exchange done every T steps at depth T instead of every step at depth 1.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys/ncu timelines

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <chrono>
#include <cstring>
#include <thread>
#include <string>
#include <vector>

#include "heat1d.h"
#include "kernels.h"

using heat1d::PassGeom;

namespace {

struct Slab {
    int64_t first = 0, count = 0;
    double *buf[2] = {nullptr, nullptr};  // base of each padded buffer
    // transport P2P: this slab's two exchange-index words (side 0 = left pad, +32 = right
    // pad), where its new edge strips go in the neighbours' buffers (indexed by buffer),
    // and the neighbours' words for those pads
    unsigned *flags = nullptr;
    double *put_left[2] = {nullptr, nullptr}, *put_right[2] = {nullptr, nullptr};
    unsigned *nflag_left = nullptr, *nflag_right = nullptr;
};

thread_local std::string g_create_error;

}  // namespace

struct heat1d_s {
    int device = 0;
    int rank = 0, nranks = 1;
    int64_t nx = 0, np = 0, N = 0, nt_default = 0;
    double k = 0, dt = 0, dx = 0, r = 0;
    double q = 0;  // per-step coefficient of the arithmetic variant (r, or c = (1-2r)/r scaled)
    int T = 8, mode = 0, den = 0, kernel = 0, ops = 4;
    int ops_fast = 0;                    // scaled fast variant chosen at create (0: none)
    unsigned long long *absmax = nullptr;  // device word for K5 (fast mode range check)
    bool blocking = true, use_graphs = true;
    int64_t pad = 16;
    int64_t first = 0, count = 0;  // this rank's range (union of its slabs)
    std::vector<Slab> slabs;
    int cur = 0;
    bool initialized = false;
    int poisoned = 0;
    int64_t steps_done = 0;
    int64_t launches = 0;
    int num_sms = 148;
    PassGeom geom{49, 4, 2, 2, 4};
    int last_grid = 0;
    bool resident = false;     // K6 path
    // K6 across ranks (or, HEAT1D_K6_MAILBOX=1, one rank routing its wrap through itself):
    // this rank's mailbox and the neighbour ranks' (CUDA IPC peer mappings)
    double *mbox = nullptr, *mbox_left = nullptr, *mbox_right = nullptr;
    bool mbox_ipc_left = false, mbox_ipc_right = false;
    unsigned k6_base = 0;  // global exchange index of the next K6 launch
    unsigned k6_tag = 1;   // edge tag of the next K6 launch's first period (resident.cu tagged words)
    void *res_scratch = nullptr;
    int res_warps = 0;
    int res_V = 0;  // cells per lane of the last K6 launch

    cudaStream_t stream = nullptr, comm = nullptr;
    bool own_stream = false, own_comm = false;
    // heat1d_solve_host: copy streams, per-slot events, per-window max|u0| words
    cudaStream_t st_h2d = nullptr, st_d2h = nullptr;
    cudaEvent_t ev_in[3] = {}, ev_comp[3] = {}, ev_out[3] = {};  // per window slot
    unsigned long long *win_absmax = nullptr;
    int64_t win_absmax_n = 0;
    int64_t stream_windows = 0;  // windows of the last heat1d_solve_host (0 = plain sequence)
    // test hooks, resolved once at create (fault injection of the tests)
    unsigned comm_delay_us = 0;  // HEAT1D_COMM_DELAY_US: hold the comm stream before each exchange
    bool poison_pads = false;    // HEAT1D_POISON_PADS=1: NaN ghost pads at every initial state
    int64_t window_cells = 0;    // > 0: streaming handle (opts.window_cells): only solve_host
    int64_t buf_len = 0;         // doubles per ping-pong buffer of slab 0 (as allocated)
    // transport P2P (several slabs): exchange-index words of this handle's slabs, the
    // neighbour ranks' allocations mapped over CUDA IPC, and the next exchange index
    int transport = HEAT1D_TRANSPORT_NCCL;
    unsigned *xflags = nullptr;
    void *peer_alloc[2] = {nullptr, nullptr}, *peer_flags[2] = {nullptr, nullptr};  // [0] left, [1] right
    bool peer_open[4] = {false, false, false, false};
    unsigned xg = 0;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    ncclComm_t nccl = nullptr;
    void *alloc = nullptr;
    bool own_alloc = true;  // false: opts.dev_buf (caller-owned, e.g. a torch tensor)

    // CUDA graphs of whole run(nt) pass sequences, keyed by (nt, starting buffer)
    struct Graph {
        int64_t nt;
        int cur0, cur1;
        int64_t launches;
        cudaGraphExec_t exec;
    };
    std::vector<Graph> graphs;

    bool prof = false;
    // profiling (heat1d_set_profiling): CUDA-event pairs around every kernel group, on the
    // stream it runs on; collected into the dominant kernel's totals and a trace
    struct ProfRec {
        cudaEvent_t a, b;
        int stream, kind;
    };
    std::vector<cudaEvent_t> ev_pool;  // free events
    std::vector<cudaEvent_t> ev_all;   // every event created (destroyed with the handle)
    std::vector<ProfRec> prof_recs;    // recorded, not yet collected
    cudaEvent_t prof_t0 = nullptr;     // the trace's time origin (compute stream)
    std::vector<heat1d_trace_event> trace;
    int64_t prof_launches = 0;
    double prof_ms = 0.0;

    std::string last_error;

    bool multi() const { return nranks > 1 || slabs.size() > 1; }
};

namespace {

int set_error(heat1d_t h, int status, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h)
        h->last_error = buf;
    else
        g_create_error = buf;
    return status;
}

struct NvtxRange {  // scoped NVTX range (no-op unless a profiler is attached)
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int fail_cuda(heat1d_t h, cudaError_t e, const char *what, int line) {
    if (h) h->poisoned = HEAT1D_ECUDA;
    cudaGetLastError();  // clear a non-sticky error so it does not leak into other handles
    return set_error(h, HEAT1D_ECUDA, "CUDA error %s (%s) at heat1d.cpp:%d: %s", cudaGetErrorName(e),
                     cudaGetErrorString(e), line, what);
}

int fail_nccl(heat1d_t h, ncclResult_t e, const char *what, int line) {
    if (h) h->poisoned = HEAT1D_ENCCL;
    return set_error(h, HEAT1D_ENCCL, "NCCL error %d (%s) at heat1d.cpp:%d: %s", (int)e, ncclGetErrorString(e),
                     line, what);
}

#define CK(call)                                                     \
    do {                                                             \
        cudaError_t e_ = (call);                                     \
        if (e_ != cudaSuccess) return fail_cuda(h, e_, #call, __LINE__); \
    } while (0)

#define NK(call)                                                     \
    do {                                                             \
        ncclResult_t e_ = (call);                                    \
        if (e_ != ncclSuccess) return fail_nccl(h, e_, #call, __LINE__); \
    } while (0)

bool is_pow2(double r) {
    if (!(r > 0.0) || !std::isfinite(r)) return false;
    int e;
    const double m = std::frexp(r, &e);
    return m == 0.5 && r >= 2.2250738585072014e-308;  // normal power of two
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

int64_t pad_for(int T) { return round_up((int64_t)T + 2, 16); }

// Exactness guard (stencil.cuh, DESIGN.md c3) of a block of Tp steps in arithmetic `ops`.
heat1d::Guard guard_for(heat1d_t h, int ops, int Tp);
heat1d::FastRange fast_range(heat1d_t h, int ops, const unsigned long long *word);

// Plain partition arithmetic (also exported as heat1d_partition).
int partition(int64_t nx, int64_t np, int32_t G, int32_t g, int64_t *first, int64_t *count) {
    if (nx < 1 || np < 1 || G < 1 || g < 0 || g >= G) return HEAT1D_EINVAL;
    if (nx > ((int64_t)1 << 62) / np) return HEAT1D_EINVAL;
    const int64_t N = nx * np;
    if (np >= G) {  // whole partitions, front-loaded remainder
        const int64_t base = np / G, rem = np % G;
        const int64_t parts = base + (g < rem ? 1 : 0);
        const int64_t p0 = (int64_t)g * base + (g < rem ? g : rem);
        *first = p0 * nx;
        *count = parts * nx;
    } else {  // fewer partitions than slabs: split cells, front-loaded
        if (N < G) return HEAT1D_EINVAL;
        const int64_t base = N / G, rem = N % G;
        *first = (int64_t)g * base + (g < rem ? g : rem);
        *count = base + (g < rem ? 1 : 0);
    }
    return HEAT1D_OK;
}

int64_t min_slab(int64_t nx, int64_t np, int32_t G) {
    int64_t mn = INT64_MAX, f, c;
    for (int g = 0; g < G; ++g)
        if (partition(nx, np, G, g, &f, &c) == HEAT1D_OK && c < mn) mn = c;
    return mn;
}

// The four halo messages of one rank (heat1d_plan_exchange): its slab of
// `count` cells sends its last and first `depth` cells to the right and left neighbours
// and receives their edges into its left and right ghost pads.  The single source of the
// offsets for every exchange the library issues (exchange(), the nt-deep halos of a
// multi-rank heat1d_solve_host).
void make_plan(int64_t count, int64_t depth, int rank, int nranks, heat1d_exchange_plan *plan) {
    plan->left = (rank - 1 + nranks) % nranks;
    plan->right = (rank + 1) % nranks;
    plan->send_right_off = count - depth;
    plan->send_left_off = 0;
    plan->recv_left_off = -depth;
    plan->recv_right_off = count;
    plan->cells = depth;
}

// Issue a plan's messages on `st` in the plan's order (matters when left == right):
// send(right edge -> right), send(left edge -> left), recv(left pad <- left), recv(right pad
// <- right).  `send_base` / `recv_base` hold cell 0 of the slab (they differ when the
// caller stages the edges elsewhere, e.g. host arrays); offsets are relative to them.
ncclResult_t issue_plan(const heat1d_exchange_plan &pl, const double *send_base, double *recv_base,
                        ncclComm_t comm, cudaStream_t st) {
    ncclResult_t e;
    const size_t n = (size_t)pl.cells;
    if ((e = ncclGroupStart()) != ncclSuccess) return e;
    if ((e = ncclSend(send_base + pl.send_right_off, n, ncclDouble, pl.right, comm, st)) != ncclSuccess) goto end;
    if ((e = ncclSend(send_base + pl.send_left_off, n, ncclDouble, pl.left, comm, st)) != ncclSuccess) goto end;
    if ((e = ncclRecv(recv_base + pl.recv_left_off, n, ncclDouble, pl.left, comm, st)) != ncclSuccess) goto end;
    e = ncclRecv(recv_base + pl.recv_right_off, n, ncclDouble, pl.right, comm, st);
end:
    const ncclResult_t e2 = ncclGroupEnd();
    return e != ncclSuccess ? e : e2;
}

int auto_T(int ops, double r) {
    // each pass moves 16/T bytes per update, so T is raised until the pass is
    // fp64-issue bound; what a deeper pass costs is redundant cells -- with feed tiles
    // (k2f_pass) only the right margin, T^2/2 cell-steps per tile -- against per-tile phases
    // that a deeper pass amortises: T = 128, the largest, is the fastest for every arithmetic
    // form (profiles/r02_feed_ab.md).  The scaled 2-op form grows by r^-T within a pass, so
    // it takes 128 only while r^-128 <= 2^512 (r >= 1/16), else 64 (r >= 1/256: <= 2^512).
    if (ops == 2 && r < 1.0 / 16.0) return 64;
    return 128;
}

// K6's period when the caller leaves T to us: every step computes all 32V
// register cells of a span (live or slack) and every period pays one halo hand-off, about
// 154 span-cell-steps' worth (fit to the C2/C5 A/B, profiles/r02_k6_tv.jsonl); so among
// T in {64, 56, 48, 40} take the one minimising V(T) * nt + ceil(nt / T) * 154, V(T) the
// plan's cells per lane for the LARGEST slab -- a global quantity, the same on every rank.
int k6_auto_T(heat1d_t h, int64_t nx, int64_t np, int G, int64_t nt, int64_t mslab) {
    int64_t nmax = 0;
    for (int g = 0; g < G; ++g) {
        int64_t f = 0, c = 0;
        partition(nx, np, G, g, &f, &c);
        nmax = std::max(nmax, c);
    }
    const int ops = h->ops_fast ? h->ops_fast : h->ops;
    const int64_t steps = nt > 0 ? nt : 1;
    int best = (int)std::min<int64_t>(64, mslab);
    double best_cost = -1.0;
    for (int T : {64, 56, 48, 40}) {
        if (T > mslab) continue;
        const int v = heat1d::resident_plan_v(ops, nmax, T, h->num_sms, G > 1);
        if (v == 0) continue;
        const double cost = (double)v * (double)steps + (double)((steps + T - 1) / T) * 154.0;
        if (best_cost < 0 || cost < best_cost) {
            best = T;
            best_cost = cost;
        }
    }
    cudaGetLastError();
    return best;
}

bool parse_geom_env(PassGeom *g) {
    const char *s = getenv("HEAT1D_GEOM");  // "V,NW,S,ctas_per_sm[,kind]" (tuning knob)
    if (!s || !*s) return false;
    int v, nw, st, c, kind = 4;
    const int got = sscanf(s, "%d,%d,%d,%d,%d", &v, &nw, &st, &c, &kind);
    if (got < 4) return false;
    *g = PassGeom{v, nw, st, c, kind};
    return true;
}

cudaEvent_t prof_event(heat1d_t h) {
    if (h->ev_pool.empty()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        h->ev_all.push_back(e);
        return e;
    }
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
}

// Open a profiled interval on stream `st` (no-op unless profiling); close it with prof_end.
int prof_begin(heat1d_t h, cudaStream_t st, heat1d_s::ProfRec *rec, int stream_id, int kind) {
    rec->a = rec->b = nullptr;
    if (!h->prof) return HEAT1D_OK;
    rec->a = prof_event(h);
    rec->b = prof_event(h);
    rec->stream = stream_id;
    rec->kind = kind;
    if (!rec->a || !rec->b) return set_error(h, HEAT1D_ECUDA, "event pool");
    CK(cudaEventRecord(rec->a, st));
    return HEAT1D_OK;
}

int prof_end(heat1d_t h, cudaStream_t st, const heat1d_s::ProfRec &rec) {
    if (!h->prof || !rec.b) return HEAT1D_OK;
    CK(cudaEventRecord(rec.b, st));
    h->prof_recs.push_back(rec);
    return HEAT1D_OK;
}

constexpr size_t kTraceMax = 1 << 20;  // trace entries kept per profiling session

int prof_collect(heat1d_t h) {
    if (h->prof_recs.empty()) return HEAT1D_OK;
    CK(cudaStreamSynchronize(h->stream));
    if (h->comm) CK(cudaStreamSynchronize(h->comm));
    for (const auto &r : h->prof_recs) {
        float ms = 0.f, t0 = 0.f;
        CK(cudaEventElapsedTime(&ms, r.a, r.b));
        if (r.stream == 0) {  // the dominant kernel: the interior pass K2 or the resident K6
            h->prof_ms += ms;
            h->prof_launches += 1;
        }
        if (h->prof_t0 && h->trace.size() < kTraceMax) {
            CK(cudaEventElapsedTime(&t0, h->prof_t0, r.a));
            h->trace.push_back(heat1d_trace_event{r.stream, r.kind, (double)t0, (double)t0 + ms});
        }
        h->ev_pool.push_back(r.a);
        h->ev_pool.push_back(r.b);
    }
    h->prof_recs.clear();
    return HEAT1D_OK;
}

double *cell0(heat1d_t h, const Slab &s, int which) { return s.buf[which] + h->pad; }

heat1d::Guard guard_for(heat1d_t h, int ops, int Tp) {
    return heat1d::guard_of(h->mode == HEAT1D_MODE_MATCHED, ops, h->r, Tp);
}

// The scaled fast forms' range (DESIGN.md c21): a pass of up to T steps grows the scaled state to
// max|u0| * r^-T, which must stay below 2^1000, i.e. max|u0| < 2^E with E the largest integer
// below 1000 - T log2(1/r).  `word` = a K5 max|u| word on the device.
heat1d::FastRange fast_range(heat1d_t h, int ops, const unsigned long long *word) {
    heat1d::FastRange f;
    if (!heat1d::ops_scaled(ops)) return f;
    const double X = 1000.0 - (double)h->T * std::log2(1.0 / h->r);
    const double E = std::ceil(X) - 1.0;
    f.absmax = word;
    f.r = h->r;
    if (E < -1074.0) {
        f.limit = 0ull;  // only an all-zero state
    } else {
        const double lim = std::ldexp(1.0, (int)E);
        unsigned long long bits;
        memcpy(&bits, &lim, sizeof bits);
        f.limit = bits - 1ull;  // |x| bits <= limit  <=>  |x| < 2^E
    }
    return f;
}

int launch_pass_slab(heat1d_t h, const Slab &s, int Tp, int64_t lo, int64_t hi, int wrapT) {
    heat1d_s::ProfRec rec;
    int rc = prof_begin(h, h->stream, &rec, 0, HEAT1D_TRACE_K2);
    if (rc) return rc;
    int grid = 0;
    CK(heat1d::launch_pass(h->geom, h->ops, cell0(h, s, h->cur), cell0(h, s, h->cur ^ 1), s.count, Tp, lo, hi,
                           wrapT, h->q, heat1d::scale_of(h->r, Tp), guard_for(h, h->ops, Tp),
                           fast_range(h, h->ops, h->absmax), h->num_sms, h->stream, &grid));
    if (grid > 0) h->launches++;
    h->last_grid = grid > 0 ? grid : h->last_grid;
    return prof_end(h, h->stream, rec);
}

// Fill the depth-Tp ghost pads of every slab of the current buffer from the
// ring neighbours (comm stream).  Message plan = heat1d_plan_exchange.
int exchange(heat1d_t h, int Tp) {
    const int ns = (int)h->slabs.size();
    const int cur = h->cur;
    if (h->nranks > 1) {
        const Slab &s = h->slabs[0];
        double *A = cell0(h, s, cur);
        heat1d_exchange_plan pl;
        make_plan(s.count, Tp, h->rank, h->nranks, &pl);
        NK(issue_plan(pl, A, A, h->nccl, h->comm));
        return HEAT1D_OK;
    }
    // virtual slabs on one device: the same messages as device copies -- slab g's receives
    // are its neighbours' sends of the same plan
    for (int g = 0; g < ns; ++g) {
        const Slab &s = h->slabs[g];
        const Slab &L = h->slabs[(g - 1 + ns) % ns];
        const Slab &R = h->slabs[(g + 1) % ns];
        heat1d_exchange_plan ps, pL, pR;
        make_plan(s.count, Tp, g, ns, &ps);
        make_plan(L.count, Tp, (g - 1 + ns) % ns, ns, &pL);
        make_plan(R.count, Tp, (g + 1) % ns, ns, &pR);
        double *A = cell0(h, s, cur);
        CK(cudaMemcpyAsync(A + ps.recv_left_off, cell0(h, L, cur) + pL.send_right_off, (size_t)Tp * 8,
                           cudaMemcpyDeviceToDevice, h->comm));
        CK(cudaMemcpyAsync(A + ps.recv_right_off, cell0(h, R, cur) + pR.send_left_off, (size_t)Tp * 8,
                           cudaMemcpyDeviceToDevice, h->comm));
    }
    return HEAT1D_OK;
}

int run_resident(heat1d_t h, int64_t nt) {
    const Slab &s = h->slabs[0];
    heat1d_s::ProfRec rec;
    int rc = prof_begin(h, h->stream, &rec, 0, HEAT1D_TRACE_K6);
    if (rc) return rc;
    heat1d::MboxArgs mb;
    if (h->mbox) {
        mb.self = h->mbox;
        mb.left = h->mbox_left;
        mb.right = h->mbox_right;
        mb.base = h->k6_base;
        mb.on = 1;
        // indices base .. base+P-1 used (initial exchange + P-1 periods); skipping one more at
        // the run boundary keeps a slot from being rewritten while a slower neighbour may
        // still read it (resident.cu, mbox_publish)
        h->k6_base += (unsigned)((nt + h->T - 1) / h->T) + 2u;
    }
    // edge tags: unique per launch and period; before the 32-bit counter would wrap, the slots
    // go back to tag 0 and the count restarts (a stale tag must never equal a live one)
    const unsigned periods = (unsigned)((nt + h->T - 1) / h->T);
    if (h->k6_tag > 0xffffffffu - periods - 4u) {
        CK(heat1d::resident_scratch_init(h->res_scratch, h->T, h->num_sms, h->stream));
        h->k6_tag = 1;
    }
    const unsigned tbase = h->k6_tag;
    h->k6_tag += periods + 2u;
    CK(heat1d::launch_resident(h->ops, cell0(h, s, h->cur), cell0(h, s, h->cur ^ 1), s.count, h->T, nt, h->q,
                               h->r, guard_for(h, h->ops, h->T), fast_range(h, h->ops, h->absmax), h->res_scratch,
                               h->num_sms, h->stream, &h->res_warps, &h->res_V, mb, tbase));
    h->launches++;
    rc = prof_end(h, h->stream, rec);
    if (rc) return rc;
    h->cur ^= 1;
    // (no periodic pads to refresh: K6 reads its halos modularly and a resident handle never
    // runs another kernel family)
    h->steps_done += nt;
    return HEAT1D_OK;
}

int run_passes(heat1d_t h, int64_t nt) {
    NvtxRange range(h->resident ? "heat1d.run K6" : h->multi() ? "heat1d.run K2+exchange" : "heat1d.run K2");
    if (h->resident) return run_resident(h, nt);
    int64_t done = 0;
    while (done < nt) {
        if (h->kernel == HEAT1D_KERNEL_NAIVE) {
            const Slab &s = h->slabs[0];
            heat1d_s::ProfRec rec;
            int rc = prof_begin(h, h->stream, &rec, 0, HEAT1D_TRACE_K1);
            if (rc) return rc;
            // one step per launch: matched mode runs the oracle's literal sequence (OPS 5), fast
            // mode the contracted 3-op form
            CK(heat1d::launch_naive(h->mode == HEAT1D_MODE_MATCHED ? 5 : 3, cell0(h, s, h->cur),
                                    cell0(h, s, h->cur ^ 1), s.count, h->r, h->stream));
            rc = prof_end(h, h->stream, rec);
            if (rc) return rc;
            h->launches++;
            h->cur ^= 1;
            done += 1;
            continue;
        }
        const int Tp = (int)((nt - done) < h->T ? (nt - done) : h->T);
        if (!h->multi()) {
            const Slab &s = h->slabs[0];
            const int wrapT = (int)(h->T < s.count ? h->T : s.count);
            int rc = launch_pass_slab(h, s, Tp, 0, s.count, wrapT);
            if (rc) return rc;
        } else {
            // comm stream: halo exchange, then the two edge strips (K3, 2 small CTAs) as soon as
            // the ghosts land -- concurrently with the interior pass on the compute stream, so
            // only the exchange latency, never K3, can reach the critical path.  K2 writes
            // B[T, n-T), K3 writes B[0,T) and B[n-T, n): disjoint; both read A.
            CK(cudaEventRecord(h->ev_ready, h->stream));
            CK(cudaStreamWaitEvent(h->comm, h->ev_ready, 0));
            heat1d_s::ProfRec crec;
            int prc = prof_begin(h, h->comm, &crec, 1, HEAT1D_TRACE_HALO);
            if (prc) return prc;
            if (h->comm_delay_us) {  // fault injection (tests)
                CK(heat1d::launch_delay(h->comm_delay_us, h->comm));
                h->launches++;
            }
            int rc = HEAT1D_OK;
            if (h->transport == HEAT1D_TRANSPORT_P2P) {
                // K3p: wait for the ghosts of index xg, update the strips, put them straight
                // into the neighbours' pads of B with index xg+1
                if (done == 0) {
                    h->xg += 1;  // skip one index at every run boundary (slot-reuse safety, §8)
                    for (const Slab &s : h->slabs) {
                        CK(heat1d::launch_push_edges(cell0(h, s, h->cur), s.count, h->T, h->xg,
                                                     s.put_left[h->cur], s.put_right[h->cur], s.nflag_left,
                                                     s.nflag_right, h->comm));
                        h->launches++;
                    }
                }
                for (const Slab &s : h->slabs) {
                    CK(heat1d::launch_edges_put(h->ops, cell0(h, s, h->cur), cell0(h, s, h->cur ^ 1), s.count, Tp,
                                                h->q, heat1d::scale_of(h->r, Tp), guard_for(h, h->ops, Tp),
                                                fast_range(h, h->ops, h->absmax), s.flags, h->xg,
                                                s.put_left[h->cur ^ 1], s.put_right[h->cur ^ 1], s.nflag_left,
                                                s.nflag_right, h->comm));
                    h->launches++;
                }
                h->xg += 1;
            } else {
                rc = exchange(h, Tp);
                if (rc) return rc;
                for (const Slab &s : h->slabs) {
                    CK(heat1d::launch_edges(h->ops, cell0(h, s, h->cur), cell0(h, s, h->cur ^ 1), s.count, Tp, h->q,
                                            heat1d::scale_of(h->r, Tp), guard_for(h, h->ops, Tp),
                                            fast_range(h, h->ops, h->absmax), h->comm));
                    h->launches++;
                }
            }
            prc = prof_end(h, h->comm, crec);
            if (prc) return prc;
            CK(cudaEventRecord(h->ev_halo, h->comm));
            for (const Slab &s : h->slabs) {
                rc = launch_pass_slab(h, s, Tp, Tp, s.count - Tp, 0);
                if (rc) return rc;
            }
            CK(cudaStreamWaitEvent(h->stream, h->ev_halo, 0));
        }
        h->cur ^= 1;
        done += Tp;
    }
    h->steps_done += nt;
    return HEAT1D_OK;
}

// Replay (or capture, then replay) the pass sequence of run(nt) as one CUDA
// graph: one host submission per run instead of ~3 launches per pass.  Used
// for K2 pass sequences (single slab, virtual slabs, NCCL); K6 is already one
// launch and profiling needs per-launch events, so both bypass it.
int run_maybe_graph(heat1d_t h, int64_t nt) {
    const int64_t passes = (nt + h->T - 1) / h->T;
    if (!h->use_graphs || h->prof || h->resident || passes < 2) return run_passes(h, nt);
    for (auto &g : h->graphs) {
        if (g.nt == nt && g.cur0 == h->cur) {
            CK(cudaGraphLaunch(g.exec, h->stream));
            h->cur = g.cur1;
            h->steps_done += nt;
            h->launches += g.launches;
            return HEAT1D_OK;
        }
    }
    const int cur0 = h->cur;
    const int64_t l0 = h->launches, s0 = h->steps_done;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    int rc = run_passes(h, nt);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
    cudaGraphExec_t exec = nullptr;
    if (rc == HEAT1D_OK && e == cudaSuccess && graph &&
        cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
        cudaGraphDestroy(graph);
        heat1d_s::Graph g{nt, cur0, h->cur, h->launches - l0, exec};
        if (h->graphs.size() >= 8) {
            cudaGraphExecDestroy(h->graphs.front().exec);
            h->graphs.erase(h->graphs.begin());
        }
        h->graphs.push_back(g);
        h->cur = cur0;  // capture only recorded the work; replay it now
        h->launches = l0;
        h->steps_done = s0;
        CK(cudaGraphLaunch(exec, h->stream));
        h->cur = g.cur1;
        h->launches += g.launches;
        h->steps_done += nt;
        return HEAT1D_OK;
    }
    // capture not possible here: run directly (clears the capture error state)
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    if (rc != HEAT1D_OK) {
        if (!h->poisoned) return rc;
        h->poisoned = 0;  // the failure was the capture, not the device
    }
    h->cur = cur0;
    h->launches = l0;
    h->steps_done = s0;
    h->use_graphs = false;
    return run_passes(h, nt);
}

// Collective min over ranks of a local int (NCCL on the comm stream; synchronous).
int vote_min(heat1d_t h, int mine, int *all) {
    int *dv = nullptr;
    CK(cudaMalloc(&dv, sizeof(int)));
    CK(cudaMemcpy(dv, &mine, sizeof(int), cudaMemcpyHostToDevice));
    NK(ncclAllReduce(dv, dv, 1, ncclInt32, ncclMin, h->nccl, h->comm));
    CK(cudaMemcpyAsync(all, dv, sizeof(int), cudaMemcpyDeviceToHost, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    CK(cudaFree(dv));
    return HEAT1D_OK;
}

// K6 across ranks (every rank's slab fits: vote_min at create): allocate this
// rank's mailbox and map the two neighbours' mailboxes (CUDA IPC handles all-gathered
// over NCCL, opened with lazy peer access: remote stores travel over NVLink).
int setup_multi_resident(heat1d_t h) {
    const int G = h->nranks;
    int *dv = nullptr;
    CK(cudaMalloc(&dv, sizeof(int)));
    CK(cudaMalloc(&h->mbox, heat1d::MBOX_BYTES));
    CK(heat1d::launch_mbox_init(h->mbox, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    cudaIpcMemHandle_t mineh;
    CK(cudaIpcGetMemHandle(&mineh, h->mbox));
    char *dh = nullptr;
    CK(cudaMalloc(&dh, (size_t)G * sizeof(cudaIpcMemHandle_t)));
    CK(cudaMemcpy(dh + (size_t)h->rank * sizeof(mineh), &mineh, sizeof(mineh), cudaMemcpyHostToDevice));
    NK(ncclAllGather(dh + (size_t)h->rank * sizeof(mineh), dh, sizeof(mineh), ncclChar, h->nccl, h->comm));
    std::vector<cudaIpcMemHandle_t> all_h((size_t)G);
    CK(cudaMemcpyAsync(all_h.data(), dh, (size_t)G * sizeof(mineh), cudaMemcpyDeviceToHost, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    CK(cudaFree(dh));
    const int left = (h->rank - 1 + G) % G, right = (h->rank + 1) % G;
    void *pl = nullptr, *pr = nullptr;
    // every rank must map both neighbours' mailboxes, else all fall back to K2 passes with the
    // NCCL transport (T = Tr is a valid K2 depth: Tr <= the smallest slab)
    int ok = cudaIpcOpenMemHandle(&pl, all_h[(size_t)left], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    h->mbox_ipc_left = ok != 0;
    if (ok && right != left) {
        ok = cudaIpcOpenMemHandle(&pr, all_h[(size_t)right], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
        h->mbox_ipc_right = ok != 0;
    } else {
        pr = pl;
    }
    cudaGetLastError();
    int all_ok = 0;
    int rc = vote_min(h, ok, &all_ok);
    if (rc) return rc;
    if (!all_ok) {
        if (h->mbox_ipc_left) cudaIpcCloseMemHandle(pl);
        if (h->mbox_ipc_right) cudaIpcCloseMemHandle(pr);
        h->mbox_ipc_left = h->mbox_ipc_right = false;
        CK(cudaFree(h->mbox));
        h->mbox = nullptr;
        CK(cudaFree(dv));
        h->transport = HEAT1D_TRANSPORT_NCCL;
        return HEAT1D_OK;
    }
    h->mbox_left = static_cast<double *>(pl);
    h->mbox_right = static_cast<double *>(pr);
    // barrier: every rank's mailbox is zeroed and mapped before any rank's first K6 launch
    CK(cudaDeviceSynchronize());
    NK(ncclAllReduce(dv, dv, 1, ncclInt32, ncclMin, h->nccl, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    CK(cudaFree(dv));
    h->resident = true;
    if (cudaMalloc(&h->res_scratch, heat1d::resident_scratch_bytes(h->T, h->num_sms)) != cudaSuccess) {
        cudaGetLastError();
        return set_error(h, HEAT1D_ENOMEM, "resident scratch");
    }
    CK(heat1d::resident_scratch_init(h->res_scratch, h->T, h->num_sms, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    return HEAT1D_OK;
}

// Transport P2P: exchange-index words for every slab, and the addresses K3p puts its
// strips to -- the other virtual slabs' buffers, or the neighbour ranks' allocations
// opened from CUDA IPC handles all-gathered over NCCL (lazy peer access: NVLink stores).
int setup_p2p(heat1d_t h, int64_t nx, int64_t np) {
    const int ns = (int)h->slabs.size();
    const size_t fbytes = (size_t)ns * 64 * sizeof(unsigned);
    CK(cudaMalloc(&h->xflags, fbytes < 256 ? 256 : fbytes));
    CK(cudaMemset(h->xflags, 0, fbytes < 256 ? 256 : fbytes));
    for (int g = 0; g < ns; ++g) h->slabs[g].flags = h->xflags + (size_t)g * 64;
    if (h->nranks == 1) {
        for (int g = 0; g < ns; ++g) {
            Slab &s = h->slabs[g];
            const Slab &L = h->slabs[(g - 1 + ns) % ns], &R = h->slabs[(g + 1) % ns];
            for (int b = 0; b < 2; ++b) {
                s.put_left[b] = cell0(h, L, b) + L.count;  // L's right pad
                s.put_right[b] = cell0(h, R, b) - h->T;    // R's left pad
            }
            s.nflag_left = L.flags + 32;
            s.nflag_right = R.flags;
        }
        return HEAT1D_OK;
    }
    const int G = h->nranks;
    cudaIpcMemHandle_t mine[2];
    memset(mine, 0, sizeof mine);
    // a caller-owned opts.dev_buf may be a sub-allocation (torch's caching allocator): its
    // IPC handle would map the containing block, so such a rank votes for NCCL below
    int ok = h->own_alloc ? 1 : 0;
    if (ok && (cudaIpcGetMemHandle(&mine[0], h->alloc) != cudaSuccess ||
               cudaIpcGetMemHandle(&mine[1], h->xflags) != cudaSuccess))
        ok = 0;
    cudaGetLastError();
    const size_t hb = sizeof(mine);
    char *dh = nullptr;
    CK(cudaMalloc(&dh, (size_t)G * hb));
    CK(cudaMemcpy(dh + (size_t)h->rank * hb, mine, hb, cudaMemcpyHostToDevice));
    NK(ncclAllGather(dh + (size_t)h->rank * hb, dh, hb, ncclChar, h->nccl, h->comm));
    std::vector<cudaIpcMemHandle_t> all((size_t)G * 2);
    CK(cudaMemcpyAsync(all.data(), dh, (size_t)G * hb, cudaMemcpyDeviceToHost, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    const int nbr[2] = {(h->rank - 1 + G) % G, (h->rank + 1) % G};
    // every rank must map both neighbours, else all fall back to NCCL; a handle of zeros
    // (a neighbour that voted no) fails to open here too
    for (int side = 0; side < 2 && ok; ++side) {
        if (side == 1 && nbr[1] == nbr[0]) {  // G = 2: one peer on both sides
            h->peer_alloc[1] = h->peer_alloc[0];
            h->peer_flags[1] = h->peer_flags[0];
            break;
        }
        for (int k = 0; k < 2 && ok; ++k) {
            void **dst = k == 0 ? &h->peer_alloc[side] : &h->peer_flags[side];
            if (cudaIpcOpenMemHandle(dst, all[(size_t)nbr[side] * 2 + k], cudaIpcMemLazyEnablePeerAccess) ==
                cudaSuccess)
                h->peer_open[side * 2 + k] = true;
            else
                ok = 0;
        }
    }
    cudaGetLastError();
    int *dok = reinterpret_cast<int *>(dh);  // (handles already copied out)
    CK(cudaMemcpy(dok, &ok, sizeof ok, cudaMemcpyHostToDevice));
    NK(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, h->nccl, h->comm));
    CK(cudaMemcpyAsync(&ok, dok, sizeof ok, cudaMemcpyDeviceToHost, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    if (!ok) {  // no peer mapping somewhere: the NCCL transport for everyone
        for (int i = 0; i < 4; ++i)
            if (h->peer_open[i]) cudaIpcCloseMemHandle(i % 2 == 0 ? h->peer_alloc[i / 2] : h->peer_flags[i / 2]);
        for (int i = 0; i < 4; ++i) h->peer_open[i] = false;
        h->peer_alloc[0] = h->peer_alloc[1] = h->peer_flags[0] = h->peer_flags[1] = nullptr;
        h->transport = HEAT1D_TRANSPORT_NCCL;
        CK(cudaFree(dh));
        return HEAT1D_OK;
    }
    Slab &s = h->slabs[0];
    for (int side = 0; side < 2; ++side) {
        int64_t f = 0, c = 0;
        partition(nx, np, G, nbr[side], &f, &c);
        const int64_t len = round_up(c + 2 * h->pad, 32);  // the neighbour's buffer layout (same T)
        double *base = static_cast<double *>(h->peer_alloc[side]);
        for (int b = 0; b < 2; ++b) {
            double *c0 = base + (size_t)b * len + h->pad;
            if (side == 0)
                s.put_left[b] = c0 + c;  // left rank's right pad
            else
                s.put_right[b] = c0 - h->T;  // right rank's left pad
        }
        if (side == 0)
            s.nflag_left = static_cast<unsigned *>(h->peer_flags[0]) + 32;
        else
            s.nflag_right = static_cast<unsigned *>(h->peer_flags[1]);
    }
    // barrier: every rank's words are zeroed and mapped before any rank's first put
    CK(cudaDeviceSynchronize());
    NK(ncclAllReduce(dh, dh, 1, ncclInt32, ncclMin, h->nccl, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    CK(cudaFree(dh));
    return HEAT1D_OK;
}

int guard(heat1d_t h) {
    if (!h) return set_error(nullptr, HEAT1D_EINVAL, "NULL handle");
    if (h->poisoned) return h->poisoned;
    if (cudaSetDevice(h->device) != cudaSuccess) return set_error(h, HEAT1D_ECUDA, "cudaSetDevice failed");
    return HEAT1D_OK;
}

}  // namespace

extern "C" {

void heat1d_opts_default(heat1d_opts *o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->size = sizeof *o;
    o->device = -1;
    o->rank = 0;
    o->nranks = 1;
    o->nccl_id = nullptr;
    o->T = 0;
    o->mode = HEAT1D_MODE_MATCHED;
    o->denominator = HEAT1D_DEN_DX2;
    o->allow_unstable = 0;
    o->virtual_slabs = 1;
    o->kernel = HEAT1D_KERNEL_AUTO;
    o->blocking = 1;
    o->use_graphs = 1;
    o->resident = -1;
    o->transport = HEAT1D_TRANSPORT_P2P;  // falls back to NCCL at create if peers cannot be mapped
}

int heat1d_version(void) { return HEAT1D_VERSION; }

const char *heat1d_strerror(int status) {
    switch (status) {
        case HEAT1D_OK: return "ok";
        case HEAT1D_EINVAL: return "invalid argument";
        case HEAT1D_EUNSTABLE: return "unstable: r = k*dt/D > 1/2 (set allow_unstable)";
        case HEAT1D_ESTATE: return "invalid state (no initial condition, or poisoned handle)";
        case HEAT1D_ENOMEM: return "out of device memory";
        case HEAT1D_ECUDA: return "CUDA error";
        case HEAT1D_ENCCL: return "NCCL error";
        case HEAT1D_EUNSUPPORTED: return "unsupported";
        default: return "unknown status";
    }
}

int heat1d_partition(int64_t nx, int64_t np, int32_t nranks, int32_t rank, int64_t *first, int64_t *count) {
    if (!first || !count) return HEAT1D_EINVAL;
    return partition(nx, np, nranks, rank, first, count);
}

int heat1d_plan_exchange(int64_t nx, int64_t np, int32_t nranks, int32_t rank, int32_t T,
                         heat1d_exchange_plan *plan) {
    if (!plan || T < 1) return HEAT1D_EINVAL;
    int64_t first, count;
    int rc = partition(nx, np, nranks, rank, &first, &count);
    if (rc) return rc;
    if (T > min_slab(nx, np, nranks)) return HEAT1D_EINVAL;
    make_plan(count, T, rank, nranks, plan);
    return HEAT1D_OK;
}

int64_t heat1d_buffer_len(int64_t nx, int64_t np, const heat1d_opts *o) {
    heat1d_opts d;
    if (!o) {
        heat1d_opts_default(&d);
        o = &d;
    }
    const int G = o->virtual_slabs > 1 ? o->virtual_slabs : o->nranks;
    const int rank = o->virtual_slabs > 1 ? -1 : o->rank;
    const int T = o->T > 0 ? o->T : HEAT1D_T_MAX;  // auto T never exceeds the maximum
    const int64_t pad = pad_for(T);
    if (o->window_cells > 0) return 3 * 2 * round_up(o->window_cells + 2 * pad, 32);  // 3 slots x 2 buffers
    int64_t total = 0, f, c;
    for (int g = 0; g < G; ++g) {
        if (rank >= 0 && g != rank) continue;
        if (partition(nx, np, G, g, &f, &c) != HEAT1D_OK) return -1;
        total += 2 * round_up(c + 2 * pad, 32);
    }
    return total;
}

int heat1d_get_unique_id(void *out128) {
    if (!out128) return HEAT1D_EINVAL;
    ncclUniqueId id;
    ncclResult_t e = ncclGetUniqueId(&id);
    if (e != ncclSuccess) return set_error(nullptr, HEAT1D_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(e));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out128, &id, sizeof id);
    return HEAT1D_OK;
}

int heat1d_create(heat1d_t *out, int64_t nx, int64_t np, int64_t nt, double k, double dt, double dx,
                  const heat1d_opts *opts) {
    if (!out) return set_error(nullptr, HEAT1D_EINVAL, "out is NULL");
    *out = nullptr;
    heat1d_opts o;
    heat1d_opts_default(&o);
    if (opts) {
        if (opts->size != sizeof(heat1d_opts))
            return set_error(nullptr, HEAT1D_EINVAL, "opts.size %u != %zu", opts->size, sizeof(heat1d_opts));
        o = *opts;
    }
    if (nx < 1 || np < 1) return set_error(nullptr, HEAT1D_EINVAL, "nx and np must be >= 1");
    if (nx > ((int64_t)1 << 62) / np) return set_error(nullptr, HEAT1D_EINVAL, "nx*np exceeds 2^62");
    if (nt < 0) return set_error(nullptr, HEAT1D_EINVAL, "nt must be >= 0");
    if (!std::isfinite(k) || !std::isfinite(dt) || !std::isfinite(dx))
        return set_error(nullptr, HEAT1D_EINVAL, "k, dt, dx must be finite");
    if (k < 0 || dt <= 0 || dx <= 0) return set_error(nullptr, HEAT1D_EINVAL, "need k >= 0, dt > 0, dx > 0");
    if (o.mode != HEAT1D_MODE_MATCHED && o.mode != HEAT1D_MODE_FAST)
        return set_error(nullptr, HEAT1D_EINVAL, "bad mode");
    if (o.denominator != HEAT1D_DEN_DX2 && o.denominator != HEAT1D_DEN_PAPER_2DX)
        return set_error(nullptr, HEAT1D_EINVAL, "bad denominator");
    if (o.kernel != HEAT1D_KERNEL_AUTO && o.kernel != HEAT1D_KERNEL_NAIVE)
        return set_error(nullptr, HEAT1D_EINVAL, "bad kernel");
    if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks)
        return set_error(nullptr, HEAT1D_EINVAL, "bad rank %d / nranks %d", o.rank, o.nranks);
    if (o.nranks > 1 && !o.nccl_id) return set_error(nullptr, HEAT1D_EINVAL, "nranks > 1 needs nccl_id");
    if (o.virtual_slabs < 1) return set_error(nullptr, HEAT1D_EINVAL, "virtual_slabs must be >= 1");
    if (o.virtual_slabs > 1 && o.nranks > 1)
        return set_error(nullptr, HEAT1D_EUNSUPPORTED, "virtual_slabs > 1 needs nranks == 1");
    if (o.transport != HEAT1D_TRANSPORT_NCCL && o.transport != HEAT1D_TRANSPORT_P2P)
        return set_error(nullptr, HEAT1D_EINVAL, "bad transport");
    if (o.window_cells < 0) return set_error(nullptr, HEAT1D_EINVAL, "window_cells must be >= 0");
    if (o.window_cells > 0 && (o.nranks > 1 || o.virtual_slabs > 1 || o.kernel != HEAT1D_KERNEL_AUTO))
        return set_error(nullptr, HEAT1D_EUNSUPPORTED, "window_cells (streaming) needs one slab on one rank");
    if (o.T < 0 || o.T > HEAT1D_T_MAX) return set_error(nullptr, HEAT1D_EINVAL, "T must be in 0..%d", HEAT1D_T_MAX);
    const int G = o.virtual_slabs > 1 ? o.virtual_slabs : o.nranks;
    if (o.kernel == HEAT1D_KERNEL_NAIVE && G > 1)
        return set_error(nullptr, HEAT1D_EUNSUPPORTED, "the naive kernel is single-slab only");

    // r once on the host, fp64 (reading c4)
    const double r = (o.denominator == HEAT1D_DEN_DX2) ? (k * dt) / (dx * dx) : (k * dt) / (2.0 * dx);
    if (!std::isfinite(r)) return set_error(nullptr, HEAT1D_EINVAL, "r is not finite");
    if (r > 0.5 && !o.allow_unstable)
        return set_error(nullptr, HEAT1D_EUNSTABLE, "r = %.17g > 1/2 (CFL); set allow_unstable", r);

    const int64_t mslab = min_slab(nx, np, G);
    if (mslab == INT64_MAX) return set_error(nullptr, HEAT1D_EINVAL, "cannot split N=%lld into %d slabs",
                                             (long long)(nx * np), G);

    heat1d_t h = new heat1d_s();
    h->nx = nx;
    h->np = np;
    h->N = nx * np;
    h->nt_default = nt;
    h->k = k;
    h->dt = dt;
    h->dx = dx;
    h->r = r;
    h->mode = o.mode;
    h->den = o.denominator;
    h->kernel = o.kernel;
    h->rank = o.rank;
    h->nranks = o.nranks;
    h->blocking = o.blocking != 0;
    // Multi-rank runs do not capture NCCL calls into CUDA graphs: NCCL sets up its p2p
    // connections lazily (cudaMalloc/IPC, illegal under capture), and a pass there is long
    // (C4 at G=8: ~1.3 ms) next to its ~3 launches.
    h->use_graphs = o.use_graphs != 0 && o.nranks == 1 && o.transport != HEAT1D_TRANSPORT_P2P;
    h->window_cells = o.window_cells;
    h->transport = o.transport;  // (P2P pass arguments carry exchange indices: never replayed)
    // Matched mode: the 3-op form for r = 2^-j (j <= 7) or 0, else the 4-op form; both guarded
    // per block of steps, falling back to the literal sequence where they could differ from it
    // (stencil.cuh; DESIGN.md c3).  j <= 7 keeps the guard's bottom bound 2^(j T_MAX - 1022)
    // far below the values a ring holds.
    int r_exp = 0;
    if (r > 0.0) std::frexp(r, &r_exp);
    const bool pow2_ok = r == 0.0 || (is_pow2(r) && 1 - r_exp <= 7);
    h->ops = (o.mode == HEAT1D_MODE_FAST || pow2_ok) ? 3 : 4;
    // r == 0: fma(0, t, b) == b + 0*t == b for finite t (identity either way)
    // Fast mode works on the scaled state v = u / r^t (stencil.cuh, DESIGN.md §3 c21): 1 DP op per
    // update at r = 1/2, 2 for 1/256 <= r < 1/2 (the state grows by at most r^-T <= 2^512 within a
    // pass, T <= 64; select_fast_ops checks max|u0| against it).  Outside that range (tiny r,
    // unstable r > 1/2) the 3-op contracted form.
    if (o.mode == HEAT1D_MODE_FAST && o.kernel != HEAT1D_KERNEL_NAIVE) {
        if (r == 0.5)
            h->ops = 1;
        else if (r >= 1.0 / 256.0 && r < 0.5)
            h->ops = 2;
    }
    if (heat1d::ops_scaled(h->ops)) h->ops_fast = h->ops;
    // the scaled forms' per-step coefficient c = (1-2r)/r; the kernels fall back to the 3-op
    // form with r themselves when K5 finds max|u0| out of range (FastRange, kernels.h)
    h->q = heat1d::ops_scaled(h->ops) ? (1.0 - 2.0 * r) / r : r;
    auto bail = [&](int rc) {
        heat1d_destroy(h);
        return rc;
    };

    if (o.device >= 0) {
        cudaError_t e = cudaSetDevice(o.device);
        if (e != cudaSuccess) {
            set_error(nullptr, HEAT1D_ECUDA, "cudaSetDevice(%d): %s", o.device, cudaGetErrorString(e));
            delete h;
            return HEAT1D_ECUDA;
        }
    }
    if (cudaGetDevice(&h->device) != cudaSuccess) {
        delete h;
        return set_error(nullptr, HEAT1D_ECUDA, "no CUDA device");
    }
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);

    // Streams, and (several ranks) the NCCL communicator -- first, so that every decision
    // below that depends on a rank's own slab is agreed collectively before anything is
    // sized by it (T, pad, the kernel family).
    if (o.stream) {
        h->stream = static_cast<cudaStream_t>(o.stream);
    } else {
        if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
            set_error(nullptr, HEAT1D_ECUDA, "stream create");
            return bail(HEAT1D_ECUDA);
        }
        h->own_stream = true;
    }
    if (G > 1) {
        if (o.comm_stream) {
            h->comm = static_cast<cudaStream_t>(o.comm_stream);
        } else {
            if (cudaStreamCreateWithFlags(&h->comm, cudaStreamNonBlocking) != cudaSuccess) {
                set_error(nullptr, HEAT1D_ECUDA, "stream create");
                return bail(HEAT1D_ECUDA);
            }
            h->own_comm = true;
        }
        if (cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming) != cudaSuccess) {
            set_error(nullptr, HEAT1D_ECUDA, "event create");
            return bail(HEAT1D_ECUDA);
        }
    }
    if (o.nranks > 1) {
        ncclUniqueId id;
        memcpy(&id, o.nccl_id, sizeof id);
        ncclResult_t ne = ncclCommInitRank(&h->nccl, o.nranks, id, o.rank);
        if (ne != ncclSuccess) {
            h->nccl = nullptr;
            set_error(nullptr, HEAT1D_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(ne));
            return bail(HEAT1D_ENCCL);
        }
    }

    // T and the kernel family.  K2 passes: T from opts or auto_T, clamped to
    // the smallest slab (and half of it for the P2P edge strips) -- the same on every rank.
    int T = o.T > 0 ? o.T : auto_T(h->ops_fast ? h->ops_fast : h->ops, r);
    if (o.kernel == HEAT1D_KERNEL_NAIVE) T = 1;
    if (T > mslab) T = (int)mslab;  // a slab must hold its own halo
    if (o.transport == HEAT1D_TRANSPORT_P2P && G > 1) {
        if (mslab < 2) {  // 1-cell slabs: K3p's two strips would overlap
            o.transport = h->transport = HEAT1D_TRANSPORT_NCCL;
            h->use_graphs = o.use_graphs != 0 && o.nranks == 1;
        }
        else if (T > mslab / 2)
            T = (int)(mslab / 2);  // K3p's two strips must not overlap
    }
    // K6 (whole solve on chip) for one slab per rank when every rank's slab fits; its period
    // Tr is again the same on every rank, but "fits" depends on the rank's own slab: the ranks
    // vote (NCCL min-reduce) and all take the same family, T and pad.
    bool res_multi = false;
    const bool res_ok = ((G == 1) || (o.nranks > 1 && o.virtual_slabs == 1)) && o.kernel == HEAT1D_KERNEL_AUTO &&
                        o.resident != 0 && o.window_cells == 0;
    if (res_ok) {
        int64_t f0 = 0, n0 = h->N;
        if (G > 1) partition(nx, np, G, o.rank, &f0, &n0);
        // K6 period (halo refresh) <= 128; auto: 40..64 by k6_auto_T (T = 32 pays twice the
        // hand-offs for -30 %, profiles/r01_k6_period_sync.jsonl; T = 96/128 needs V = 49 spans,
        // -25 %, profiles/r01_k6_period_v.jsonl)
        int Tr = o.T > 0 ? std::min(o.T, 128) : 64;
        if (Tr > mslab) Tr = (int)mslab;
        if (o.T == 0) Tr = k6_auto_T(h, nx, np, G, nt, mslab);
        int coop = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device);
        bool fits = coop && n0 <= heat1d::resident_capacity(Tr, h->num_sms) && n0 >= Tr &&
                    heat1d::resident_fits(h->ops, n0, Tr, h->num_sms, G > 1) &&
                    (!h->ops_fast || heat1d::resident_fits(h->ops_fast, n0, Tr, h->num_sms, G > 1));
        cudaGetLastError();
        if (o.nranks > 1) {
            int all = 0;
            int rc = vote_min(h, fits ? 1 : 0, &all);
            if (rc) {
                set_error(nullptr, rc, "resident vote: %s", h->last_error.c_str());
                return bail(rc);
            }
            fits = all != 0;
        }
        if (fits) {
            T = Tr;
            if (G > 1)
                res_multi = true;  // mailboxes mapped below
            else
                h->resident = true;
        } else if (o.resident == 1) {
            set_error(nullptr, HEAT1D_EUNSUPPORTED, "a slab of %lld cells does not fit the resident kernel%s",
                      (long long)n0, o.nranks > 1 ? " (on some rank)" : "");
            return bail(HEAT1D_EUNSUPPORTED);
        }
    } else if (o.resident == 1) {
        set_error(nullptr, HEAT1D_EUNSUPPORTED, "resident kernel needs one slab on one rank");
        return bail(HEAT1D_EUNSUPPORTED);
    }
    h->T = T;
    h->pad = pad_for(T);

    // slabs
    const int ns = o.virtual_slabs;
    int64_t total = 0;
    for (int g = 0; g < ns; ++g) {
        Slab s;
        const int idx = (ns > 1) ? g : o.rank;
        partition(nx, np, G, idx, &s.first, &s.count);
        h->slabs.push_back(s);
        total += o.window_cells > 0 ? 3 * 2 * round_up(o.window_cells + 2 * h->pad, 32)
                                    : 2 * round_up(s.count + 2 * h->pad, 32);
    }
    h->first = h->slabs.front().first;
    h->count = 0;
    for (auto &s : h->slabs) h->count += s.count;

    if (o.dev_buf) {  // caller-owned device memory (>= heat1d_buffer_len doubles, 256-B aligned)
        if (reinterpret_cast<uintptr_t>(o.dev_buf) % 256) {
            set_error(nullptr, HEAT1D_EINVAL, "dev_buf must be 256-byte aligned");
            return bail(HEAT1D_EINVAL);
        }
        h->alloc = o.dev_buf;
        h->own_alloc = false;
    } else {
        cudaError_t e = cudaMalloc(&h->alloc, (size_t)total * sizeof(double));
        if (e != cudaSuccess) {
            cudaGetLastError();
            set_error(nullptr, HEAT1D_ENOMEM, "cudaMalloc(%lld bytes): %s", (long long)total * 8,
                      cudaGetErrorString(e));
            return bail(HEAT1D_ENOMEM);
        }
    }
    double *p = static_cast<double *>(h->alloc);
    for (auto &s : h->slabs) {
        const int64_t len = o.window_cells > 0 ? 3 * round_up(o.window_cells + 2 * h->pad, 32)
                                               : round_up(s.count + 2 * h->pad, 32);
        h->buf_len = len;
        s.buf[0] = p;
        s.buf[1] = p + len;
        p += 2 * len;
    }

    if (o.nranks > 1) {
        // one warm-up exchange (contents irrelevant: the first pass's exchange overwrites the
        // pads) so NCCL's p2p connections exist before the first timed pass and a broken
        // transport fails here, at create
        int rc = exchange(h, h->T);
        if (rc == HEAT1D_OK && cudaStreamSynchronize(h->comm) != cudaSuccess) rc = HEAT1D_ECUDA;
        if (rc) {
            set_error(nullptr, rc, "warm-up halo exchange failed: %s", h->last_error.c_str());
            return bail(rc);
        }
        if (res_multi) {
            rc = setup_multi_resident(h);
            if (rc) {
                set_error(nullptr, rc, "multi-rank resident setup: %s", h->last_error.c_str());
                return bail(rc);
            }
            if (!h->resident && o.resident == 1) {  // (agreed: every rank sees the same outcome)
                set_error(nullptr, HEAT1D_EUNSUPPORTED, "resident kernel across ranks needs peer access");
                return bail(HEAT1D_EUNSUPPORTED);
            }
        }
    }
    if (h->transport == HEAT1D_TRANSPORT_P2P && h->multi() && !h->resident) {
        int rc = setup_p2p(h, nx, np);
        if (rc) {
            set_error(nullptr, rc, "transport p2p setup: %s", h->last_error.c_str());
            return bail(rc);
        }
    }
    if (h->resident && h->nranks == 1 && getenv("HEAT1D_K6_MAILBOX") && atoi(getenv("HEAT1D_K6_MAILBOX")) == 1 &&
        heat1d::resident_fits(h->ops, h->N, h->T, h->num_sms, true) &&
        (!h->ops_fast || heat1d::resident_fits(h->ops_fast, h->N, h->T, h->num_sms, true))) {
        // test knob: route the single rank's wrap through its own mailbox (the multi-rank protocol)
        if (cudaMalloc(&h->mbox, heat1d::MBOX_BYTES) != cudaSuccess ||
            heat1d::launch_mbox_init(h->mbox, h->stream) != cudaSuccess ||
            cudaStreamSynchronize(h->stream) != cudaSuccess) {
            cudaGetLastError();
            set_error(nullptr, HEAT1D_ENOMEM, "mailbox");
            return bail(HEAT1D_ENOMEM);
        }
        h->mbox_left = h->mbox_right = h->mbox;
    }
    if (const char *dl = getenv("HEAT1D_COMM_DELAY_US")) h->comm_delay_us = (unsigned)atoi(dl);
    if (const char *k0 = getenv("HEAT1D_K6_COUNTER0")) {  // test hook: K6 tag / exchange counters start
        h->k6_tag = h->k6_base = (unsigned)strtoul(k0, nullptr, 0);  // here (near 2^32: the wrap path)
        if (h->k6_tag == 0) h->k6_tag = 1;
    }
    if (const char *pp = getenv("HEAT1D_POISON_PADS")) h->poison_pads = atoi(pp) == 1;
    // HEAT1D_GEOM (tuning knob) only where the pass kernel exists for every arithmetic variant
    // this handle may run (its matched/fast form and the 3-op fallback); else the default
    if (!parse_geom_env(&h->geom) || !heat1d::pass_supported(h->geom, h->ops) ||
        (h->ops_fast && !heat1d::pass_supported(h->geom, h->ops_fast)) || !heat1d::pass_supported(h->geom, 3))
        h->geom = heat1d::choose_geom(h->slabs[0].count, h->T, h->num_sms, h->ops_fast ? h->ops_fast : h->ops);
    if (h->ops_fast && cudaMalloc(&h->absmax, sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        set_error(nullptr, HEAT1D_ENOMEM, "absmax word");
        return bail(HEAT1D_ENOMEM);
    }
    if (h->resident && !h->res_scratch) {
        if (cudaMalloc(&h->res_scratch, heat1d::resident_scratch_bytes(h->T, h->num_sms)) != cudaSuccess) {
            cudaGetLastError();
            set_error(nullptr, HEAT1D_ENOMEM, "resident scratch");
            return bail(HEAT1D_ENOMEM);
        }
        if (heat1d::resident_scratch_init(h->res_scratch, h->T, h->num_sms, h->stream) != cudaSuccess ||
            cudaStreamSynchronize(h->stream) != cudaSuccess) {
            cudaGetLastError();
            set_error(nullptr, HEAT1D_ECUDA, "resident scratch init");
            return bail(HEAT1D_ECUDA);
        }
    }
    *out = h;
    return HEAT1D_OK;
}

int heat1d_local_range(heat1d_t h, int64_t *first, int64_t *count) {
    if (!h || !first || !count) return HEAT1D_EINVAL;
    *first = h->first;
    *count = h->count;
    return HEAT1D_OK;
}

// Fast mode: the scaled state of a pass reaches at most max|u0| * r^-T (max principle,
// r <= 1/2).  K5 writes max|u0| to a device word; the scaled kernels compare it with their
// limit themselves (FastRange) and run the 3-op form if it is out of range -- no host round
// trip, so a non-blocking set_initial only enqueues.
static int check_fast_range(heat1d_t h) {
    if (!h->ops_fast) return HEAT1D_OK;
    CK(cudaMemsetAsync(h->absmax, 0, sizeof(unsigned long long), h->stream));
    for (const Slab &s : h->slabs) {
        CK(heat1d::launch_absmax(cell0(h, s, h->cur), s.count, h->absmax, h->stream));
        h->launches++;
    }
    return HEAT1D_OK;
}

static int after_initial(heat1d_t h) {
    if (h->multi() && h->nranks == 1 && h->poison_pads) {
        // fault injection (tests): NaN in every ghost pad of both buffers -- any pad value
        // read before the exchange refreshed it would poison the result
        for (const Slab &s : h->slabs)
            for (int b = 0; b < 2; ++b) {
                CK(cudaMemsetAsync(s.buf[b], 0xff, (size_t)h->pad * 8, h->stream));
                CK(cudaMemsetAsync(cell0(h, s, b) + s.count, 0xff, (size_t)h->pad * 8, h->stream));
            }
    }
    if (!h->multi() && !h->resident) {
        const Slab &s = h->slabs[0];
        CK(heat1d::launch_wrap_fill(cell0(h, s, h->cur), s.count, h->pad, h->stream));
        h->launches++;
    }
    int rc = check_fast_range(h);
    if (rc) return rc;
    // blocking handles return with the copy done (the caller may reuse u0 at once); non-blocking
    // ones only enqueue it on the stream
    if (h->blocking) CK(cudaStreamSynchronize(h->stream));
    h->initialized = true;
    h->steps_done = 0;
    return HEAT1D_OK;
}

int heat1d_set_initial(heat1d_t h, const double *u0, int64_t count) {
    int rc = guard(h);
    if (rc) return rc;
    if (h->window_cells)
        return set_error(h, HEAT1D_EUNSUPPORTED, "streaming handle (window_cells): use heat1d_solve_host");
    if (!u0) return set_error(h, HEAT1D_EINVAL, "u0 is NULL");
    if (count != h->count)
        return set_error(h, HEAT1D_EINVAL, "count %lld != local slab %lld", (long long)count, (long long)h->count);
    int64_t off = 0;
    for (const Slab &s : h->slabs) {
        CK(cudaMemcpyAsync(cell0(h, s, h->cur), u0 + off, (size_t)s.count * 8, cudaMemcpyDefault, h->stream));
        off += s.count;
    }
    return after_initial(h);
}

int heat1d_init_uniform(heat1d_t h, uint64_t seed, double lo, double hi) {
    int rc = guard(h);
    if (rc) return rc;
    if (h->window_cells)
        return set_error(h, HEAT1D_EUNSUPPORTED, "streaming handle (window_cells): use heat1d_solve_host");
    if (!std::isfinite(lo) || !std::isfinite(hi)) return set_error(h, HEAT1D_EINVAL, "lo/hi not finite");
    for (const Slab &s : h->slabs) {
        CK(heat1d::launch_init_uniform(cell0(h, s, h->cur), s.count, s.first, seed, lo, hi, h->stream));
        h->launches++;
    }
    return after_initial(h);
}

int heat1d_run(heat1d_t h, int64_t nt) {
    int rc = guard(h);
    if (rc) return rc;
    if (h->window_cells)
        return set_error(h, HEAT1D_EUNSUPPORTED, "streaming handle (window_cells): use heat1d_solve_host");
    if (!h->initialized) return set_error(h, HEAT1D_ESTATE, "run before set_initial");
    if (nt < 0) nt = h->nt_default;
    if (nt == 0) return HEAT1D_OK;
    rc = run_maybe_graph(h, nt);
    if (rc) return rc;
    if (h->blocking) {
        CK(cudaStreamSynchronize(h->stream));
        if (h->nccl) {  // a peer's failure surfaces asynchronously on the communicator
            ncclResult_t ae = ncclSuccess;
            NK(ncclCommGetAsyncError(h->nccl, &ae));
            if (ae != ncclSuccess) return fail_nccl(h, ae, "ncclCommGetAsyncError", __LINE__);
        }
        if (h->prof) {
            rc = prof_collect(h);
            if (rc) return rc;
        }
    }
    return HEAT1D_OK;
}

int heat1d_get(heat1d_t h, double *out, int64_t count) {
    int rc = guard(h);
    if (rc) return rc;
    if (h->window_cells)
        return set_error(h, HEAT1D_EUNSUPPORTED, "streaming handle (window_cells): use heat1d_solve_host");
    if (!out) return set_error(h, HEAT1D_EINVAL, "out is NULL");
    if (!h->initialized) return set_error(h, HEAT1D_ESTATE, "get before set_initial");
    if (count != h->count)
        return set_error(h, HEAT1D_EINVAL, "count %lld != local slab %lld", (long long)count, (long long)h->count);
    int64_t off = 0;
    for (const Slab &s : h->slabs) {
        CK(cudaMemcpyAsync(out + off, cell0(h, s, h->cur), (size_t)s.count * 8, cudaMemcpyDefault, h->stream));
        off += s.count;
    }
    if (h->blocking) CK(cudaStreamSynchronize(h->stream));
    return HEAT1D_OK;
}

// ------------------------------------------------------------------ heat1d_solve_host
namespace {

// Copy ring cells [a, a+len) (indices mod n, at most one wrap per side) host -> device.
// Copy slab cells [a, a+len) to dst, a >= -H and a+len <= n+H: cells < 0 come from `left`
// (the H cells preceding the slab, left[H-1] next to cell 0), cells >= n from `right` (the H
// cells following it); host or device pointers.  For one slab that is the whole ring,
// left = u0 + n - H and right = u0 (the periodic wrap).
int copy_window_in(heat1d_t h, double *dst, const double *u0, const double *left, const double *right, int64_t H,
                   int64_t n, int64_t a, int64_t len) {
    int64_t done = 0;
    while (done < len) {
        const int64_t g = a + done;
        const double *src;
        int64_t run;
        if (g < 0) {
            src = left + (H + g);
            run = std::min(len - done, -g);
        } else if (g < n) {
            src = u0 + g;
            run = std::min(len - done, n - g);
        } else {
            src = right + (g - n);
            run = len - done;
        }
        CK(cudaMemcpyAsync(dst + done, src, (size_t)run * 8, cudaMemcpyDefault, h->st_h2d));
        done += run;
    }
    return HEAT1D_OK;
}

// nt steps of one light-cone window X[0, Lw) on the compute stream (ping-pong with Y);
// pass p writes only the cells still inside the cone.  Returns the result buffer.
int solve_window(heat1d_t h, int ops, double *X, double *Y, int64_t Lw, int64_t nt, double **res,
                 const unsigned long long *range_word) {
    const double q = heat1d::ops_scaled(ops) ? (1.0 - 2.0 * h->r) / h->r : h->r;
    double *a = X, *b = Y;
    int64_t done = 0;
    while (done < nt) {
        const int Tp = (int)std::min<int64_t>(h->T, nt - done);
        int grid = 0;
        CK(heat1d::launch_pass(h->geom, ops, a, b, Lw, Tp, done + Tp, Lw - done - Tp, 0, q,
                               heat1d::scale_of(h->r, Tp), guard_for(h, ops, Tp), fast_range(h, ops, range_word),
                               h->num_sms, h->stream, &grid));
        h->launches++;
        std::swap(a, b);
        done += Tp;
    }
    *res = a;
    return HEAT1D_OK;
}

int ensure_stream_objects(heat1d_t h, int64_t nwin) {
    if (!h->st_h2d) CK(cudaStreamCreateWithFlags(&h->st_h2d, cudaStreamNonBlocking));
    if (!h->st_d2h) CK(cudaStreamCreateWithFlags(&h->st_d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 3; ++i) {
        if (!h->ev_in[i]) CK(cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming));
        if (!h->ev_comp[i]) CK(cudaEventCreateWithFlags(&h->ev_comp[i], cudaEventDisableTiming));
        if (!h->ev_out[i]) CK(cudaEventCreateWithFlags(&h->ev_out[i], cudaEventDisableTiming));
    }
    if (h->win_absmax_n < nwin) {
        if (h->win_absmax) CK(cudaFree(h->win_absmax));
        h->win_absmax = nullptr;
        h->win_absmax_n = 0;
        CK(cudaMalloc(&h->win_absmax, (size_t)nwin * sizeof(unsigned long long)));
        h->win_absmax_n = nwin;
    }
    return HEAT1D_OK;
}

constexpr int kWinSlots = 3;  // light-cone window slots per ping-pong buffer (heat1d_solve_host)

// Window plan: C chunks of L cells, windows of L + 2H cells (H = nt), two slots of two
// ping-pong buffers carved out of the handle's two ring buffers.  false = not worth it.
bool stream_plan(heat1d_t h, int64_t nt, int64_t *C, int64_t *L, int64_t *half) {
    if (h->slabs.size() > 1 || h->resident || h->kernel == HEAT1D_KERNEL_NAIVE || nt < 1) return false;
    const int64_t n = h->slabs[0].count;
    // a window's halos come from at most one neighbour slab (or one wrap) per side
    if (nt > n) return false;
    *half = h->buf_len / kWinSlots / 32 * 32;  // window slots per ping-pong buffer
    const int64_t lw_max = *half - 2 * h->pad;
    const int64_t lmax = lw_max - 2 * nt;
    if (lmax < 16 * nt || lmax < 4096) return false;
    // up to 16 windows when the ring allows (pipeline fill + drain ~ 2/C of the transfers)
    int64_t c = (n + lmax - 1) / lmax;
    while (c < 16 && (n / (c + 1)) >= 16 * nt && n / (c + 1) >= (int64_t)1 << 22) ++c;
    *C = c;
    *L = (n + c - 1) / c;
    return *L + 2 * nt <= lw_max;
}

// The streamed solve of this handle's single slab given its nt-deep neighbour halos
// (stream_plan must have succeeded).
int solve_windows(heat1d_t h, const double *u0, const double *left, const double *right, int64_t nt, double *out,
                  int64_t C, int64_t L, int64_t half) {
    int rc = ensure_stream_objects(h, C);
    if (rc) return rc;
    const Slab &s = h->slabs[0];
    const int64_t n = s.count;
    const int ops = h->ops;  // (scaled fast forms check each window's own max|u0|: FastRange)
    // three window slots: the H2D of window c+1, the compute of window c and the D2H of
    // window c-1 each own one, so the three run fully concurrently (two slots serialise
    // a D2H before the next H2D into the same slot)
    double *X[kWinSlots], *Y[kWinSlots];
    for (int k = 0; k < kWinSlots; ++k) {
        X[k] = s.buf[0] + k * half + h->pad;
        Y[k] = s.buf[1] + k * half + h->pad;
    }
    h->initialized = false;  // the ring buffers now hold windows
    if (h->ops_fast) CK(cudaMemsetAsync(h->win_absmax, 0, (size_t)C * 8, h->stream));
    CK(cudaEventRecord(h->ev_comp[0], h->stream));  // memset before any K5
    CK(cudaStreamWaitEvent(h->st_h2d, h->ev_comp[0], 0));
    for (int64_t c = 0; c < C; ++c) {
        const int sl = (int)(c % kWinSlots);
        const int64_t a = c * L, len = std::min(L, n - a), Lw = len + 2 * nt;
        if (c >= kWinSlots) CK(cudaStreamWaitEvent(h->st_h2d, h->ev_out[sl], 0));  // slot free again
        rc = copy_window_in(h, X[sl], u0, left, right, nt, n, a - nt, Lw);
        if (rc) return rc;
        CK(cudaEventRecord(h->ev_in[sl], h->st_h2d));
        CK(cudaStreamWaitEvent(h->stream, h->ev_in[sl], 0));
        if (h->ops_fast) {
            CK(heat1d::launch_absmax(X[sl], Lw, h->win_absmax + c, h->stream));
            h->launches++;
        }
        double *res = nullptr;
        rc = solve_window(h, ops, X[sl], Y[sl], Lw, nt, &res, h->ops_fast ? h->win_absmax + c : nullptr);
        if (rc) return rc;
        CK(cudaEventRecord(h->ev_comp[sl], h->stream));
        CK(cudaStreamWaitEvent(h->st_d2h, h->ev_comp[sl], 0));
        CK(cudaMemcpyAsync(out + a, res + nt, (size_t)len * 8, cudaMemcpyDefault, h->st_d2h));
        CK(cudaEventRecord(h->ev_out[sl], h->st_d2h));
    }
    CK(cudaStreamSynchronize(h->st_h2d));
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaStreamSynchronize(h->st_d2h));
    h->steps_done = nt;
    h->stream_windows = C;
    return HEAT1D_OK;
}

int solve_checks(heat1d_t h, const double *u0, int64_t count, double *out) {
    if (!u0 || !out) return set_error(h, HEAT1D_EINVAL, "u0/out is NULL");
    if (count != h->count)
        return set_error(h, HEAT1D_EINVAL, "count %lld != local slab %lld", (long long)count, (long long)h->count);
    if (out < u0 + count && u0 < out + count)  // the last windows re-read u0 after early chunks are written
        return set_error(h, HEAT1D_EINVAL, "u0 and out must not overlap");
    return HEAT1D_OK;
}

}  // namespace

int heat1d_solve_host(heat1d_t h, const double *u0, int64_t count, int64_t nt, double *out) {
    int rc = guard(h);
    if (rc) return rc;
    if ((rc = solve_checks(h, u0, count, out))) return rc;
    if (nt < 0) nt = h->nt_default;
    int64_t C = 0, L = 0, half = 0;
    bool plan = stream_plan(h, nt, &C, &L, &half);
    if (h->nranks > 1) {
        // every rank must take the same branch (the plain sequence exchanges halos every pass)
        int *d = nullptr;
        int v = plan ? 1 : 0;
        CK(cudaMalloc(&d, sizeof(int)));
        CK(cudaMemcpy(d, &v, sizeof v, cudaMemcpyHostToDevice));
        NK(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, h->nccl, h->comm));
        CK(cudaMemcpyAsync(&v, d, sizeof v, cudaMemcpyDeviceToHost, h->comm));
        CK(cudaStreamSynchronize(h->comm));
        CK(cudaFree(d));
        plan = v != 0;
    }
    if (!plan) {  // the plain sequence
        if (h->window_cells)
            return set_error(h, HEAT1D_EUNSUPPORTED,
                             "streaming needs window_cells >= 18 nt and nt <= ring cells (window %lld, nt %lld, N %lld)",
                             (long long)h->window_cells, (long long)nt, (long long)count);
        rc = heat1d_set_initial(h, u0, count);
        if (!rc) rc = heat1d_run(h, nt);
        if (!rc) rc = heat1d_get(h, out, count);
        if (!rc && !h->blocking) CK(cudaStreamSynchronize(h->stream));  // out is filled on return
        return rc;
    }
    if (h->nranks == 1)  // one slab = the whole ring: the halos are its own ends (periodic wrap)
        return solve_windows(h, u0, u0 + (count - nt), u0, nt, out, C, L, half);
    // several ranks: ONE exchange of nt-deep halos (the light cone of the whole solve), then
    // every rank streams its windows with no further communication
    // staging in device memory (u0 is a host array): hb = [left halo (nt) | the slab's first nt
    // cells | gap | its last nt cells | right halo (nt)] laid out so that the plan's offsets
    // apply unchanged with "cell 0" at hb + nt and a virtual slab of 3 nt cells
    heat1d_exchange_plan pl;
    make_plan(3 * nt, nt, h->rank, h->nranks, &pl);
    double *hb = nullptr;
    CK(cudaMalloc(&hb, (size_t)5 * nt * sizeof(double)));
    double *c0 = hb + nt;
    CK(cudaMemcpyAsync(c0 + pl.send_left_off, u0, (size_t)nt * 8, cudaMemcpyDefault, h->comm));
    CK(cudaMemcpyAsync(c0 + pl.send_right_off, u0 + (count - nt), (size_t)nt * 8, cudaMemcpyDefault, h->comm));
    NK(issue_plan(pl, c0, c0, h->nccl, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    rc = solve_windows(h, u0, c0 + pl.recv_left_off, c0 + pl.recv_right_off, nt, out, C, L, half);
    if (rc) {
        cudaFree(hb);
        return rc;
    }
    // leave together: the windows occupy the slab buffers, pads included, which a neighbour's
    // next run would start pushing edges into (P2P transport)
    NK(ncclAllReduce(hb, hb, 1, ncclDouble, ncclSum, h->nccl, h->comm));
    CK(cudaStreamSynchronize(h->comm));
    CK(cudaFree(hb));
    return HEAT1D_OK;
}

int heat1d_solve_host_halo(heat1d_t h, const double *u0, const double *left, const double *right, int64_t count,
                           int64_t nt, double *out) {
    int rc = guard(h);
    if (rc) return rc;
    if ((rc = solve_checks(h, u0, count, out))) return rc;
    if (!left || !right) return set_error(h, HEAT1D_EINVAL, "left/right halo is NULL");
    if (nt < 0) nt = h->nt_default;
    int64_t C = 0, L = 0, half = 0;
    if (!stream_plan(h, nt, &C, &L, &half))
        return set_error(h, HEAT1D_EUNSUPPORTED, "slab of %lld cells too small for light-cone windows of nt=%lld",
                         (long long)count, (long long)nt);
    return solve_windows(h, u0, left, right, nt, out, C, L, half);
}

int64_t heat1d_steps_done(heat1d_t h) { return h ? h->steps_done : -1; }

int heat1d_info(heat1d_t h, heat1d_info_t *info) {
    if (!h || !info) return HEAT1D_EINVAL;
    if (info->size != sizeof(heat1d_info_t)) return HEAT1D_EINVAL;
    info->T = h->T;
    info->mode = h->mode;
    info->denominator = h->den;
    info->kernel = h->kernel;
    info->dp_ops = h->ops;
    info->nslabs = (int32_t)h->slabs.size();
    info->rank = h->rank;
    info->nranks = h->nranks;
    info->device = h->device;
    info->r = h->r;
    info->N = h->N;
    info->first = h->first;
    info->count = h->count;
    info->steps_done = h->steps_done;
    info->launches = h->launches;
    info->pad = h->pad;
    info->tile_cells = (int32_t)h->geom.tile_out(h->T);
    info->grid = h->last_grid;
    info->pass_kind = h->geom.kind;
    info->pass_V = h->geom.V;
    info->pass_NW = h->geom.NW;
    info->pass_S = h->geom.S;
    info->resident = h->resident ? 1 : 0;
    info->resident_warps = h->res_warps;
    info->resident_V = h->res_V;
    info->pass_feed = heat1d::pass_uses_feed(h->geom, h->ops_fast ? h->ops_fast : h->ops, h->T) ? 1 : 0;
    info->stream_windows = h->stream_windows;
    info->transport = h->transport;
    return HEAT1D_OK;
}

int heat1d_set_profiling(heat1d_t h, int on) {
    int rc = guard(h);
    if (rc) return rc;
    rc = prof_collect(h);
    if (rc) return rc;
    h->prof = on != 0;
    h->prof_ms = 0.0;
    h->prof_launches = 0;
    h->trace.clear();
    if (h->prof) {
        if (!h->prof_t0) CK(cudaEventCreate(&h->prof_t0));
        CK(cudaEventRecord(h->prof_t0, h->stream));
    }
    return HEAT1D_OK;
}

int heat1d_profile(heat1d_t h, int64_t *launches, double *ms) {
    int rc = guard(h);
    if (rc) return rc;
    rc = prof_collect(h);
    if (rc) return rc;
    if (launches) *launches = h->prof_launches;
    if (ms) *ms = h->prof_ms;
    return HEAT1D_OK;
}

int heat1d_trace(heat1d_t h, heat1d_trace_event *events, int64_t cap, int64_t *count) {
    int rc = guard(h);
    if (rc) return rc;
    if (!count || (cap > 0 && !events)) return set_error(h, HEAT1D_EINVAL, "trace: NULL output");
    rc = prof_collect(h);
    if (rc) return rc;
    const int64_t n = (int64_t)h->trace.size();
    for (int64_t i = 0; i < n && i < cap; ++i) events[i] = h->trace[(size_t)i];
    *count = n;
    return HEAT1D_OK;
}

void *heat1d_stream(heat1d_t h) { return h ? (void *)h->stream : nullptr; }

int heat1d_destroy(heat1d_t h) {
    if (!h) return HEAT1D_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->comm) cudaStreamSynchronize(h->comm);
    const bool peers = h->peer_open[0] || h->peer_open[1] || h->peer_open[2] || h->peer_open[3] ||
                       h->mbox_ipc_left || h->mbox_ipc_right;
    if (h->nccl && peers && !h->poisoned) {
        // collective: a neighbour's last edge kernel may still be putting into this rank's
        // pads (it writes ahead of any wait of ours), so nobody unmaps or frees until every
        // rank's streams are idle
        int *d = nullptr;
        if (cudaMalloc(&d, sizeof(int)) == cudaSuccess) {
            cudaMemsetAsync(d, 0, sizeof(int), h->comm);
            if (ncclAllReduce(d, d, 1, ncclInt32, ncclSum, h->nccl, h->comm) == ncclSuccess) {
                // a rank that never destroys (it died, or leaked its handle) must not hang the
                // others forever: give up after 30 s and abort the communicator
                const auto t0 = std::chrono::steady_clock::now();
                while (cudaStreamQuery(h->comm) == cudaErrorNotReady) {
                    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30)) {
                        ncclCommAbort(h->nccl);
                        h->nccl = nullptr;
                        break;
                    }
                    std::this_thread::sleep_for(std::chrono::microseconds(50));
                }
            }
            if (h->nccl) cudaFree(d);  // (after an abort the stream may still hold the reduce)
        }
        cudaGetLastError();
    }
    if (h->nccl) ncclCommDestroy(h->nccl);
    for (auto &g : h->graphs) cudaGraphExecDestroy(g.exec);
    for (cudaEvent_t e : h->ev_all) cudaEventDestroy(e);
    if (h->prof_t0) cudaEventDestroy(h->prof_t0);
    if (h->ev_ready) cudaEventDestroy(h->ev_ready);
    if (h->ev_halo) cudaEventDestroy(h->ev_halo);
    if (h->own_comm && h->comm) cudaStreamDestroy(h->comm);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    if (h->alloc && h->own_alloc) cudaFree(h->alloc);
    if (h->res_scratch) cudaFree(h->res_scratch);
    if (h->absmax) cudaFree(h->absmax);
    if (h->mbox_ipc_left) cudaIpcCloseMemHandle(h->mbox_left);
    if (h->mbox_ipc_right) cudaIpcCloseMemHandle(h->mbox_right);
    if (h->mbox) cudaFree(h->mbox);
    for (int i = 0; i < 4; ++i)
        if (h->peer_open[i]) cudaIpcCloseMemHandle(i % 2 == 0 ? h->peer_alloc[i / 2] : h->peer_flags[i / 2]);
    if (h->xflags) cudaFree(h->xflags);
    if (h->win_absmax) cudaFree(h->win_absmax);
    for (int i = 0; i < 3; ++i) {
        if (h->ev_in[i]) cudaEventDestroy(h->ev_in[i]);
        if (h->ev_comp[i]) cudaEventDestroy(h->ev_comp[i]);
        if (h->ev_out[i]) cudaEventDestroy(h->ev_out[i]);
    }
    if (h->st_h2d) cudaStreamDestroy(h->st_h2d);
    if (h->st_d2h) cudaStreamDestroy(h->st_d2h);
    delete h;
    return HEAT1D_OK;
}

const char *heat1d_last_error(heat1d_t h) { return h ? h->last_error.c_str() : g_create_error.c_str(); }

}  // extern "C"
