/*
 * heat1d.h -- C ABI of libheat1d, a B200 (sm_100a) implementation of the
 * explicit forward-Euler, 3-point finite-difference update of the 1D heat
 * equation on a periodic ring of fp64 cells (arxiv 2307.01117, §2):
 *
 *     u(t+dt, x_i) = u(t,x_i) + dt*k*(u(t,x_{i-1}) - 2u(t,x_i) + u(t,x_{i+1})) / D
 *
 * (Eq. 2), grid x_i = i*dx, i = 0..N-1,
 * periodic boundary u(t,x) = u(t,L+x), D = dx^2 by default
 * (reading c1; the literal "2h" of PAPER.md:68 is HEAT1D_DEN_PAPER_2DX).
 * The ring is cut into np partitions of nx cells (N = nx*np) whose ghost
 * zones are exchanged between neighbours; here the ring is cut
 * into contiguous slabs, one per GPU rank, exchanging depth-T halos every T
 * steps (the edge kernel's own puts into the neighbour's ghost pads over NVLink
 * peer memory, or NCCL send/recv), and each GPU advances T steps per HBM pass.
 *
 * Conventions
 *   - All functions return int status (heat1d_status) unless stated.
 *   - Pointers are plain host (pageable or pinned) or device pointers; copies
 *     use cudaMemcpyDefault (unified addressing).  No torch types cross this
 *     boundary.
 *   - Arithmetic (reading c3): r = (k*dt)/(dx*dx) once on the host;
 *     every update is v = b + r*((a - 2b) + c), a=u[i-1], b=u[i], c=u[i+1],
 *     binary64 RNE.  HEAT1D_MODE_MATCHED evaluates exactly that sequence (the
 *     result is bitwise independent of T, np, the slab count and the GPU
 *     count, and bitwise equal to the CPU oracle); HEAT1D_MODE_FAST evaluates
 *     the algebraically equal form u' = (1-2r)u_i + r(u_{i-1}+u_{i+1}) on the
 *     scaled state v = u/r^t (one fp64 add per update at r = 1/2, add + fma
 *     for 1/256 <= r < 1/2, rescaled once per T-step pass; else the contracted
 *     3-op form), error <= 1e-12*max|u0|*nt (BASELINE.json north_star).
 *   - Threading: one host thread per handle.  A handle whose CUDA or NCCL
 *     call failed is "poisoned": every later call except heat1d_destroy
 *     returns the same error.
 */
#ifndef HEAT1D_H
#define HEAT1D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HEAT1D_VERSION 10000 /* 1.0.0 */

#if defined(__GNUC__)
#define HEAT1D_API __attribute__((visibility("default")))
#else
#define HEAT1D_API
#endif

typedef struct heat1d_s *heat1d_t; /* opaque; one per rank (per GPU) */

typedef enum {
    HEAT1D_OK = 0,
    HEAT1D_EINVAL = 1,       /* bad argument: sizes, non-finite k/dt/dx, count mismatch, ranks */
    HEAT1D_EUNSTABLE = 2,    /* r > 1/2 without allow_unstable               */
    HEAT1D_ESTATE = 3,       /* run/get before set_initial, or use of a poisoned handle         */
    HEAT1D_ENOMEM = 4,       /* device allocation failed                                        */
    HEAT1D_ECUDA = 5,        /* CUDA runtime / kernel error (handle poisoned)                   */
    HEAT1D_ENCCL = 6,        /* NCCL error (handle poisoned)                                    */
    HEAT1D_EUNSUPPORTED = 7  /* valid request this build does not implement                     */
} heat1d_status;

enum { HEAT1D_MODE_MATCHED = 0, HEAT1D_MODE_FAST = 1 };
enum { HEAT1D_DEN_DX2 = 0, HEAT1D_DEN_PAPER_2DX = 1 };
enum {
    HEAT1D_KERNEL_AUTO = 0,   /* temporal-blocked TMA pass kernel (K2)                        */
    HEAT1D_KERNEL_NAIVE = 1   /* one step per launch, modular indexing (K1; T forced to 1)    */
};

enum {
    HEAT1D_TRANSPORT_NCCL = 0, /* halo exchange of several slabs: ncclSend/ncclRecv (ranks) or
                                  device copies (virtual slabs), then the edge kernel K3      */
    HEAT1D_TRANSPORT_P2P = 1   /* K3 itself puts its new edge strips into the neighbours' ghost
                                  pads (NVLink peer memory via CUDA IPC for ranks) and releases
                                  a system-scope flag the neighbour's next K3 acquires        */
};

#define HEAT1D_T_MAX 128

/* Options.  Always initialise with heat1d_opts_default(); `size` versions the struct. */
typedef struct {
    uint32_t size;          /* = sizeof(heat1d_opts)                                        */
    int32_t device;         /* CUDA ordinal; -1 = the calling thread's current device       */
    int32_t rank, nranks;   /* position in the GPU ring; (0,1) = single GPU                 */
    const void *nccl_id;    /* 128-byte ncclUniqueId from heat1d_get_unique_id on rank 0;
                               required iff nranks > 1                                      */
    int32_t T;              /* steps fused per HBM pass = halo depth, 1..HEAT1D_T_MAX;
                               0 = auto (chosen per arithmetic mode)          */
    int32_t mode;           /* HEAT1D_MODE_*                                                */
    int32_t denominator;    /* HEAT1D_DEN_*                                                 */
    int32_t allow_unstable; /* nonzero: accept r > 1/2                                      */
    int32_t virtual_slabs;  /* >= 1; with nranks == 1, split the ring into this many slabs on
                               ONE device that exchange halos by device copies -- the exact
                               multi-GPU schedule with the transport replaced (test harness) */
    int32_t kernel;         /* HEAT1D_KERNEL_*                                              */
    int32_t blocking;       /* nonzero (default): heat1d_set_initial / heat1d_run / heat1d_get
                               return after the device is done; zero: they only enqueue on
                               `stream` (stream-ordered: keep u0 intact and read `out` only
                               after synchronising the stream)                              */
    int32_t use_graphs;     /* nonzero (default): replay pass sequences as CUDA graphs      */
    int32_t resident;       /* -1 (default) auto, 0 never, 1 required: solve a ring that fits
                               on chip (single slab, single rank, <= ~1.8 M cells) in ONE
                               cooperative launch with the slab held in registers (K6)      */
    void *stream;           /* cudaStream_t for compute (e.g. torch's current stream);
                               NULL = a stream owned by the handle                          */
    void *comm_stream;      /* cudaStream_t for halo exchange; NULL = owned by the handle   */
    int32_t transport;      /* HEAT1D_TRANSPORT_* for the K2 schedule of several slabs; default
                               P2P, which create turns into NCCL (on every rank) if any rank
                               cannot map its neighbours' memory                            */
    double *dev_buf;        /* optional caller-owned device memory for the state (e.g. a torch
                               tensor): >= heat1d_buffer_len(nx, np, opts) doubles, 256-byte
                               aligned, outliving the handle; NULL = the handle cudaMallocs   */
    int64_t window_cells;   /* > 0: STREAMING handle for rings larger than device memory: the
                               device holds only three light-cone windows of this many cells
                               (x2 ping-pong buffers); only heat1d_solve_host is available
                               (window_cells >= 18*nt); 0 (default) = the whole ring on device */
} heat1d_opts;

/* Read-only facts about a handle (heat1d_info). */
typedef struct {
    uint32_t size;          /* = sizeof(heat1d_info_t)                                     */
    int32_t T;              /* effective halo depth / steps per pass                        */
    int32_t mode, denominator, kernel;
    int32_t dp_ops;         /* fp64 instructions per cell update in the pass kernel (1..4)  */
    int32_t nslabs;         /* slabs held by this handle (virtual_slabs, else 1)            */
    int32_t rank, nranks, device;
    double r;               /* k*dt/D as used by the kernels                                */
    int64_t N, first, count;/* ring size, this rank's slab [first, first+count)             */
    int64_t steps_done;
    int64_t launches;       /* kernels launched by this handle so far (all kinds)           */
    int64_t pad;            /* ghost cells allocated on each side of a slab                 */
    int32_t tile_cells;     /* output cells per CTA tile of the pass kernel (at T)          */
    int32_t grid;           /* CTAs per pass-kernel launch (persistent)                     */
    int32_t pass_kind;      /* pass-kernel variant: 3 / 4 = warps trading 8- / 16-deep ghosts */
    int32_t pass_V, pass_NW, pass_S; /* cells/lane, compute warps/CTA, TMA stages            */
    int32_t resident;       /* 1 if runs use the register-resident kernel K6                */
    int32_t resident_warps; /* warps of the last K6 launch                                  */
    int64_t stream_windows; /* light-cone windows of the last heat1d_solve_host (0: plain)  */
    int32_t transport;      /* HEAT1D_TRANSPORT_* in use (after create's fallback)          */
    int32_t resident_V;     /* cells per lane of the last K6 launch (0: none yet)           */
    int32_t pass_feed;      /* 1: full passes run feed tiles (k2f_pass: strips, left-fed tiles) */
    int32_t reserved1;
} heat1d_info_t;

/* Exchange plan of one rank (pure host logic; usable without a GPU).  Offsets
 * are in cells relative to cell 0 of the rank's slab (negative = left pad). */
typedef struct {
    int32_t left, right;        /* neighbour ranks (g-1) mod G, (g+1) mod G                 */
    int64_t send_right_off;     /* = count - T : last T cells, sent first  to `right`       */
    int64_t send_left_off;      /* = 0         : first T cells, sent second to `left`       */
    int64_t recv_left_off;      /* = -T        : left pad, received first  from `left`      */
    int64_t recv_right_off;     /* = count     : right pad, received second from `right`    */
    int64_t cells;              /* T cells per message (8T bytes)                           */
} heat1d_exchange_plan;

/* Citation key: P:NN = PAPER.md line NN (Section 2 "Model problem": Eq. 1 at P:61, Eq. 2 at
 * P:66-70, the grid at P:64-65, u(0,x_i) = x_i and the periodic loop at P:71, the segmented
 * ghost-zone algorithm at; "cells processed per second" at P:228).  Unless stated,
 * every call returns HEAT1D_EINVAL for a NULL handle / output pointer and leaves all state
 * unchanged on EINVAL; ECUDA / ENCCL poison the handle. */

/* Fill *o with the defaults (matched mode, D = dx^2, auto T, one rank, P2P transport).
 * NULL-safe.  Not from the paper: the ABI's option conventions. */
HEAT1D_API void heat1d_opts_default(heat1d_opts *o);
HEAT1D_API int heat1d_version(void);
/* Static string for a status code (never NULL). */
HEAT1D_API const char *heat1d_strerror(int status);

/* Slab [*first, *first + *count) of `rank` when the ring of N = nx*np cells (the paper's
 * np segments of nx cells) is split over `nranks` contiguous slabs:
 * partition-granular and front-loaded when np >= nranks, else
 * cell-granular front-loaded.  Pure host function (no GPU).  EINVAL: nx < 1, np < 1,
 * N > 2^62, rank outside [0, nranks), or fewer cells than slabs. */
HEAT1D_API int heat1d_partition(int64_t nx, int64_t np, int32_t nranks, int32_t rank,
                     int64_t *first, int64_t *count);

/* The ghost-zone exchange of P:73 at depth T: the four messages of `rank` (offsets in cells
 * from cell 0 of its slab; negative = left pad).  Pure host function, and the single
 * source of the offsets every exchange the library issues uses.  Order matters when
 * left == right (nranks == 2): send(right edge), send(left edge), recv(left pad),
 * recv(right pad).  EINVAL: as heat1d_partition, T < 1, or T > the smallest slab. */
HEAT1D_API int heat1d_plan_exchange(int64_t nx, int64_t np, int32_t nranks, int32_t rank, int32_t T,
                         heat1d_exchange_plan *plan);

/* Doubles of device memory a handle with these arguments needs for its state (both
 * ping-pong buffers of every local slab -- the Jacobi double buffer of Eq. 2, which reads
 * time-t values only, P:68 -- with pads for T = opts->T or, if 0, HEAT1D_T_MAX): the
 * minimum size of opts->dev_buf.  opts may be NULL (defaults).  -1 on invalid arguments. */
HEAT1D_API int64_t heat1d_buffer_len(int64_t nx, int64_t np, const heat1d_opts *opts);

/* rank 0 only: writes a 128-byte ncclUniqueId to out128 (caller-owned host memory), to be
 * broadcast to every rank's opts.nccl_id.  ENCCL if NCCL fails.  (Plumbing, not the paper.) */
HEAT1D_API int heat1d_get_unique_id(void *out128);

/* Set up the model problem of P:57-71 for nt steps: N = nx*np grid points x_i = i*dx
 * (P:64-65), diffusivity k (alpha) and time step dt, r = (k*dt)/(dx*dx) computed once
 * on the host in fp64 (Eq. 2, with the denominator of DESIGN.md reading c1; the
 * literal "2h" is opts->denominator = HEAT1D_DEN_PAPER_2DX).  Validates, picks T and the
 * kernel family (agreed over the ranks), allocates 2 buffers of (count + 2*pad) fp64 per
 * slab (or uses opts->dev_buf), creates streams/events and, with nranks > 1, joins the
 * NCCL ring and maps the neighbours' memory -- collective over all ranks.  nt is the
 * default step count of heat1d_run(h, -1).  On error *out = NULL.
 * Errors: EINVAL (nx < 1, np < 1, N > 2^62, nt < 0, k < 0, dt <= 0, dx <= 0, non-finite
 * arguments, bad rank/nranks/T/virtual_slabs/mode, nranks > 1 without nccl_id), EUNSTABLE
 * (r > 1/2 without allow_unstable), EUNSUPPORTED (a combination this build does
 * not run, e.g. resident = 1 for a slab that does not fit), ENOMEM, ECUDA, ENCCL. */
HEAT1D_API int heat1d_create(heat1d_t *out, int64_t nx, int64_t np, int64_t nt,
                  double k, double dt, double dx, const heat1d_opts *opts);

/* This handle's slab [*first, *first + *count) of the ring (heat1d_partition of its rank;
 * all virtual slabs together).  Host-only, never fails on a valid handle. */
HEAT1D_API int heat1d_local_range(heat1d_t h, int64_t *first, int64_t *count);

/* The initial condition u(0, x_i) of this rank's slab (P:71 gives u(0, x_i) = x_i; any
 * values are accepted).  u0: `count` (= the local slab) fp64 values, host or device
 * pointer, COPIED before return (the caller may free u0 at once; the caller owns it) --
 * on a non-blocking handle (opts.blocking = 0) the copy is only enqueued on the stream.
 * Resets steps_done to 0; in fast mode K5 computes max|u0| on the device, where the scaled
 * kernels read it (DESIGN.md c21; no host round trip).
 * EINVAL: NULL u0 or count != local count.  EUNSUPPORTED on a streaming handle. */
HEAT1D_API int heat1d_set_initial(heat1d_t h, const double *u0, int64_t count);

/* Device-side initial condition u0[i] = lo + (hi-lo)*U(seed, i) for the global cell
 * indices i of this slab, U = splitmix64 counter form (reading c12 for
 * BASELINE.json's "uniform from seed s"; identical to synth.uniform).  Not from the
 * paper: the synthetic inputs of BASELINE.json configs[1], [3].  Resets steps_done.
 * EINVAL on non-finite lo/hi. */
HEAT1D_API int heat1d_init_uniform(heat1d_t h, uint64_t seed, double lo, double hi);

/* Advance nt >= 0 steps of Eq. 2 on the periodic loop, cumulative over
 * calls (nt < 0 = create's nt): T steps per pass over the state, depth-T ghost zones
 * exchanged between slabs every T steps -- the segmented algorithm of P:73 at depth T.
 * Matched mode is bitwise equal to nt sweeps of the literal update (the oracle) for any
 * T, slab and rank count.  Blocking by default (opts.blocking).  Collective over ranks
 * when nranks > 1.  ESTATE before an initial state; ECUDA/ENCCL poison the handle. */
HEAT1D_API int heat1d_run(heat1d_t h, int64_t nt);

/* Copy this slab's current state u(t, x_i) (t = steps_done) to out: `count` (= the local
 * slab) fp64, host or device pointer, caller-owned; synchronous (non-blocking handles:
 * enqueued on the stream).  EINVAL: NULL out or
 * count mismatch.  ESTATE before an initial state. */
HEAT1D_API int heat1d_get(heat1d_t h, double *out, int64_t count);

/* One whole solve between HOST arrays with the transfers hidden behind the compute:
 * u0 (count = local n cells) -> nt steps -> out (count cells); same result as
 * heat1d_set_initial(u0) + heat1d_run(nt) + heat1d_get(out) (bitwise in matched mode).
 * By the domain of dependence of Eq. 2 (a cell at step t depends on cells within t
 * of it at step 0), the ring is cut into C chunks and each chunk is solved on its own
 * light-cone window [chunk - nt, chunk + nt) (indices mod N); the H2D copy of window c+1
 * and the D2H copy of chunk c-1 run on their own streams while window c computes, so a
 * solve costs ~max(transfers, compute) instead of their sum.  Used for one slab per rank
 * when the chunks are >= 16 nt cells and nt <= the slab (redundant work <= 2nt/chunk);
 * with nranks > 1 the ranks first trade nt-deep halos once (the plan of
 * heat1d_plan_exchange at depth nt, NCCL; collective, every rank takes the same branch);
 * otherwise it IS the plain three-call sequence.  u0/out (caller-owned) should be pinned
 * (cudaHostAlloc / torch pin_memory) for the copies to overlap.  In fast mode every
 * window's own max|u0| (K5) decides on the device whether it runs the scaled form or the
 * 3-op form (DESIGN.md c21).  Afterwards the device state is consumed: call
 * set_initial before run/get.  EINVAL: NULL or overlapping u0/out, count mismatch.
 * EUNSUPPORTED: a streaming handle whose window cannot hold nt.  Else as run. */
HEAT1D_API int heat1d_solve_host(heat1d_t h, const double *u0, int64_t count, int64_t nt, double *out);

/* heat1d_solve_host for ONE slab whose neighbour cells the caller supplies: left = the nt
 * cells preceding the slab (left[nt-1] next to u0[0]), right = the nt cells following it
 * (host or device pointers, caller-owned).  The result depends on nothing else (the light
 * cone of nt steps), so a caller that decomposes a ring itself needs no further
 * communication.  EUNSUPPORTED if the slab is too small for the windows. */
HEAT1D_API int heat1d_solve_host_halo(heat1d_t h, const double *u0, const double *left, const double *right,
                                      int64_t count, int64_t nt, double *out);

/* Steps advanced since the last initial state (t of u(t, x_i)); -1 if h is NULL. */
HEAT1D_API int64_t heat1d_steps_done(heat1d_t h);
/* Read-only facts (heat1d_info_t); info->size must equal sizeof(heat1d_info_t) (EINVAL). */
HEAT1D_API int heat1d_info(heat1d_t h, heat1d_info_t *info);

/* Profiling: while on, every kernel group is bracketed by CUDA events on
 * the stream it runs on -- the interior pass K2 / the resident K6 / K1 on the compute
 * stream, the halo exchange + edge strips (K3/K3p, several slabs) on the comm stream.
 * CUDA graphs are bypassed while profiling.  heat1d_set_profiling(h, 1) resets the totals
 * and the trace and records the trace's time origin on the compute stream.
 * heat1d_profile: launches and summed milliseconds of the compute-stream groups (the
 * dominant kernel) since profiling was enabled (synchronises both streams). */
HEAT1D_API int heat1d_set_profiling(heat1d_t h, int on);
HEAT1D_API int heat1d_profile(heat1d_t h, int64_t *launches, double *ms);

enum { HEAT1D_TRACE_K1 = 1, HEAT1D_TRACE_K2 = 2, HEAT1D_TRACE_HALO = 3, HEAT1D_TRACE_K6 = 6 };
typedef struct {
    int32_t stream;         /* 0 = compute stream, 1 = comm stream                          */
    int32_t kind;           /* HEAT1D_TRACE_*                                               */
    double t0_ms, t1_ms;    /* interval, ms after heat1d_set_profiling(h, 1)                */
} heat1d_trace_event;

/* The profiling session's intervals (the overlap timeline of the two streams; the
 * first min(cap, *count) are copied to events, caller-owned host memory; at most 2^20
 * are kept).  *count = how many exist.  EINVAL on NULL count (or NULL events with
 * cap > 0); synchronises both streams. */
HEAT1D_API int heat1d_trace(heat1d_t h, heat1d_trace_event *events, int64_t cap, int64_t *count);

/* Compute stream of the handle as a cudaStream_t (for the caller's events). */
HEAT1D_API void *heat1d_stream(heat1d_t h);

/* NULL-safe; frees library-owned memory, streams, events and the NCCL comm.  With
 * peer-memory transports (nranks > 1) it is collective: it waits until every rank's
 * streams are idle before unmapping or freeing anything a neighbour writes into. */
HEAT1D_API int heat1d_destroy(heat1d_t h);

/* Message for the last failing call on h ("" if none). */
HEAT1D_API const char *heat1d_last_error(heat1d_t h);

#ifdef __cplusplus
}
#endif
#endif /* HEAT1D_H */
