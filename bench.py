#!/usr/bin/env python
"""Benchmark of libheat1d: fp64 cell-updates/s (GLUPS) of Eq. 2 on a periodic ring.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--T 0] [--mode matched]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...
    python bench.py --impl reference ...      # the CPU oracle on a bounded sample

`--gpus N` outside torchrun re-launches itself under torch.distributed.run with N
ranks (one per GPU, NCCL_DEBUG=INFO so the communicator's rank count is logged);
it exits non-zero if fewer than N GPUs are visible.

A step is one full solve of the workload through the C ABI: load u0 (device
resident copy -> state) and advance nt steps (BASELINE.json configs[3] = C4 by
default: 2^31 cells, nt = 10,000, the ring the metric's 1/2/4/8-GPU scaling
is quoted on).  value = N*nt*K / (max over ranks of the CUDA-event time of
the K timed steps).  The headline arithmetic is matched mode (Eq. 2's own
rounding sequence, bitwise = the oracle); fast mode is timed beside it under
`other_mode`.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 cell-updates/sec (GLUPS) at 1/2/4/8 B200 and % of HBM/FP64 roofline"
FALLBACK_HBM_GBS = 6650.0
SMS, FP64_LANES, SM_MHZ_MAX = 148, 64, 1965.0             # B200: fp64 lanes per SM, max SM clock
BJ_FLOP_PER_UPDATE = 4.0                                  # BASELINE.json north_star: "4 flops per update"
PARITY_STEPS = 100                                        # BASELINE.json configs[3]: "oracle checked on the first 100 steps"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5, help="timed solves (SURVEY §8(d): 5 repetitions)")
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    p.add_argument("--T", type=int, default=0)
    p.add_argument("--mode", default="matched", choices=["matched", "fast"],
                   help="headline arithmetic: matched (bitwise = oracle) or fast (north_star bound)")
    p.add_argument("--virtual-slabs", type=int, default=1,
                   help="split each rank's ring into this many slabs on its GPU (multi-slab schedule on 1 GPU)")
    p.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    p.add_argument("--no-other-mode", action="store_true", help="skip timing the other mode")
    p.add_argument("--nt", type=int, default=0, help="override the config's nt (testing only)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-parity", action="store_true", help="skip the post-run check against the oracle")
    p.add_argument("--out", default="", help="also append the JSON line to this file")
    return p.parse_args()


# ------------------------------------------------------------------ launch
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(args):
    """--gpus N > 1 without a torchrun environment: become N ranks (one per GPU)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write("bench.py: --gpus %d but only %d CUDA device(s) visible\n" % (args.gpus, have))
        sys.exit(3)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


def fp64_peak():
    """fp64 pipe peak in T lane-instructions/s: measured by tools/fp64_peak.cu on a B200 of this
    pool (profiles/fp64_peak.json, best DADD rate), else derived from 148 SM x 64 lanes x 1.965 GHz."""
    derived = SMS * FP64_LANES * SM_MHZ_MAX * 1e6 / 1e12
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        best = max(r["dadd_tinst_s"] for r in d["results"])
        return best, "measured (tools/fp64_peak.cu: independent DADD chains, profiles/fp64_peak.json)"
    except Exception:
        return derived, "derived: 148 SM x 64 fp64 lanes x 1.965 GHz"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi samples DURING the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = set(gpus)
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-lms", "200", "-f", self.path], stdout=subprocess.DEVNULL,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9 or not p[0].isdigit() or int(p[0]) not in self.gpus:
                    continue
                try:
                    sm.append(float(p[1]))
                    mx.append(float(p[2]))
                    power.append(float(p[3]))
                except ValueError:
                    continue
                for nm, v in zip(names, p[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            os.unlink(self.path)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------ oracle baseline (CPU)
def host_identity():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except Exception:
        avail = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "cores_available": avail}


class PinOneCore:
    """Pin the calling process to one core for the single-threaded oracle."""

    def __enter__(self):
        self.prev = None
        self.core = None
        try:
            self.prev = os.sched_getaffinity(0)
            self.core = max(self.prev)
            os.sched_setaffinity(0, {self.core})
        except Exception:
            pass
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            try:
                os.sched_setaffinity(0, self.prev)
            except Exception:
                pass


def cpu_oracle_sample(cfg, target_s=12.0):
    """Time the oracle (O3 light-cone window == O1 on the window) on a contiguous
    window of the workload's ring for its first steps, single-threaded, pinned."""
    import oracle
    r = oracle.r_of(cfg.k, cfg.dt, cfg.dx)
    t = min(cfg.nt, 100)
    m = min(cfg.N, 1 << 20)
    with PinOneCore() as pin:
        if cfg.N < m + 2 * t:  # tiny ring: whole-ring O1
            u0 = cfg.u0()
            t0 = time.perf_counter()
            oracle.run(u0, r, cfg.nt)
            dt = time.perf_counter() - t0
            return cfg.N * cfg.nt / dt / 1e9, "whole ring N=%d x %d steps (O1)" % (cfg.N, cfg.nt), pin.core
        w0 = cfg.u0(0 - t, m + 2 * t)
        t0 = time.perf_counter()
        oracle.window(w0, t, r)
        dt = time.perf_counter() - t0
        rate = (m + t) * t / dt
        m2 = int(min(cfg.N - 2 * t, max(m, rate * target_s / t - t)))
        m2 = max(1024, m2)
        w0 = cfg.u0(0 - t, m2 + 2 * t)
        t0 = time.perf_counter()
        oracle.window(w0, t, r)
        dt = time.perf_counter() - t0
    upd = sum(m2 + 2 * (t - s) - 2 for s in range(t))  # cells updated per shrinking step
    return upd / dt / 1e9, "O3 window of %d cells x first %d steps of %s (%.3g updates, %.1f s)" % (
        m2, t, cfg.name, upd, dt), pin.core


def cpu_baseline_obj(value, sample, core):
    d = {"value": value, "unit": "GLUPS", "cores": 1, "kind": "oracle", "sample": sample,
         "threads": 1, "pinned_core": core}
    d.update(host_identity())
    return d


def reference_arm(args, cfg, rank):
    """--impl reference: the oracle as it stands, on rank 0's host cores (one pinned core)."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    vals = []
    sample, core = "", None
    for i in range(args.warmup + args.steps):
        v, sample, core = cpu_oracle_sample(cfg, target_s=4.0)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GLUPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "N": cfg.N, "nx": cfg.nx, "np": cfg.np, "nt": cfg.nt, "k": cfg.k,
                   "dt": cfg.dt, "dx": cfg.dx, "mode": "oracle (canonical order, bitwise = matched mode)",
                   "parallelism": "cpu, 1 core"},
        "cpu_baseline": cpu_baseline_obj(value, sample, core),
        "e2e": {"value": value, "unit": "GLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")


# ------------------------------------------------------------------ roofline
def flops_executed(dp_ops, steps_per_pass):
    """fp64 flops the kernel's arithmetic executes per update (FMA = 2): the 4-op and 3-op
    matched forms and the literal form compute Eq. 2's 5 flops; the scaled fast forms 1 (r=1/2)
    or 3 (+ one rescale DMUL per cell per pass)."""
    return {1: 1.0, 2: 3.0}.get(dp_ops, 5.0) + (1.0 / steps_per_pass if dp_ops <= 2 else 0.0)


def kernel_roofline(info, cfg, count, world, steps, k_launches, k_ms, ms, value, mode):
    """Roofline of the dominant kernel (K2 pass or K6 whole solve), as SURVEY §8(d) /
    BASELINE.json north_star define it: min(HBM / (16/T B), FP64 peak / 4 flop) per update."""
    if not k_launches:
        return None
    hbm, hbm_kind = hbm_peak()
    pipe, pipe_kind = fp64_peak()                            # T fp64 lane-instructions / s
    fp64_tflops = 2.0 * pipe                                 # FMA = 2 flop
    T = info["T"]
    avg_ms = k_ms / k_launches
    upd_launch = count * cfg.nt * steps / k_launches         # cell updates per launch, this rank
    steps_per_pass = cfg.nt if info["resident"] else T       # steps per HBM round trip of the state
    alg_bytes = 16.0 * upd_launch / steps_per_pass           # 8 B read + 8 B written per cell per pass
    hbm_glups = hbm / (16.0 / steps_per_pass)                # GLUPS bound by HBM
    fp64_glups = fp64_tflops * 1e3 / BJ_FLOP_PER_UPDATE      # GLUPS bound by FP64 peak / 4 flop
    secs = avg_ms / 1e3
    achieved_gbs = alg_bytes / secs / 1e9
    achieved_tflops = BJ_FLOP_PER_UPDATE * upd_launch / secs / 1e12
    if hbm_glups <= fp64_glups:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                "frac": achieved_gbs / hbm, "peak_kind": hbm_kind}
    else:
        roof = {"bound": "alu", "achieved": achieved_tflops, "peak": fp64_tflops,
                "unit": "TFLOP/s (4 flop/update, SURVEY §8(d))", "frac": achieved_tflops / fp64_tflops,
                "peak_kind": pipe_kind + " x 2 flop/FMA"}
    kind = info["pass_kind"]
    kernel = ("k6_resident<V=%d>" % info["resident_V"] if info["resident"] else
              "%s<V=%d,NW=%d,S=%d,KX=%d>" % ("k2f_pass" if info.get("pass_feed") else "k2p_pass", info["pass_V"],
                                             info["pass_NW"], info["pass_S"], 8 if kind == 3 else 16)) + \
        "<OPS=%d>" % info["dp_ops"]
    # the kernel's own bound: fp64 instructions it must issue per update (dp_ops; the scaled
    # fast variants add one rescale DMUL per cell per pass) against the fp64 pipe's issue rate
    inst_per_upd = info["dp_ops"] + (1.0 / steps_per_pass if info["dp_ops"] <= 2 else 0.0)
    dpi = inst_per_upd * upd_launch / secs / 1e12
    flops_x = flops_executed(info["dp_ops"], steps_per_pass)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("%s_T%d_%s" % (cfg.name, T, mode))
    except Exception:
        pass
    roof.update({
        "traffic": traffic, "kernel": kernel, "launches": k_launches, "avg_launch_ms": avg_ms,
        "steps_per_launch": upd_launch / count, "updates_per_launch": upd_launch,
        "alg_bytes_per_launch": alg_bytes, "alg_flop_per_launch": BJ_FLOP_PER_UPDATE * upd_launch,
        "roofline_glups": min(hbm_glups, fp64_glups) * world,
        "hbm_gbs_achieved": achieved_gbs, "hbm_frac": achieved_gbs / hbm,
        # what the kernel itself executes (not §8(d)'s algorithmic count)
        "fp64_inst_per_update": inst_per_upd, "fp64_flop_per_update_executed": flops_x,
        "reduced_op_form": flops_x < BJ_FLOP_PER_UPDATE,
        "fp64_pipe_frac": dpi / pipe,
        "kernel_issue_bound_glups": min(hbm_glups, pipe * 1e3 / inst_per_upd) * world,
        "kernel_share_of_step": k_ms / ms if world == 1 else None})
    return roof


# ------------------------------------------------------------------ GPU arm
def fresh_nccl_id(h1, world, rank):
    """One ncclUniqueId per communicator (each handle owns one), broadcast from rank 0."""
    if world == 1:
        return None
    import torch.distributed as dist
    obj = [h1.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor(x if isinstance(x, list) else [x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    v = t.tolist()
    return v if isinstance(x, list) else v[0]


def timed_steps(fn, steps, stream, world):
    """K back-to-back calls bracketed by barrier + synchronize, CUDA events on `stream` around
    each; returns (total ms, per-step ms), both max over ranks."""
    import torch
    import torch.distributed as dist
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs[0].record(stream)
    for i in range(steps):
        fn()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    total = evs[0].elapsed_time(evs[steps])
    both = max_over_ranks([total] + per, world)
    return both[0], both[1:]


def step_stats(per, updates_per_step):
    return {"ms_median": statistics.median(per), "ms_min": min(per), "ms_max": max(per),
            "glups_median": updates_per_step / (statistics.median(per) / 1e3) / 1e9,
            "glups_best": updates_per_step / (min(per) / 1e3) / 1e9, "ms_all": per}


def measure(h1, cfg, mode, args, world, rank, local_rank, stream, u0_dev, with_e2e, sampler_on):
    """Time K steps (after W warm-ups) of one full solve in `mode`; max over ranks."""
    import torch
    # non-blocking handle: set_initial/run/get are stream-ordered (no host synchronisation between
    # the steps; the timed region is bracketed by synchronize + CUDA events on that stream)
    h = h1.Heat1D(cfg.nx, cfg.np, cfg.nt, cfg.k, cfg.dt, cfg.dx, T=args.T, mode=mode, rank=rank,
                  nranks=world, nccl_id=fresh_nccl_id(h1, world, rank), device=local_rank, stream=stream,
                  virtual_slabs=args.virtual_slabs, transport=args.transport, blocking=False)
    first, count = h.local_range

    def step():
        h.set_initial(u0_dev)
        h.run(cfg.nt)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(range(torch.cuda.device_count())) if (rank == 0 and sampler_on) else None
    launches0 = h.info()["launches"]
    h.set_profiling(True)
    if sampler:
        sampler.start()
        time.sleep(0.3)
    ms, per = timed_steps(step, args.steps, stream, world)
    clocks = sampler.stop() if sampler else None
    k_launches, k_ms = h.profile()
    h.set_profiling(False)
    launches = h.info()["launches"] - launches0
    info = h.info()
    updates = cfg.N * cfg.nt
    value = updates * args.steps / (ms / 1e3) / 1e9

    # ---- end to end through the C ABI from/to pinned HOST memory (copies inside the timed region)
    e2e = None
    if with_e2e:
        host_in = torch.empty(count, dtype=torch.float64, pin_memory=True)
        host_out = torch.empty(count, dtype=torch.float64, pin_memory=True)
        host_in.copy_(u0_dev)
        torch.cuda.synchronize()

        def plain():
            h.set_initial(host_in)
            h.run(cfg.nt)
            h.get(host_out)

        def windows():
            h.solve_host(host_in, cfg.nt, host_out)

        res = {}
        for name, fn in (("set_initial+run+get", plain), ("solve_host", windows)):
            ems, eper = timed_steps(fn, args.steps, stream, world)
            res[name] = {"value": updates * args.steps / (ems / 1e3) / 1e9, "ms_per_step": ems / args.steps,
                         "windows": h.info()["stream_windows"] if name == "solve_host" else 0}
        # the headline e2e: at one rank the light-cone-window solve (transfers hidden behind the
        # compute); across ranks the plain sequence, whose run() exchanges depth-T halos every T
        # steps (the multi-rank solve_host trades nt-deep halos once instead)
        head = "solve_host" if world == 1 else "set_initial+run+get"
        e2e = {"value": res[head]["value"], "unit": "GLUPS", "h2d_bytes_per_step": 8 * count,
               "d2h_bytes_per_step": 8 * count, "ms_per_step": res[head]["ms_per_step"],
               "path": {"solve_host": "heat1d_solve_host(pinned host u0 -> nt steps -> pinned host out): "
                                      "light-cone windows, H2D/D2H overlapped with compute",
                        "set_initial+run+get": "heat1d_set_initial(pinned host) + heat1d_run(nt) + "
                                               "heat1d_get(pinned host)"}[head],
               "variants": res}
        del host_in, host_out
    roof = kernel_roofline(info, cfg, count, world, args.steps, k_launches, k_ms, ms, value, mode)
    return {"value": value, "ms": ms, "per": per, "info": info, "roof": roof, "e2e": e2e, "clocks": clocks,
            "launches": launches, "handle": h, "first": first, "count": count}


def parity_check(h1, h, cfg, u0_dev, first, count, world, mode):
    """After the timed region: the first min(nt, 100) steps of the same handle vs the oracle's
    light-cone windows (O3) at both ends of this rank's slab (the slab boundaries, where the
    halo exchange acts) and in its middle.  Matched: bitwise; fast: north_star's bound."""
    import numpy as np
    import oracle
    t = min(cfg.nt, PARITY_STEPS)
    r = oracle.r_of(cfg.k, cfg.dt, cfg.dx)
    import torch
    h.set_initial(u0_dev)
    h.run(t)
    got_dev = torch.empty(count, dtype=torch.float64, device="cuda")
    h.get(got_dev)
    w = min(count, 4096)
    bad = 0
    checked = 0
    worst = 0.0
    bound = 0.0
    for a in sorted({0, max(0, count // 2 - w // 2), count - w}):
        w0 = cfg.u0(first + a - t, w + 2 * t)
        want = oracle.window(w0, t, r)
        g = got_dev[a:a + w].cpu().numpy()
        checked += w
        if mode == "matched":
            bad += int(np.count_nonzero(g.view(np.uint64) != want.view(np.uint64)))
        else:
            worst = max(worst, float(np.max(np.abs(g - want))))
            bound = max(bound, 1e-12 * float(np.max(np.abs(w0))) * t)
    del got_dev
    ok = bad == 0 if mode == "matched" else worst <= bound
    ok_all = max_over_ranks(0.0 if ok else 1.0, world) == 0.0
    return {"steps": t, "cells_checked_per_rank": checked, "windows": "O3 at slab start, middle, end (every rank)",
            "criterion": "bitwise" if mode == "matched" else "<= 1e-12*max|u0|*t", "ok": bool(ok_all),
            "mismatches_rank0": bad, "max_abs_err_rank0": worst}


def main():
    args = parse()
    from synth.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.nt:
        from dataclasses import replace
        cfg = replace(cfg, nt=args.nt)
    in_torchrun = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, cfg, rank)
        return
    if args.gpus > 1 and not in_torchrun:
        relaunch_under_torchrun(args)
    if in_torchrun and world != args.gpus:
        sys.stderr.write("bench.py: WORLD_SIZE=%d but --gpus %d\n" % (world, args.gpus))
        sys.exit(3)

    import torch
    import torch.distributed as dist
    from paper_2307_01117_b200 import _build
    _build.build()
    import paper_2307_01117_b200 as h1

    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    # a real stream (torch's default stream has handle 0, which the C ABI reads as "create
    # your own"): the handles, the timing events and torch's own copies all run on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    # device-resident u0 for this rank's slab (inputs in HBM before the timed region)
    first, count = h1.partition(cfg.nx, cfg.np, world, rank)
    u0_dev = torch.empty(count, dtype=torch.float64, device="cuda")
    if cfg.u0_kind == "uniform":
        with h1.Heat1D(cfg.nx, cfg.np, 0, cfg.k, cfg.dt, cfg.dx, rank=rank, nranks=world,
                       nccl_id=fresh_nccl_id(h1, world, rank), device=local_rank, stream=stream) as hg:
            hg.init_uniform(cfg.seed, cfg.lo, cfg.hi)
            hg.get(u0_dev)
    else:
        u0_dev.copy_(torch.from_numpy(cfg.u0(first, count)))
    torch.cuda.synchronize()

    main_m = measure(h1, cfg, args.mode, args, world, rank, local_rank, stream, u0_dev, not args.no_e2e, True)
    parity = None
    if not args.no_parity:
        parity = parity_check(h1, main_m["handle"], cfg, u0_dev, first, count, world, args.mode)
    main_m["handle"].close()
    other = None
    if not args.no_other_mode:
        om = "matched" if args.mode == "fast" else "fast"
        o = measure(h1, cfg, om, args, world, rank, local_rank, stream, u0_dev, False, False)
        o["handle"].close()
        other = {"mode": om, "value": o["value"], "ms_per_step": o["ms"] / args.steps,
                 "step_stats": step_stats(o["per"], cfg.N * cfg.nt),
                 "dp_ops": o["info"]["dp_ops"], "T": o["info"]["T"], "gpu_launches": o["launches"],
                 "roofline": o["roof"],
                 "parity": "bitwise = oracle" if om == "matched" else "<= 1e-12*max|u0|*nt vs oracle"}
    info = main_m["info"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, sample, core = cpu_oracle_sample(cfg)
            cpu = cpu_baseline_obj(v, sample, core)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "GLUPS", "cores": 1, "kind": "oracle", "sample": "failed: %s" % e}

    if world > 1:
        dist.barrier()  # every rank is quiet (no NCCL logging) while rank 0 prints its line
    if rank == 0:
        ms = main_m["ms"]
        nslab = world * args.virtual_slabs
        line = {
            "metric": METRIC, "value": main_m["value"], "unit": "GLUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE.json %s recipe, seeded)" % cfg.name,
            "config": {"workload": cfg.name, "N": cfg.N, "nx": cfg.nx, "np": cfg.np, "nt": cfg.nt, "k": cfg.k,
                       "dt": cfg.dt, "dx": cfg.dx, "r": info["r"], "T": info["T"], "mode": args.mode,
                       "parity": ("bitwise = oracle (Eq. 2's rounding sequence)" if args.mode == "matched"
                                  else "<= 1e-12*max|u0|*nt vs oracle (north_star fast-mode bound)"),
                       "dp_ops": info["dp_ops"], "parallelism": "slabs%d" % nslab,
                       "ranks": world, "virtual_slabs_per_rank": args.virtual_slabs,
                       "halo_transport": ("none (one slab)" if nslab == 1 else
                                          "k6 mailbox (NVLink peer memory)" if info["resident"] else
                                          ["nccl send/recv" if world > 1 else "device copies + K3",
                                           "p2p puts from K3 (peer memory)"][info["transport"]]),
                       "l2": "inputs larger than L2" if 16 * cfg.N // world > 126 * 2 ** 20
                       else "L2-resident ring (no flush; each step re-reads u0 from HBM copy)",
                       "tile_cells": info["tile_cells"], "grid": info["grid"]},
            "step_stats": step_stats(main_m["per"], cfg.N * cfg.nt),
            "roofline": main_m["roof"], "other_mode": other, "parity_check": parity, "cpu_baseline": cpu,
            "e2e": main_m["e2e"], "clocks": main_m["clocks"], "gpu_launches": main_m["launches"],
        }
        emit(line, args)
    if world > 1:
        # the JSON line is the last thing on stdout: tearing down the process group (or letting
        # interpreter exit do it) would print NCCL's INIT-subsystem "Destroy/Abort COMPLETE"
        # lines after it; every GPU stream is idle and every library handle is closed by now
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)


if __name__ == "__main__":
    main()
