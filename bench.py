#!/usr/bin/env python
"""Benchmark of libheat1d: fp64 cell-updates/s (GLUPS) of Eq. 2 on a periodic ring.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--T 0] [--mode matched]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...
    python bench.py --impl reference ...      # the CPU oracle on a bounded sample

A step is one full solve of the workload through the C ABI: load u0 (device
resident copy -> state) and advance nt steps (BASELINE.json configs[3] = C4 by
default: 2^31 cells, nt = 10,000, the ring the metric's 1/2/4/8-GPU scaling
is quoted on).  value = N*nt*K / (max over ranks of the CUDA-event time of
the K timed steps).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 cell-updates/sec (GLUPS) at 1/2/4/8 B200 and % of HBM/FP64 roofline"
FALLBACK_HBM_GBS = 6650.0
SMS, FP64_LANES, SM_MHZ_MAX = 148, 64, 1965.0             # B200: fp64 lanes per SM, max SM clock
FP64_TFLOPS = SMS * FP64_LANES * 2 * SM_MHZ_MAX * 1e6 / 1e12  # 37.2 TFLOP/s (FMA = 2 flop)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    p.add_argument("--T", type=int, default=0)
    p.add_argument("--mode", default="fast", choices=["matched", "fast"],
                   help="headline arithmetic: fast (north_star bound) or matched (bitwise = oracle)")
    p.add_argument("--no-other-mode", action="store_true", help="skip timing the other mode")
    p.add_argument("--nt", type=int, default=0, help="override the config's nt (testing only)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--out", default="", help="also append the JSON line to this file")
    return p.parse_args()


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


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


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
def cpu_oracle_sample(cfg, target_s=12.0):
    """Time the oracle (O3 light-cone window == O1 on the window) on a contiguous
    window of the workload's ring for its first steps, single-threaded."""
    import numpy as np
    import oracle
    r = oracle.r_of(cfg.k, cfg.dt, cfg.dx)
    t = min(cfg.nt, 100)
    m = min(cfg.N, 1 << 20)
    w0 = cfg.u0(0 - t, m + 2 * t) if cfg.N >= m + 2 * t else None
    if w0 is None:  # tiny ring: whole-ring O1
        u0 = cfg.u0()
        t0 = time.perf_counter()
        oracle.run(u0, r, cfg.nt)
        dt = time.perf_counter() - t0
        return cfg.N * cfg.nt / dt / 1e9, "whole ring N=%d x %d steps (O1)" % (cfg.N, cfg.nt)
    # calibrate, then scale the window to ~target_s
    t0 = time.perf_counter()
    oracle.window(w0, t, r)
    dt = time.perf_counter() - t0
    upd = (m + t) * t
    rate = upd / dt
    m2 = int(min(cfg.N - 2 * t, max(m, rate * target_s / t - t)))
    m2 = max(1024, m2)
    w0 = cfg.u0(0 - t, m2 + 2 * t)
    t0 = time.perf_counter()
    oracle.window(w0, t, r)
    dt = time.perf_counter() - t0
    upd = sum(m2 + 2 * (t - s) - 2 for s in range(t))  # cells updated per shrinking step
    return upd / dt / 1e9, "O3 window of %d cells x first %d steps of %s (%.3g updates, %.1f s)" % (
        m2, t, cfg.name, upd, dt)


def host_cores_used():
    return 1  # the oracle is a plain single-threaded C loop


def reference_arm(args, cfg, rank):
    """--impl reference: the oracle as it stands, on rank 0's host cores."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    vals = []
    sample = ""
    for i in range(args.warmup + args.steps):
        v, sample = cpu_oracle_sample(cfg, target_s=4.0)
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
        "cpu_baseline": {"value": value, "unit": "GLUPS", "cores": host_cores_used(), "kind": "oracle",
                         "sample": sample},
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


# ------------------------------------------------------------------ GPU arm
def kernel_roofline(info, cfg, count, world, steps, k2_launches, k2_ms, ms, value, mode):
    """Roofline of the dominant kernel (K2 pass or K6 whole solve), this rank."""
    if not k2_launches:
        return None
    hbm, peak_kind = peaks()
    T = info["T"]
    avg_ms = k2_ms / k2_launches
    upd_launch = count * cfg.nt * steps / k2_launches       # cell updates per launch, this rank
    steps_per_pass = cfg.nt if info["resident"] else T       # steps per HBM round trip of the state
    alg_bytes = 16.0 * count * (upd_launch / count) / steps_per_pass  # 8 B read + 8 B written per cell per pass
    hbm_term = hbm / (16.0 / steps_per_pass)                 # GLUPS bound by HBM (BASELINE.json)
    fp64_term = FP64_TFLOPS * 1e3 / 4.0                      # GLUPS bound by FP64 peak / 4 flop
    bj_roof = min(hbm_term, fp64_term) * world
    kind = info["pass_kind"]
    k6v = 17 if T <= 32 else 33 if T <= 64 else 49          # resident.cu rv_of(T)
    kernel = ("k6_resident<V=%d>" % k6v if info["resident"] else
              ["k2_pass", "k2w_pass", "k2p_pass", "k2p_pass", "k2p_pass"][kind] + "<V=%d,NW=%d,S=%d%s>" % (
                  info["pass_V"], info["pass_NW"], info["pass_S"],
                  {3: ",KX=8", 4: ",KX=16"}.get(kind, ""))) + "<OPS=%d>" % info["dp_ops"]
    # the kernel's own bounds: HBM (16 B per cell per pass) and the fp64 pipe's issue rate
    # 148 SM x 64 lanes x 1.965 GHz against its algorithmic fp64 instructions per update
    # (dp_ops; the scaled fast variants add one rescale DMUL per cell per pass)
    inst_per_upd = info["dp_ops"] + (1.0 / steps_per_pass if info["dp_ops"] <= 2 else 0.0)
    pipe, pipe_kind = fp64_peak()                            # T fp64 lane-instructions / s
    alu_term = pipe * 1e3 / inst_per_upd                     # GLUPS
    achieved_gbs = alg_bytes / (avg_ms / 1e3) / 1e9
    dpi = inst_per_upd * upd_launch / (avg_ms / 1e3) / 1e12
    if hbm_term <= alu_term:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                "frac": achieved_gbs / hbm, "peak_kind": peak_kind}
    else:
        roof = {"bound": "alu", "achieved": dpi, "peak": pipe, "unit": "Tinst/s (fp64 DFMA/DADD/DMUL)",
                "frac": dpi / pipe, "peak_kind": pipe_kind}
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get("%s_T%d_%s" % (cfg.name, T, mode))
    except Exception:
        pass
    roof.update({
        "traffic": traffic, "kernel": kernel, "launches": k2_launches, "avg_launch_ms": avg_ms,
        "steps_per_launch": upd_launch / count,
        "alg_bytes_per_launch": alg_bytes, "alg_fp64_inst_per_launch": inst_per_upd * upd_launch,
        "fp64_inst_per_update": inst_per_upd, "hbm_gbs_achieved": achieved_gbs,
        "hbm_frac": achieved_gbs / hbm, "fp64_pipe_frac": dpi / pipe,
        "kernel_roofline_glups": min(hbm_term, alu_term) * world,
        "baseline_json_roofline_glups": bj_roof,
        "baseline_json_frac": value / bj_roof,
        "baseline_json_bound": "hbm" if hbm_term < fp64_term else "fp64 (37.2 TFLOP/s / 4 flop)",
        "kernel_share_of_step": k2_ms / ms if world == 1 else None})
    return roof


def fresh_nccl_id(h1, world, rank):
    """One ncclUniqueId per communicator (each handle owns one), broadcast from rank 0."""
    if world == 1:
        return None
    import torch.distributed as dist
    obj = [h1.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def measure(h1, cfg, mode, args, world, rank, local_rank, stream, u0_dev, with_e2e, sampler_on):
    """Time K steps (after W warm-ups) of one full solve in `mode`; max over ranks."""
    import torch
    import torch.distributed as dist
    h = h1.Heat1D(cfg.nx, cfg.np, cfg.nt, cfg.k, cfg.dt, cfg.dx, T=args.T, mode=mode, rank=rank,
                  nranks=world, nccl_id=fresh_nccl_id(h1, world, rank), device=local_rank, stream=stream)
    first, count = h.local_range

    def step():
        h.set_initial(u0_dev)
        h.run(cfg.nt)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(range(world)) if (rank == 0 and sampler_on) else None
    launches0 = h.info()["launches"]
    h.set_profiling(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    ms = ev0.elapsed_time(ev1)
    k2_launches, k2_ms = h.profile()
    h.set_profiling(False)
    launches = h.info()["launches"] - launches0
    info = h.info()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    updates = cfg.N * cfg.nt * args.steps
    value = updates / (ms / 1e3) / 1e9

    # ---- end to end: pinned host u0 -> set_initial -> run -> get -> pinned host
    e2e = None
    if with_e2e:
        host_in = torch.empty(count, dtype=torch.float64, pin_memory=True)
        host_out = torch.empty(count, dtype=torch.float64, pin_memory=True)
        host_in.copy_(u0_dev)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            h.solve_host(host_in, cfg.nt, host_out)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": updates / (ems / 1e3) / 1e9, "unit": "GLUPS", "h2d_bytes_per_step": 8 * count,
               "d2h_bytes_per_step": 8 * count, "ms_per_step": ems / args.steps,
               "path": "heat1d_solve_host(pinned host u0 -> nt steps -> pinned host out)",
               "windows": h.info()["stream_windows"]}
        del host_in, host_out
    roof = kernel_roofline(info, cfg, count, world, args.steps, k2_launches, k2_ms, ms, value, mode)
    h.close()
    return {"value": value, "ms": ms, "info": info, "roof": roof, "e2e": e2e, "clocks": clocks,
            "launches": launches}


def main():
    args = parse()
    from synth.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.nt:
        from dataclasses import replace
        cfg = replace(cfg, nt=args.nt)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2307_01117_b200 import _build
    _build.build()
    import paper_2307_01117_b200 as h1

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stream = torch.cuda.current_stream()

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

    main_m = measure(h1, cfg, args.mode, args, world, rank, local_rank, stream, u0_dev,
                     not args.no_e2e, True)
    other = None
    if not args.no_other_mode:
        om = "matched" if args.mode == "fast" else "fast"
        o = measure(h1, cfg, om, args, world, rank, local_rank, stream, u0_dev, False, False)
        other = {"mode": om, "value": o["value"], "ms_per_step": o["ms"] / args.steps,
                 "dp_ops": o["info"]["dp_ops"], "T": o["info"]["T"], "gpu_launches": o["launches"],
                 "roofline": o["roof"],
                 "parity": "bitwise = oracle" if om == "matched" else "<= 1e-12*max|u0|*nt vs oracle"}
    info = main_m["info"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, sample = cpu_oracle_sample(cfg)
            cpu = {"value": v, "unit": "GLUPS", "cores": host_cores_used(), "kind": "oracle", "sample": sample}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "GLUPS", "cores": 1, "kind": "oracle", "sample": "failed: %s" % e}

    if rank == 0:
        ms = main_m["ms"]
        line = {
            "metric": METRIC, "value": main_m["value"], "unit": "GLUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE.json %s recipe, seeded)" % cfg.name,
            "config": {"workload": cfg.name, "N": cfg.N, "nx": cfg.nx, "np": cfg.np, "nt": cfg.nt, "k": cfg.k,
                       "dt": cfg.dt, "dx": cfg.dx, "r": info["r"], "T": info["T"], "mode": args.mode,
                       "parity": ("bitwise = oracle" if args.mode == "matched"
                                  else "<= 1e-12*max|u0|*nt vs oracle (north_star fast-mode bound)"),
                       "dp_ops": info["dp_ops"], "parallelism": "slabs%d" % world,
                       "halo_transport": ("none (one slab)" if world == 1 else
                                          "k6 mailbox (NVLink peer memory)" if info["resident"] else
                                          ["nccl send/recv", "p2p puts from K3 (NVLink peer memory)"][info["transport"]]),
                       "l2": "inputs larger than L2" if 16 * cfg.N // world > 126 * 2 ** 20
                       else "L2-resident ring (no flush; each step re-reads u0 from HBM copy)",
                       "tile_cells": info["tile_cells"], "grid": info["grid"]},
            "roofline": main_m["roof"], "other_mode": other, "cpu_baseline": cpu, "e2e": main_m["e2e"],
            "clocks": main_m["clocks"], "gpu_launches": main_m["launches"],
        }
        emit(line, args)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
