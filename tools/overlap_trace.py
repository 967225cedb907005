#!/usr/bin/env python
"""Multi-slab schedule on one GPU: throughput of G virtual slabs vs one slab, and the
two-stream timeline (heat1d_trace) showing the halo exchange + edge strips on the comm
stream inside the interior passes on the compute stream.  Measurement aid (not product).

    python tools/overlap_trace.py --config C4 --nt 1000 --slabs 8 --out profiles/r02_overlap_c4.json

Per configuration: best of `reps` timed runs (CUDA events, profiling off), then one
profiled run whose trace gives, per pass, the comm-stream interval [h0, h1] and the
compute-stream span of that pass's K2 launches [k0, k1]; "hidden" = h1 <= k1 (the edge
strips were done before the interior finished, so the exchange cost nothing).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C4")
    p.add_argument("--nt", type=int, default=1000)
    p.add_argument("--slabs", type=int, default=8)
    p.add_argument("--mode", default="matched")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--out", default="")
    a = p.parse_args()
    import torch
    import paper_2307_01117_b200 as h1
    from synth.configs import CONFIGS
    cfg = CONFIGS[a.config]
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    results = []
    for vs, transport in ((1, "p2p"), (a.slabs, "p2p"), (a.slabs, "nccl")):
        with h1.Heat1D(cfg.nx, cfg.np, a.nt, cfg.k, cfg.dt, cfg.dx, mode=a.mode, virtual_slabs=vs,
                       transport=transport, stream=st) as h:
            h.init_uniform(cfg.seed, cfg.lo, cfg.hi)
            h.run(a.nt)  # warm-up (+ graph capture where used)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e30
            for _ in range(a.reps):
                h.init_uniform(cfg.seed, cfg.lo, cfg.hi)
                e0.record(st)
                h.run(a.nt)
                e1.record(st)
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            info = h.info()
            # one profiled run: the timeline
            h.init_uniform(cfg.seed, cfg.lo, cfg.hi)
            h.set_profiling(True)
            h.run(a.nt)
            tr = h.trace()
            h.set_profiling(False)
        glups = cfg.N * a.nt / (best / 1e3) / 1e9
        rec = {"config": cfg.name, "nt": a.nt, "slabs": vs, "transport": transport if vs > 1 else "none",
               "T": info["T"], "mode": a.mode, "dp_ops": info["dp_ops"], "best_ms": best, "glups": glups}
        if vs > 1:
            k2 = [e for e in tr if e[1] == "K2"]
            halo = [e for e in tr if e[1] == "halo"]
            passes = len(halo)
            hidden, lag = 0, []
            for i, hv in enumerate(halo):
                ks = k2[i * vs:(i + 1) * vs]  # the pass's interior launches (one per slab)
                k0, k1 = min(e[2] for e in ks), max(e[3] for e in ks)
                hidden += hv[3] <= k1
                lag.append(hv[3] - k1)
            rec.update({"passes": passes, "halo_hidden_passes": hidden,
                        "halo_ms_median": sorted(e[3] - e[2] for e in halo)[passes // 2],
                        "k2_pass_ms_median": sorted(max(e[3] for e in k2[i * vs:(i + 1) * vs]) -
                                                    min(e[2] for e in k2[i * vs:(i + 1) * vs])
                                                    for i in range(passes))[passes // 2],
                        "halo_end_minus_interior_end_ms_max": max(lag),
                        "timeline_first_pass": [list(e) for e in tr[:vs + 1]]})
        results.append(rec)
        print(json.dumps(rec), flush=True)
    base = results[0]["glups"]
    summary = {"ratio_vs_one_slab": {"%s_%d" % (r["transport"], r["slabs"]): r["glups"] / base for r in results[1:]}}
    print(json.dumps(summary), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"results": results, "summary": summary}, f, indent=1)


if __name__ == "__main__":
    main()
