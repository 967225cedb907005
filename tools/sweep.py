#!/usr/bin/env python
"""Tuning sweep of the pass kernel: (geometry, T, arithmetic) on an HBM-resident ring.

    python tools/sweep.py --N 268435456 --nt 240 --geoms 17,8,3,2 25,8,3,1 --T 8 12 16 --k 0.4 0.5

Times heat1d_run with CUDA events (3 repetitions after 1 warm-up), prints one
JSON line per point.  Not part of the product; a measurement aid.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--N", type=int, default=1 << 28)
    p.add_argument("--nt", type=int, default=240)
    p.add_argument("--geoms", nargs="*", default=[""])
    p.add_argument("--T", nargs="*", type=int, default=[8, 12, 16])
    p.add_argument("--k", nargs="*", type=float, default=[0.4, 0.5])
    p.add_argument("--mode", default="matched")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    import torch
    import paper_2307_01117_b200 as h1
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    for g in a.geoms:
        if g:
            os.environ["HEAT1D_GEOM"] = g
        else:
            os.environ.pop("HEAT1D_GEOM", None)
        for k in a.k:
            for T in a.T:
              try:
                with h1.Heat1D(a.N, 1, a.nt, k, 1.0, 1.0, T=T, mode=a.mode, stream=st) as h:
                    h.init_uniform(1234, -1.0, 1.0)
                    h.run(a.nt)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    best = 1e30
                    for _ in range(a.reps):
                        e0.record(st)
                        h.run(a.nt)
                        e1.record(st)
                        torch.cuda.synchronize()
                        best = min(best, e0.elapsed_time(e1))
                    info = h.info()
                glups = a.N * a.nt / (best / 1e3) / 1e9
                roof = min(6544.0 * T / 16.0, 9306.0)
                print(json.dumps({"geom": g or "auto", "k": k, "T": T, "ops": info["dp_ops"], "mode": a.mode,
                                  "glups": round(glups, 1), "frac": round(glups / roof, 3), "ms": round(best, 3),
                                  "grid": info["grid"], "tile": info["tile_cells"]}), flush=True)
              except Exception as e:  # noqa: BLE001 -- an invalid geometry for this T: skip the point
                print(json.dumps({"geom": g or "auto", "k": k, "T": T, "mode": a.mode, "error": str(e)[:120]}),
                      flush=True)


if __name__ == "__main__":
    main()
