#!/usr/bin/env python
"""Time variant builds (tools/ab_build.py) on the same workloads, one process per variant.

    python tools/ab_time.py --variants base noguard --N 268435456 --nt 384 --cases 0.5:matched 0.4:matched:64:51,4,2,2,3

A case is k:mode[:T[:geometry]] (geometry = HEAT1D_GEOM "V,NW,S,ctas,kind").

Prints one JSON line per (variant, case): best-of-reps GLUPS of heat1d_run (CUDA events).
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, torch
sys.path.insert(0, %(root)r)
import paper_2307_01117_b200 as h1
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
for case in %(cases)r:
    parts = case.split(":")
    k, mode = float(parts[0]), parts[1]
    T = int(parts[2]) if len(parts) > 2 and parts[2] else 0
    if len(parts) > 3 and parts[3]:
        os.environ["HEAT1D_GEOM"] = parts[3]   # read at create
    else:
        os.environ.pop("HEAT1D_GEOM", None)
    try:
      with h1.Heat1D(%(N)d, 1, %(nt)d, k, 1.0, 1.0, T=T, mode=mode, stream=st, resident=%(resident)s,
                   virtual_slabs=%(vs)d) as h:
        h.init_uniform(1234, -1.0, 1.0)
        h.run(%(nt)d)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(%(reps)d):
            e0.record(st); h.run(%(nt)d); e1.record(st); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        info = h.info()
    except Exception as ex:
        print(json.dumps({"variant": %(name)r, "case": case, "error": str(ex)[:100]}), flush=True)
        continue
    print(json.dumps({"variant": %(name)r, "case": case, "T": info["T"], "ops": info["dp_ops"],
                      "geom": "%%d,%%d,%%d,k%%d" %% (info["pass_V"], info["pass_NW"], info["pass_S"], info["pass_kind"]),
                      "glups": round(%(N)d * %(nt)d / (best / 1e3) / 1e9, 1), "ms": round(best, 3)}), flush=True)
'''


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--variants", nargs="+", required=True)
    p.add_argument("--N", type=int, default=1 << 28)
    p.add_argument("--nt", type=int, default=384)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--cases", nargs="+", default=["0.5:matched", "0.4:matched", "0.5:fast"])
    p.add_argument("--resident", default="False")
    p.add_argument("--vs", type=int, default=1)
    a = p.parse_args()
    for rnd in range(2):  # two rounds, interleaved, to expose drift
        for v in a.variants:
            lib = os.path.join(ROOT, "paper_2307_01117_b200", "build", "variants", v + ".so")
            env = dict(os.environ, HEAT1D_LIB=lib)
            code = CHILD % dict(root=ROOT, cases=a.cases, N=a.N, nt=a.nt, reps=a.reps, name=v + "#%d" % rnd,
                                resident=a.resident, vs=a.vs)
            subprocess.run([sys.executable, "-c", code], env=env, check=False)


if __name__ == "__main__":
    main()
