#!/usr/bin/env python
"""A/B of K6 variants inside ONE process (box and clock effects cancel).
Variants are env knobs read at each launch: HEAT1D_K6_SPW, HEAT1D_K6_EARLY, HEAT1D_K6_RELAXED."""
import argparse, itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C5")
    p.add_argument("--nt", type=int, default=2000)
    p.add_argument("--T", nargs="*", type=int, default=[16, 32])
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    import torch
    import paper_2307_01117_b200 as h1
    from synth.configs import CONFIGS
    cfg = CONFIGS[a.config]
    st = torch.cuda.current_stream()
    variants = list(itertools.product([1, 2], [0, 1], [1]))  # spw, early, (relaxed: always)
    res = {}
    for T in a.T:
        with h1.Heat1D(cfg.nx, cfg.np, a.nt, cfg.k, cfg.dt, cfg.dx, T=T, resident=True, stream=st) as h:
            u0 = torch.from_numpy(cfg.u0()).cuda()
            for rep in range(a.reps + 1):
                for spw, early, relaxed in variants:
                    os.environ["HEAT1D_K6_SPW"] = str(spw)
                    os.environ["HEAT1D_K6_EARLY"] = str(early)
                    os.environ["HEAT1D_K6_RELAXED"] = str(relaxed)
                    h.set_initial(u0)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st); h.run(a.nt); e1.record(st); torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    if rep:
                        k = (T, spw, early, relaxed)
                        res[k] = min(res.get(k, 1e9), ms)
    for k, ms in sorted(res.items()):
        print(json.dumps({"config": a.config, "T": k[0], "spw": k[1], "early": k[2], "relaxed": k[3], "ms": round(ms, 3),
                          "glups": round(cfg.N * a.nt / (ms / 1e3) / 1e9, 1)}))

if __name__ == "__main__":
    main()
