import os, sys
sys.path.insert(0, '/root/repo')
import paper_2307_01117_b200 as h1
for sync in ("0", "3"):
    os.environ["HEAT1D_K6_SYNC"] = sync
    for k, mode in ((0.4, "matched"), (0.5, "matched"), (0.4, "fast"), (0.5, "fast")):
        for T in (16, 32, 64):
            try:
                with h1.Heat1D(1_400_000, 1, 10, k, 1.0, 1.0, T=T, mode=mode, resident=True) as h:
                    print(sync, k, mode, T, "fits", h.info()["dp_ops"])
            except h1.Heat1DError as e:
                print(sync, k, mode, T, "NO", e)
