import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HEAT1D_DEBUG"] = "1"
import torch, numpy as np
import paper_2307_01117_b200 as h1
for N, T in [(1_400_000, 1), (1_400_000, 16), (1, 5), (1_000_000, 1)]:
    try:
        with h1.Heat1D(N, 1, 10, 0.4, 1.0, 1.0, T=T, resident=True) as h:
            print("created", N, T, h.info()["T"], flush=True)
            h.set_initial(np.zeros(N))
            h.run(3 * T + 2)
            print("ok", N, T, flush=True)
    except Exception as e:
        print("ERR", N, T, e, flush=True)
        import ctypes
        print("last", torch.cuda.is_available())
