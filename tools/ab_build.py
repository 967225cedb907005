#!/usr/bin/env python
"""Build measurement variants of libheat1d.so with extra -D flags (A/B timing aid, not product).

    python tools/ab_build.py base= noguard=HEAT1D_NO_GUARD ...

Each NAME=DEF1,DEF2 builds paper_2307_01117_b200/build/variants/NAME.so; tools/ab_time.py
loads each in its own process (HEAT1D_LIB) and times the same workloads.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2307_01117_b200 import _build  # noqa: E402

out_dir = os.path.join(ROOT, "paper_2307_01117_b200", "build", "variants")
os.makedirs(out_dir, exist_ok=True)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    path = os.path.join(out_dir, name + ".so")
    _build.build(out=path, defines=[d for d in defs.split(",") if d])
    print(path)
