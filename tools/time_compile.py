"""Compile (K1) timing per workload: cold (first in the process: lazy module loading, first
allocations) and warm (repeat), host wall clock around compile_layer for every layer incl. the
spec upload. Usage: python tools/time_compile.py [workload ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_03332_b200 as lk  # noqa: E402
from bench import WORKLOADS  # noqa: E402

eng = lk.Engine(0)
for wl in sys.argv[1:] or ["c2"]:
    cfg, rows, L, scheme, bm, op = WORKLOADS[wl]
    dims, _, _, _ = lk.recipe_dims(cfg)
    qc = lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme))
    oob = lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op))
    for rep in range(3):
        specs = [lk.recipe_layer(cfg, l) for l in range(len(dims) - 1)]
        t0 = time.perf_counter()
        arts = [lk.compile_layer(s, qc, oob, engine=eng) for s in specs]
        eng.synchronize()
        t1 = time.perf_counter()
        print(f"{wl} rep {rep}: {1e3 * (t1 - t0):.2f} ms ({len(specs)} layers)", flush=True)
        del arts, specs
