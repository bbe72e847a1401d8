"""Throughput of GPU eval_accuracy (csrc/eval.cu) against the reference's metrics.cpp on the host.

Usage: python tools/bench_eval.py [cfg] [rows] [L] [cpu_rows]
Prints one JSON line: evaluations/s (rows x d x m per call) on the GPU (CUDA events around
lkg_eval_accuracy on device-resident X) and for the reference's eval_accuracy (oracle/_ref, all
host threads, a bounded row sample), plus the two reports' agreement."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from helpers import to_oracle_spec, to_product_artifact  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
L = int(sys.argv[3]) if len(sys.argv) > 3 else 64
cpu_rows = int(sys.argv[4]) if len(sys.argv) > 4 else 512

o = Oracle("auto")
spec = lk.recipe_layer(cfg, 0)
so = to_oracle_spec(spec)
ao = o.compile_layer(so, L, 0, 1, 0, 1, 0)
art = to_product_artifact(lk, ao)
X = lk.recipe_inputs(cfg, 0, rows)
evals = rows * spec.in_dim * spec.out_dim
eng = lk.default_engine()
Xd = torch.from_numpy(X).cuda()
r = lk.eval_accuracy(spec, art, Xd, engine=eng)  # warm-up (uploads spec and artifact)
st = torch.cuda.ExternalStream(eng.stream)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r = lk.eval_accuracy(spec, art, Xd, engine=eng)
    e1.record(st)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
nt = os.cpu_count() or 1
t0 = time.perf_counter()
ro = o.eval_accuracy(so, ao, X[:cpu_rows].astype(np.float64), nthreads=nt)
cpu_s = time.perf_counter() - t0
rs = lk.eval_accuracy(spec, art, X[:cpu_rows])
agree = (rs.n_inrange_evals == ro["n_inrange_evals"] and rs.n_oob_evals == ro["n_oob_evals"]
         and abs(rs.mae_inrange - ro["mae_inrange"]) <= 1e-9 * ro["mae_inrange"])
print(json.dumps({"metric": "eval_accuracy evaluations/s", "cfg": cfg, "L": L, "rows": rows,
                  "gpu": {"value": evals / (ms * 1e-3), "ms": ms},
                  "cpu_reference": {"value": cpu_rows * spec.in_dim * spec.out_dim / cpu_s, "threads": nt,
                                    "rows": cpu_rows, "kind": o.kind},
                  "mae_inrange": r.mae_inrange, "maxabs_inrange": r.maxabs_inrange, "mae_oob": r.mae_oob,
                  "agree_on_cpu_sample": bool(agree)}))
