"""Per-call latency of a small chain forward (configs[0] = C1 [2,5,1], 4096 rows by default):
direct C-ABI calls (lkg_model_forward per call) against a CUDA-graph replay (lkg_graph_launch),
both on device-resident buffers, back to back; host wall time per call and device time per call.
Usage: python tools/latency.py [cfg] [rows] [iters]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json  # noqa: E402

import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from paper_2601_03332_b200._capi import lib  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
dims, _, _, _ = lk.recipe_dims(cfg)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
eng = lk.Engine(0, s.cuda_stream)
oob = lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX) if cfg == 1 else lk.OobConfig()
chain = [lk.compile_layer(lk.recipe_layer(cfg, l), lk.QuantConfig(64), oob, engine=eng) for l in range(len(dims) - 1)]
dev = [a.device(eng) for a in chain]
hs = (C.c_void_p * len(dev))(*[d.handle for d in dev])
X = torch.from_numpy(lk.recipe_inputs(cfg, 0, rows)).cuda()
Y = torch.empty((rows, dims[-1]), device="cuda")


def direct():
    lib().lkg_model_forward(eng.handle, hs, len(dev), C.c_void_p(X.data_ptr()), rows, C.c_void_p(Y.data_ptr()), None)


g = lk.ChainGraph(chain, X, Y, engine=eng)
out = {"cfg": f"configs[{cfg - 1}]", "dims": dims, "rows": rows, "iters": iters}
for name, fn in (("direct", direct), ("graph", g)):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    out[name] = {"device_us_per_call": e0.elapsed_time(e1) * 1e3 / iters,
                 "host_us_per_call": (time.perf_counter() - t0) * 1e6 / iters,
                 "kernels_per_call": None}
    eng.collect(len(dev))
print(json.dumps(out))
