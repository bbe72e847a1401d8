"""Time one layer forward (CUDA events, device-resident X) for kernel tuning experiments.
Usage: python tools/time_layer.py [workload] [layer] [iters] [L]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from bench import WORKLOADS  # noqa: E402
from paper_2601_03332_b200._capi import lib  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 50
cfg, rows, L, scheme, bm, op = WORKLOADS[wl]
if len(sys.argv) > 4:
    L = int(sys.argv[4])
dims, _, _, _ = lk.recipe_dims(cfg)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
eng = lk.Engine(0, s.cuda_stream)
a = lk.compile_layer(lk.recipe_layer(cfg, layer), lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme)),
                     lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op)), engine=eng)
dl = a.device(eng)
X = torch.from_numpy(lk.recipe_inputs(cfg, 0, rows)).cuda() if layer == 0 else \
    torch.empty((rows, dims[layer]), device="cuda").uniform_(-1.2, 1.2)
Y = torch.empty((rows, dims[layer + 1]), device="cuda")


def f():
    lib().lkg_layer_forward(eng.handle, dl.handle, C.c_void_p(X.data_ptr()), rows, C.c_void_p(Y.data_ptr()), None)


for _ in range(5):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(iters):
    f()
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
ee = rows * dims[layer] * dims[layer + 1]
print(f"{wl} layer {layer} cfg={os.environ.get('LKG_TILED_CFG', 'default')}: {ms:.4f} ms  {ee / ms / 1e9:.3e} edge-evals/s")
