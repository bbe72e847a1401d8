"""Time the same-GPU spline forward (tensor-core GEMM form by default, LKG_SPLINE_SIMT=1 for the SIMT
table kernel) on a workload's layer, next to the LUT layer forward. Usage:
python tools/time_spline.py [workload] [layer] [iters]"""
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
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cfg, rows, L, scheme, bm, op = WORKLOADS[wl]
dims, _, _, _ = lk.recipe_dims(cfg)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
eng = lk.Engine(0, s.cuda_stream)
spec = lk.recipe_layer(cfg, layer)
sd = spec.device(eng)
X = torch.from_numpy(lk.recipe_inputs(cfg, 0, rows)).cuda() if layer == 0 else \
    torch.empty((rows, dims[layer]), device="cuda").uniform_(-1.2, 1.2)
Y = torch.empty((rows, dims[layer + 1]), device="cuda")


def f():
    lk.lutkan.check(lib().lkg_spline_forward(eng.handle, sd.handle, C.c_void_p(X.data_ptr()), rows,
                                             C.c_void_p(Y.data_ptr())))


for _ in range(2):
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
mode = "SIMT" if os.environ.get("LKG_SPLINE_SIMT") == "1" else "TC"
print(f"spline[{mode}] {wl} layer {layer}: {ms:.4f} ms  {ee / ms * 1e3:.3e} edge-evals/s")
