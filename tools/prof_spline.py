"""Profiling driver for the spline kernels: a workload layer's spline forward launched a few times
(no timing), for ncu -k regex:spline. Usage: python tools/prof_spline.py [workload] [layer] [iters]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from bench import WORKLOADS  # noqa: E402
from paper_2601_03332_b200._capi import lib  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg, rows, L, scheme, bm, op = WORKLOADS[wl]
dims, _, _, _ = lk.recipe_dims(cfg)
eng = lk.Engine(0)
spec = lk.recipe_layer(cfg, layer)
sd = spec.device(eng)
X = torch.from_numpy(lk.recipe_inputs(cfg, 0, rows)).cuda() if layer == 0 else \
    torch.empty((rows, dims[layer]), device="cuda").uniform_(-1.2, 1.2)
Y = torch.empty((rows, dims[layer + 1]), device="cuda")
torch.cuda.synchronize()
for _ in range(iters):
    lk.lutkan.check(lib().lkg_spline_forward(eng.handle, sd.handle, C.c_void_p(X.data_ptr()), rows,
                                             C.c_void_p(Y.data_ptr())))
torch.cuda.synchronize()
