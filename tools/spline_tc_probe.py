"""First-light probe of the tensor-core spline (spline_tc.cu): tiny shapes against the SIMT spline
kernel and the f64 oracle. Usage: python tools/spline_tc_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from oracle.pyoracle import Oracle, Spec  # noqa: E402

o = Oracle("auto")
for (d, m, G, rows) in ((8, 16, 5, 128), (78, 16, 5, 1000), (64, 64, 8, 3000), (300, 40, 8, 777), (1024, 128, 8, 512)):
    spec = lk.gen_layer(7, d, m, G)
    X = np.random.default_rng(1).uniform(-1.3, 1.3, (rows, d)).astype(np.float32)
    Y = lk.layer_forward_batch(spec, torch.from_numpy(X).cuda()).cpu().numpy()
    so = Spec(spec.in_dim, spec.out_dim, spec.grid.breakpoints, spec.coeffs, spec.base_scale, spec.spline_scale,
              spec.out_scale, 3)
    Yo = o.spline_forward(so, X.astype(np.float64), 1, 8)
    err = np.abs(Y - Yo)
    print(f"d={d} m={m} G={G} rows={rows}: max|err| {err.max():.3e} (max|y| {np.abs(Yo).max():.3f})", flush=True)
