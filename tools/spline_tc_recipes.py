"""Tensor-core spline (spline_tc.cu) vs the f64 reference on the BASELINE recipe layers (the honest
baseline's parity bar: <= 1e-5 abs, 1e-5 rel where |y| > 1). Usage: python tools/spline_tc_recipes.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from helpers import to_oracle_spec  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

o = Oracle("auto")
for cfg, layer, rows in ((1, 0, 4096), (1, 1, 4096), (2, 0, 20000), (2, 1, 20000), (3, 0, 4000), (3, 1, 4000),
                         (4, 0, 256), (4, 1, 256), (4, 2, 1024), (4, 2, -256), (5, 0, 32)):
    spec = lk.recipe_layer(cfg, layer) if cfg != 5 else lk.recipe_layer(5, 0, 0, 256)
    wide = rows < 0      # tests/test_gpu_parity.py::test_spline_forward's hidden inputs U(-2.5, 2.5)
    rows = abs(rows)
    if layer == 0:
        X = lk.recipe_inputs(cfg, 0, rows)
    elif wide:
        X = np.random.default_rng(1000 * cfg + layer).uniform(-2.5, 2.5, (rows, spec.in_dim)).astype(np.float32)
    else:
        X = np.random.default_rng(cfg).uniform(-1.3, 1.3, (rows, spec.in_dim)).astype(np.float32)
    Y = lk.layer_forward_batch(spec, torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    Yo = o.spline_forward(to_oracle_spec(spec), X.astype(np.float64), 1, os.cpu_count() or 1)
    err = np.abs(Y - Yo)
    tol = np.where(np.abs(Yo) > 1, 1e-5 * np.abs(Yo), 1e-5)
    print(f"C{cfg} layer {layer} ({spec.in_dim}->{spec.out_dim}, {rows} rows): max|err| {err.max():.3e}, "
          f"worst err/tol {np.max(err / tol):.3f}, max|y| {np.abs(Yo).max():.3f}", flush=True)
