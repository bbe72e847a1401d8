"""Small launches of every forward kernel variant for compute-sanitizer (memcheck / racecheck /
synccheck): C1 chain (fwd_small), C3 layer 0 (fwd_tiled, balanced rows off, 4 j-blocks), C2 layer 0
(balanced rows, two x buffers), C3 L=128 (codes in global, GC), a C4-shaped 1024 -> 1024 layer on
2048 rows (transposed-input TMA boxes + TMEM f64 accumulators), the spline kernels and the compile
kernel. Usage: compute-sanitizer --tool racecheck python tools/sanitize_driver.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402


def run(tag, spec, X, L=64, scheme=0, bm=1, op=0, spline=False):
    a = lk.compile_layer(spec, lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme)),
                         lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op)))
    Y, st = lk.lut_layer_forward_batch(a, X)
    if spline:
        lk.layer_forward_batch(spec, X)
    torch.cuda.synchronize()
    print(f"{tag}: ok, oob {st.n_oob_inputs}/{st.n_inputs}", flush=True)


def main():
    Xc1 = torch.from_numpy(lk.recipe_inputs(1, 0, 4096)).cuda()
    ch = lk.compile_model([lk.recipe_layer(1, l) for l in range(2)], lk.QuantConfig(64),
                          lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX))
    lk.lut_model_forward_batch(ch, Xc1)
    print("C1 chain (fwd_chain_small, one launch): ok", flush=True)
    for a in ch:
        Xc1, _ = lk.lut_layer_forward_batch(a, Xc1)
    print("C1 layers (fwd_small): ok", flush=True)
    run("C2 layer 0 (fwd_tiled BAL, XB=2)", lk.recipe_layer(2, 0), torch.from_numpy(lk.recipe_inputs(2, 0, 3000)).cuda(),
        spline=True)
    X3 = torch.from_numpy(lk.recipe_inputs(3, 0, 2500)).cuda()
    run("C3 layer 0 (fwd_tiled, 4 j-blocks)", lk.recipe_layer(3, 0), X3, bm=0, op=1, spline=True)
    run("C3 layer 0 L=128 asym (codes in global)", lk.recipe_layer(3, 0), X3, L=128, scheme=1)
    spec4 = lk.gen_layer(5, 1024, 1024, 8)
    X4 = torch.empty((2048, 1024), device="cuda").uniform_(-1.2, 1.2)
    run("C4-shaped 1024->1024, 2048 rows (XT TMA boxes, TMEM f64)", spec4, X4, bm=0)
    run("C4-shaped 1024->1024, 2047 rows (row-major x, TMEM f64)", spec4, X4[:2047].contiguous(), bm=0)


if __name__ == "__main__":
    main()
