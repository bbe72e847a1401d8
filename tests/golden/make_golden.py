"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container, where /root/reference exists:
    make -C oracle ref && python tests/golden/make_golden.py
It loads oracle/_ref/liblutkan_ref.so — the reference's own sources compiled in place
(oracle/Makefile) — and records, for seeded BASELINE-shaped inputs:
  * SHA-256 digests of compiled q_table / scale / y_min bytes (compile_layer),
  * SHA-256 digests of lut_layer_forward_batch / lut_model_forward_batch outputs (f64
    bits) and OobStats, and of layer_forward_batch (spline) outputs,
  * eval_accuracy reports (metrics.cpp), exact f64 values as hex,
  * a few explicit values for readability.
tests/test_oracle.py checks the plain-C restatement (oracle/lk_oracle.c) against these
digests, so the port is pinned to the reference even where /root/reference is absent.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.pyoracle import Oracle  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    o = Oracle("reference")
    assert o.kind == "reference"
    out = {"generator": "tests/golden/make_golden.py", "oracle": "oracle/_ref (reference sources)", "cases": []}
    # C1..C3 layer 0/1 compile + forward at small batches; all 32 C3 cells at L in {16, 128} x schemes x OOB.
    plans = []
    for cfg, rows in ((1, 4096), (2, 2000), (3, 512)):
        for layer in (0, 1):
            for L in ((64,) if cfg != 3 else (16, 32, 64, 128)):
                for scheme in (0, 1):
                    for bm in (0, 1):
                        for op in (0, 1):
                            if cfg != 3 and (bm, op) not in ((0, 0), (1, 1)):
                                continue
                            plans.append((cfg, layer, L, scheme, bm, op, rows))
    for cfg, layer, L, scheme, bm, op, rows in plans:
        spec = o.recipe_layer(cfg, layer)
        art = o.compile_layer(spec, L, scheme, 1, 0, bm, op)
        if layer == 0:
            X = o.recipe_inputs(cfg, 0, rows).astype(np.float64)
        else:  # hidden-layer inputs: seeded uniform over 1.3x the knot range
            rng = np.random.default_rng(1000 * cfg + layer)
            X = rng.uniform(-1.3, 1.3, size=(rows, spec.in_dim)).astype(np.float32).astype(np.float64)
        Y, st = o.lut_forward(art, X, tier=1)
        Ys, _ = o.lut_forward(art, X[:64], tier=0)
        Yspl = o.spline_forward(spec, X, tier=1)
        out["cases"].append(dict(
            cfg=cfg, layer=layer, L=L, scheme=scheme, boundary_mode=bm, oob_policy=op, rows=rows,
            q=sha(art.q), scale=sha(art.scale), y_min=sha(art.y_min), y_opt=sha(Y), y_scalar64=sha(Ys),
            y_spline=sha(Yspl), stats=[int(v) for v in st], y00=float(Y[0, 0]), yspl00=float(Yspl[0, 0])))
    # f16 params and phi representation on C2 layer 0
    spec = o.recipe_layer(2, 0)
    for vr in (0, 1):
        for pd in (0, 1):
            art = o.compile_layer(spec, 32, 1, vr, pd, 1, 0)
            out["cases"].append(dict(cfg=2, layer=0, L=32, scheme=1, value_repr=vr, param_dtype=pd,
                                     q=sha(art.q), scale=sha(art.scale), y_min=sha(art.y_min)))
    # chained C1 / C2 models
    for cfg, rows, L, scheme, bm, op in ((1, 4096, 64, 0, 0, 0), (2, 2000, 64, 0, 1, 0), (2, 2000, 64, 1, 1, 0)):
        chain = [o.compile_layer(o.recipe_layer(cfg, l), L, scheme, 1, 0, bm, op) for l in range(2)]
        X = o.recipe_inputs(cfg, 0, rows).astype(np.float64)
        Y, st = o.lut_model_forward(chain, X)
        out["cases"].append(dict(cfg=cfg, chain=True, L=L, scheme=scheme, boundary_mode=bm, oob_policy=op, rows=rows,
                                 y=sha(Y), stats=st.astype(int).tolist(), argmax=sha(np.argmax(Y, 1).astype(np.int64))))
    # eval_accuracy (metrics.cpp:30-103): exact values (f64 repr) on C1 / C3 cells
    out["eval"] = []
    for cfg, rows, L, scheme, bm, op, vr in ((1, 512, 64, 0, 0, 0, 1), (1, 512, 16, 1, 1, 1, 1), (3, 128, 16, 0, 1, 0, 1),
                                             (3, 128, 32, 1, 0, 1, 1), (3, 128, 16, 1, 1, 1, 0)):
        spec = o.recipe_layer(cfg, 0)
        art = o.compile_layer(spec, L, scheme, vr, 0, bm, op)
        X = o.recipe_inputs(cfg, 0, rows).astype(np.float64)
        r = o.eval_accuracy(spec, art, X)
        out["eval"].append(dict(cfg=cfg, rows=rows, L=L, scheme=scheme, boundary_mode=bm, oob_policy=op, value_repr=vr,
                                report={k: (float(v).hex() if isinstance(v, float) else v) for k, v in r.items()}))
    # rng / input streams
    out["rng"] = dict(normal_7=sha(o.rng_normal(7, 1000)), uniform_7=sha(o.rng_uniform(7, 1000)),
                      inputs={str(c): sha(o.recipe_inputs(c, 0, 64)) for c in (1, 2, 3, 4, 5)})
    with open(os.path.join(HERE, "reference_digests.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {len(out['cases'])} cases")


if __name__ == "__main__":
    main()
