"""Argmax-agreement report of a GPU chain forward against the reference (TEST INFRASTRUCTURE ONLY:
used by tests/test_fullsize.py and bench.py's CPU-baseline leg as the checker, never by the product).

SURVEY §8(c) parity protocol for chains: per layer, the reference is fed THE GPU'S OWN fp32 layer
input (float outputs within 1e-5, OobStats exact); end to end, the argmax class of the GPU chain is
compared with the reference's own chain on the same X (lut_model_forward_batch, runtime.cpp:298-314)
and every mismatching row must be explained by the per-layer diagnostics:

  * near_tie      — the reference chain's two top logits are within 2e-5 (twice the float bar), so
                    the <= 1e-5 per-layer float differences may order them either way;
  * knot_straddle — some hidden value of the row lies on the other side of a knot or of the mask edge
                    of the next layer than the reference's own hidden value (segment index k or the
                    in-range mask differ: the compiled table is discontinuous there), and
                    the reference's next layer evaluated on the GPU's hidden values picks the GPU's
                    class (the layer itself agrees; only the fp32-vs-f64 hidden value moved).

Anything else is `unexplained`, which the tests require to be 0.
"""
from __future__ import annotations

import numpy as np

TIE_TOL = 2e-5


def _top2_gap(Y: np.ndarray) -> np.ndarray:
    if Y.shape[1] < 2:
        return np.full(Y.shape[0], np.inf)
    s = np.sort(Y, axis=1)
    return s[:, -1] - s[:, -2]


def chain_agreement(oracle, chain_o, X: np.ndarray, hidden_gpu: list, Y_gpu: np.ndarray, nthreads: int = 1,
                    Y_ref_chain: np.ndarray | None = None) -> dict:
    """chain_o: oracle artifacts; X: fp32 [rows, d0]; hidden_gpu[l]: the GPU's output of layer l for
    l < n-1 (fp32); Y_gpu: the GPU chain output. Returns the report dict (counts are ints)."""
    n = len(chain_o)
    if Y_ref_chain is None:
        Y_ref_chain, _ = oracle.lut_model_forward(chain_o, X.astype(np.float64), 1, nthreads)
    cls_g = np.argmax(Y_gpu, axis=1)
    cls_r = np.argmax(Y_ref_chain, axis=1)
    mis = np.nonzero(cls_g != cls_r)[0]
    rep = {"rows": int(X.shape[0]), "agree": int(X.shape[0] - len(mis)), "mismatch": int(len(mis)),
           "near_tie": 0, "knot_straddle": 0, "unexplained": 0, "tie_tol": TIE_TOL, "rows_explained": []}
    if len(mis) == 0:
        rep["agreement"] = 1.0
        return rep
    # the reference's own hidden values on the mismatching rows (its chain, layer by layer)
    ref_hidden = []
    cur = X[mis].astype(np.float64)
    for l in range(n - 1):
        cur, _ = oracle.lut_forward(chain_o[l], cur, 1, 1)
        ref_hidden.append(cur)
    gap = _top2_gap(Y_ref_chain[mis])
    # the reference's last layer on the GPU's own last hidden values
    last_in = hidden_gpu[-1][mis].astype(np.float64) if n > 1 else X[mis].astype(np.float64)
    y_on_gpu_h, _ = oracle.lut_forward(chain_o[-1], last_in, 1, 1)
    for t, r in enumerate(mis):
        tie = bool(gap[t] < TIE_TOL)
        straddle = False
        for l in range(n - 1):
            hg = hidden_gpu[l][r].astype(np.float64)
            hr = ref_hidden[l][t]
            cg, cr = oracle.coords(chain_o[l + 1], hg), oracle.coords(chain_o[l + 1], hr)
            if np.any(cg["k"] != cr["k"]) or np.any(cg["in_range"] != cr["in_range"]):
                straddle = True
        layer_agrees = int(np.argmax(y_on_gpu_h[t])) == int(cls_g[r])
        kind = "near_tie" if tie else ("knot_straddle" if (straddle and layer_agrees) else "unexplained")
        rep[kind] += 1
        rep["rows_explained"].append({"row": int(r), "kind": kind, "logit_gap": float(gap[t]),
                                      "gpu_class": int(cls_g[r]), "ref_class": int(cls_r[r])})
    rep["rows_explained"] = rep["rows_explained"][:32]
    rep["agreement"] = rep["agree"] / rep["rows"]
    return rep
