"""Pin the CPU oracle before trusting it (CPU only, no GPU).

1. The plain-C restatement (oracle/lk_oracle.c) reproduces the committed reference
   digests (tests/golden/reference_digests.json, generated from the reference's own
   sources by tests/golden/make_golden.py) bit for bit: LUT bytes, scales, y_mins,
   forward outputs, OOB counts, spline outputs, RNG streams.
2. Where the in-place reference build exists (oracle/_ref), port == reference on fresh
   randomized cases.
3. The reference test suite's known answers hold for the oracle.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from kat import (ASYM_EXAMPLE, CARDINAL, HAND_CLOSED_CLIPX, HAND_CLOSED_ZS, HAND_HALFOPEN_ZS, SYM_EXAMPLE,
                 hand_artifact_arrays)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_digests.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _inputs(o, cfg, layer, rows, in_dim):
    if layer == 0:
        return o.recipe_inputs(cfg, 0, rows).astype(np.float64)
    rng = np.random.default_rng(1000 * cfg + layer)
    return rng.uniform(-1.3, 1.3, size=(rows, in_dim)).astype(np.float32).astype(np.float64)


def test_port_matches_reference_digests_compile_and_forward(port, golden):
    n = 0
    for c in golden["cases"]:
        if c.get("chain") or "y_opt" not in c:
            continue
        spec = port.recipe_layer(c["cfg"], c["layer"])
        art = port.compile_layer(spec, c["L"], c["scheme"], 1, 0, c["boundary_mode"], c["oob_policy"])
        assert sha(art.q) == c["q"] and sha(art.scale) == c["scale"] and sha(art.y_min) == c["y_min"], c
        X = _inputs(port, c["cfg"], c["layer"], c["rows"], spec.in_dim)
        Y, st = port.lut_forward(art, X, tier=1)
        assert sha(Y) == c["y_opt"], c
        assert [int(v) for v in st] == c["stats"], c
        Ys, _ = port.lut_forward(art, X[:64], tier=0)
        assert sha(Ys) == c["y_scalar64"], c
        assert sha(port.spline_forward(spec, X, tier=1)) == c["y_spline"], c
        n += 1
    assert n >= 40


def test_port_matches_reference_digests_repr_and_f16(port, golden):
    cases = [c for c in golden["cases"] if "value_repr" in c]
    assert len(cases) == 4
    spec = port.recipe_layer(2, 0)
    for c in cases:
        art = port.compile_layer(spec, c["L"], c["scheme"], c["value_repr"], c["param_dtype"], 1, 0)
        assert (sha(art.q), sha(art.scale), sha(art.y_min)) == (c["q"], c["scale"], c["y_min"]), c


def test_port_matches_reference_digests_chains(port, golden):
    cases = [c for c in golden["cases"] if c.get("chain")]
    assert cases
    for c in cases:
        chain = [port.compile_layer(port.recipe_layer(c["cfg"], l), c["L"], c["scheme"], 1, 0, c["boundary_mode"],
                                    c["oob_policy"]) for l in range(2)]
        X = port.recipe_inputs(c["cfg"], 0, c["rows"]).astype(np.float64)
        Y, st = port.lut_model_forward(chain, X)
        assert sha(Y) == c["y"] and st.astype(int).tolist() == c["stats"], c
        assert sha(np.argmax(Y, 1).astype(np.int64)) == c["argmax"]


def test_port_rng_streams(port, golden):
    g = golden["rng"]
    assert sha(port.rng_normal(7, 1000)) == g["normal_7"]
    assert sha(port.rng_uniform(7, 1000)) == g["uniform_7"]
    for cfg, h in g["inputs"].items():
        assert sha(port.recipe_inputs(int(cfg), 0, 64)) == h


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_port_equals_reference_randomized(port, ref, seed):
    """Fresh random specs (uneven knots, mixed gains) through both libraries."""
    from oracle.pyoracle import Spec
    rng = np.random.default_rng(seed)
    d, m, K, deg = int(rng.integers(1, 6)), int(rng.integers(1, 6)), int(rng.integers(1, 7)), int(rng.integers(0, 4))
    bp = np.cumsum(rng.uniform(0.1, 1.0, K + 1)) - 2.0
    E, R = d * m, K + deg
    spec = Spec(d, m, bp, rng.normal(0, 0.3, (E, R)), rng.uniform(-1, 1, E), rng.uniform(0.5, 1.5, E),
                rng.uniform(0.5, 1.5, E), deg)
    X = rng.uniform(bp[0] - 1, bp[-1] + 1, (300, d)).astype(np.float32).astype(np.float64)
    X[::17, 0] = bp[rng.integers(0, K + 1)]
    for L in (2, 7, 33):
        for scheme in (0, 1):
            for vr in (0, 1):
                for pd in (0, 1):
                    a = port.compile_layer(spec, L, scheme, vr, pd, seed % 2, (seed // 2) % 2, keep_float=True)
                    b = ref.compile_layer(spec, L, scheme, vr, pd, seed % 2, (seed // 2) % 2, keep_float=True)
                    assert np.array_equal(a.q, b.q) and np.array_equal(a.scale.view(np.uint32), b.scale.view(np.uint32))
                    assert np.array_equal(a.y_min.view(np.uint32), b.y_min.view(np.uint32))
                    assert np.array_equal(a.float_table, b.float_table)
                    for tier in (0, 1):
                        ya, sa = port.lut_forward(a, X, tier)
                        yb, sb = ref.lut_forward(b, X, tier)
                        assert np.array_equal(ya, yb) and np.array_equal(sa, sb)
    for tier in (0, 1):
        assert np.array_equal(port.spline_forward(spec, X, tier), ref.spline_forward(spec, X, tier))
    for vr in (0, 1):  # eval_accuracy (metrics.cpp:30-103), one thread: identical reports
        a = port.compile_layer(spec, 9, seed % 2, vr, 0, seed % 2, (seed // 2) % 2)
        assert port.eval_accuracy(spec, a, X) == ref.eval_accuracy(spec, a, X)


def test_port_matches_reference_eval_golden(port, golden):
    """eval_accuracy + memory_breakdown against the reference's reports (exact f64 values)."""
    assert len(golden["eval"]) >= 5
    for c in golden["eval"]:
        spec = port.recipe_layer(c["cfg"], 0)
        art = port.compile_layer(spec, c["L"], c["scheme"], c["value_repr"], 0, c["boundary_mode"], c["oob_policy"])
        r = port.eval_accuracy(spec, art, port.recipe_inputs(c["cfg"], 0, c["rows"]).astype(np.float64))
        for k, v in c["report"].items():
            assert r[k] == (float.fromhex(v) if isinstance(v, str) else v), (c, k)


def _hand(o, bm, op):
    from oracle.pyoracle import Artifact
    h = hand_artifact_arrays(bm, op)
    return Artifact(h["in_dim"], h["out_dim"], h["L"], h["knots"], h["q"], h["scale"], h["y_min"],
                    value_repr=0, scheme=1, boundary_mode=bm, oob_policy=op)


def test_kat_hand_table(oracle):
    a = _hand(oracle, 1, 0)
    for x, want, oob in HAND_CLOSED_CLIPX:
        v, o = oracle.eval_value(a, 0, x)
        assert v == pytest.approx(want, rel=1e-15, abs=0) and o == oob
    a = _hand(oracle, 0, 1)
    for x, want, oob in HAND_HALFOPEN_ZS:
        v, o = oracle.eval_value(a, 0, x)
        assert o == oob and (want is None or v == want)
    a = _hand(oracle, 0, 0)
    v, o = oracle.eval_value(a, 0, 2.0)  # one f32 ulp below the knot
    assert o and v < 70.0 and v == pytest.approx(70.0, rel=1e-6)
    a = _hand(oracle, 1, 1)
    for x, want, oob in HAND_CLOSED_ZS:
        assert oracle.eval_value(a, 0, x) == (want, oob)


def test_kat_coords(oracle):
    a = _hand(oracle, 1, 0)
    c = oracle.coords(a, np.array([0.0, 0.5, 1.0, 1.5, 2.0]))
    assert c["k"].tolist() == [0, 0, 1, 1, 1]                        # test_runtime.cpp:98-109
    assert (c["l0"][1], c["l1"][1], c["w"][1]) == (1, 2, 0.5)        # u=.5, L=4 -> (1,2,.5)
    assert (c["l0"][4], c["l1"][4], c["w"][4]) == (3, 3, 0.0)        # u=1 -> (L-1, L-1, 0)
    ho = _hand(oracle, 0, 0)
    c = oracle.coords(ho, np.array([2.0, 9.0]))
    assert c["x_clip"][0] == float(np.nextafter(np.float32(2), np.float32(-np.inf)))
    assert not c["in_range"][0]


def test_kat_quantization(oracle):
    v, q, s = SYM_EXAMPLE
    qq, sc, ym = oracle.quantize_segment(v, 0)
    assert qq.tolist() == q and sc == pytest.approx(s, rel=1e-12) and ym == 0.0
    v, q, s, y = ASYM_EXAMPLE
    qq, sc, ym = oracle.quantize_segment(v, 1)
    assert qq.tolist() == q and sc == pytest.approx(s, rel=1e-12) and ym == y
    qq, sc, ym = oracle.quantize_segment([5.0, 5.0, 5.0], 1)   # degenerate
    assert sc == 0.0 and qq.tolist() == [0, 0, 0]


def test_kat_f16_and_basis(oracle):
    for f in (0.0, 1.0, -2.5, 65504.0, 2.0**-14, 2.0**-24):
        assert oracle.f16_round(f) == f
    assert math.isinf(oracle.f16_round(70000.0))
    for bp, deg, x, want in CARDINAL:
        assert np.allclose(oracle.basis_values(np.array(bp), deg, x), want, atol=1e-15)


def test_oob_stats_kat(oracle):
    """test_runtime.cpp:346-370: per-coordinate and per-sample OOB counting."""
    spec = oracle.recipe_layer(1, 0)
    spec = spec.edge_slice(0, 2)
    spec = type(spec)(2, 1, spec.breakpoints, spec.coeffs[::5][:2], spec.base_scale[:2], spec.spline_scale[:2],
                      spec.out_scale[:2])
    a = oracle.compile_layer(spec, 8, 0, 1, 0, 0, 0)
    tK = spec.breakpoints[-1]
    X = np.array([[0.0, 0.0], [tK, 0.0], [tK, tK + 5.0]])
    _, st = oracle.lut_forward(a, X)
    assert st.tolist() == [3, 2, 6, 3]


def test_nonfinite_rejected(oracle):
    from oracle.pyoracle import OracleError
    a = _hand(oracle, 1, 0)
    with pytest.raises(OracleError) as e:
        oracle.lut_forward(a, np.array([[-np.inf]]))
    assert e.value.code == 3


def test_reference_chain_session_matches_direct_call():
    """bench.py times the reference through a prepared session (artifacts converted and per-thread
    Matrix shards cut outside the timed region): same outputs and OobStats as the direct call."""
    from oracle.pyoracle import Oracle
    o = Oracle("auto")
    chain = [o.compile_layer(o.recipe_layer(2, l), 64, 1, 1, 0, 1, 0) for l in range(2)]
    X = o.recipe_inputs(2, 0, 5001).astype(np.float64)
    sess = o.chain_session(chain, X, 1, 3)
    if sess is None:
        pytest.skip("the C port has no session entry (reference library only)")
    Y, st = o.lut_model_forward(chain, X, 1, 3)
    for _ in range(2):
        Y2, st2 = sess.run()
        assert np.array_equal(Y, Y2) and np.array_equal(st, st2)
    sess.close()
