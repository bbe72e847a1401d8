"""Shared helpers for the GPU parity tests: conversions between oracle and product
objects, and the parity bar of BASELINE.json's north_star."""
import numpy as np

# north_star: float outputs agree within max-abs 1e-5 (relative 1e-5 where |y| > 1).
ABS_TOL = 1e-5
REL_TOL = 1e-5


def assert_close(y_gpu, y_ref, what=""):
    y_gpu = np.asarray(y_gpu, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    assert y_gpu.shape == y_ref.shape, (y_gpu.shape, y_ref.shape)
    err = np.abs(y_gpu - y_ref)
    big = np.abs(y_ref) > 1.0
    bad = np.where(big, err > REL_TOL * np.abs(y_ref), err > ABS_TOL)
    if bad.any():
        idx = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} outside 1e-5 (first {tuple(idx)}: "
                             f"gpu {y_gpu[tuple(idx)]!r} ref {y_ref[tuple(idx)]!r}); max abs {err.max():.3e}")
    return float(err.max()) if err.size else 0.0


def to_product_artifact(lk, a):
    """oracle.pyoracle.Artifact -> paper_2601_03332_b200.LutLayerArtifact (host arrays)."""
    sr = a.value_repr == 1
    return lk.LutLayerArtifact(
        a.in_dim, a.out_dim, a.L, a.value_repr, a.scheme, a.scheme, a.param_dtype,
        lk.OobConfig(lk.BoundaryMode(a.boundary_mode), lk.OobPolicy(a.oob_policy)), "silu" if sr else "",
        knots=a.knots, q_table=a.q, scale=a.scale, y_min=a.y_min,
        edge_base_scale=a.base_scale if sr else None, edge_spline_scale=a.spline_scale if sr else None,
        edge_out_scale=a.out_scale if sr else None, float_table=a.float_table)


def to_product_spec(lk, s):
    return lk.KanLayerSpec(s.in_dim, s.out_dim, lk.KnotGrid(np.asarray(s.breakpoints, np.float64), s.degree),
                           np.asarray(s.coeffs, np.float64).reshape(s.in_dim * s.out_dim, -1),
                           np.asarray(s.base_scale, np.float64), np.asarray(s.spline_scale, np.float64),
                           np.asarray(s.out_scale, np.float64))


def to_oracle_spec(s):
    from oracle.pyoracle import Spec
    return Spec(s.in_dim, s.out_dim, s.grid.breakpoints, s.coeffs, s.base_scale, s.spline_scale, s.out_scale,
                s.grid.degree)


def stats_list(st):
    return [int(st.n_samples), int(st.n_oob_samples), int(st.n_inputs), int(st.n_oob_inputs)]


def hidden_inputs(cfg, layer, rows, in_dim, lo=-1.3, hi=1.3):
    """Seeded fp32 inputs for a hidden layer tested on its own (per-layer parity)."""
    rng = np.random.default_rng(1000 * cfg + layer)
    return rng.uniform(lo, hi, size=(rows, in_dim)).astype(np.float32)
