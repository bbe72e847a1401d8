"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads either the plain-C restatement (``oracle/liblk_oracle.so``, kind "port") or
the reference's own sources built in place (``oracle/_ref/liblutkan_ref.so``,
kind "reference"); both export ``oracle/lk_oracle.h``. Only tests/, smoke() and
bench.py's CPU-baseline legs import this module — the product never does.

Arrays follow the reference layouts: edges input-major ``e = i*m + j``
(spline.hpp:43), q_table ``[E, K, L]``, scale / y_min ``[E, K]``
(runtime.hpp:31-63).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liblk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblutkan_ref.so")

_P = C.POINTER
_f64p, _f32p, _u8p = _P(C.c_double), _P(C.c_float), _P(C.c_uint8)
_i32p, _u64p = _P(C.c_int32), _P(C.c_uint64)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class _Spec(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("out_dim", C.c_int32), ("K", C.c_int32), ("degree", C.c_int32),
                ("breakpoints", _f64p), ("coeffs", _f64p), ("base_scale", _f64p),
                ("spline_scale", _f64p), ("out_scale", _f64p)]


class _Art(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("out_dim", C.c_int32), ("K", C.c_int32), ("L", C.c_int32),
                ("value_repr", C.c_int32), ("scheme", C.c_int32), ("param_dtype", C.c_int32),
                ("boundary_mode", C.c_int32), ("oob_policy", C.c_int32),
                ("knots", _f32p), ("q", _u8p), ("scale", _f32p), ("y_min", _f32p),
                ("base_scale", _f32p), ("spline_scale", _f32p), ("out_scale", _f32p),
                ("float_table", _f64p)]


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


@dataclass
class Spec:
    """KanLayerSpec (spline.hpp:35-74) as numpy arrays."""
    in_dim: int
    out_dim: int
    breakpoints: np.ndarray          # f64 [K+1]
    coeffs: np.ndarray               # f64 [E, R]
    base_scale: np.ndarray           # f64 [E]
    spline_scale: np.ndarray
    out_scale: np.ndarray
    degree: int = 3

    @property
    def K(self):
        return len(self.breakpoints) - 1

    def _c(self):
        self._keep = [np.ascontiguousarray(x, np.float64) for x in
                      (self.breakpoints, self.coeffs, self.base_scale, self.spline_scale, self.out_scale)]
        b, c, bs, ss, os_ = self._keep
        return _Spec(self.in_dim, self.out_dim, self.K, self.degree, _ptr(b, _f64p), _ptr(c, _f64p),
                     _ptr(bs, _f64p), _ptr(ss, _f64p), _ptr(os_, _f64p))

    def edge_slice(self, i0: int, i1: int) -> "Spec":
        """Sub-spec of input rows [i0, i1): compiles to bytes [(i0*m)*K*L, (i1*m)*K*L)."""
        m = self.out_dim
        sl = slice(i0 * m, i1 * m)
        return Spec(i1 - i0, m, self.breakpoints, self.coeffs[sl], self.base_scale[sl],
                    self.spline_scale[sl], self.out_scale[sl], self.degree)


@dataclass
class Artifact:
    """LutLayerArtifact (runtime.hpp:31-63) as numpy arrays."""
    in_dim: int
    out_dim: int
    L: int
    knots: np.ndarray                # f32 [K+1]
    q: np.ndarray                    # u8 [E*K*L]
    scale: np.ndarray                # f32 [E*K]
    y_min: np.ndarray                # f32 [E*K]
    base_scale: np.ndarray | None = None
    spline_scale: np.ndarray | None = None
    out_scale: np.ndarray | None = None
    value_repr: int = 1              # 0 phi, 1 spline_component
    scheme: int = 0                  # 0 symmetric/int8, 1 asymmetric/uint8
    param_dtype: int = 0
    boundary_mode: int = 1           # 0 half_open, 1 closed (runtime.hpp:19-22 default closed)
    oob_policy: int = 0              # 0 clip_x, 1 zero_spline
    float_table: np.ndarray | None = None
    _keep: list = field(default_factory=list, repr=False)

    @property
    def K(self):
        return len(self.knots) - 1

    def _c(self):
        conv = lambda a, t: None if a is None else np.ascontiguousarray(a, t)
        kn, q, sc, ym = conv(self.knots, np.float32), conv(self.q, np.uint8), conv(self.scale, np.float32), conv(self.y_min, np.float32)
        bs, ss, os_ = conv(self.base_scale, np.float32), conv(self.spline_scale, np.float32), conv(self.out_scale, np.float32)
        ft = conv(self.float_table, np.float64)
        self._keep = [kn, q, sc, ym, bs, ss, os_, ft]
        return _Art(self.in_dim, self.out_dim, self.K, self.L, self.value_repr, self.scheme, self.param_dtype,
                    self.boundary_mode, self.oob_policy, _ptr(kn, _f32p), _ptr(q, _u8p), _ptr(sc, _f32p),
                    _ptr(ym, _f32p), _ptr(bs, _f32p), _ptr(ss, _f32p), _ptr(os_, _f32p), _ptr(ft, _f64p))


def build(ref: bool = True) -> None:
    """Build the port (always) and the in-place reference build (only where /root/reference exists)."""
    targets = ["port"]
    if ref and os.path.isdir("/root/reference/proj/core/src"):
        targets += ["ref", "sweep"]  # sweep: the reference's run_sweep/collect_results (tests/test_sweep.py)
        lib = os.path.join(os.path.dirname(HERE), "paper_2601_03332_b200", "liblutkan_b200.so")
        if os.path.exists(lib):
            targets.append("shim")  # C++ drop-in shim test against the reference library
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class _ChainSession:
    def __init__(self, o, chain, X, tier, nthreads):
        X = np.ascontiguousarray(X, np.float64)
        self.o, self.rows, self.n = o, X.shape[0], len(chain)
        arr = (_Art * len(chain))(*[a._c() for a in chain])
        o.lib.ork_chain_session_create.restype = C.c_void_p
        self.h = o.lib.ork_chain_session_create(arr, len(chain), _ptr(X, _f64p), self.rows, tier, nthreads)
        if not self.h:
            raise RuntimeError("ork_chain_session_create failed")
        self.Y = np.zeros((self.rows, chain[-1].out_dim), np.float64)
        self.st = np.zeros((len(chain), 4), np.uint64)

    def run(self):
        self.o._chk(self.o.lib.ork_chain_session_run(C.c_void_p(self.h), _ptr(self.Y, _f64p), _ptr(self.st, _u64p)))
        return self.Y, self.st

    def close(self):
        if self.h:
            self.o.lib.ork_chain_session_free.restype = None
            self.o.lib.ork_chain_session_free(C.c_void_p(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Oracle:
    def __init__(self, kind: str = "auto"):
        if kind == "auto":
            kind = "reference" if os.path.exists(REF_SO) else "port"
        path = REF_SO if kind == "reference" else PORT_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.kind = kind
        self.lib = L = C.CDLL(path)
        L.ork_last_error.restype = C.c_char_p
        L.ork_impl_name.restype = C.c_char_p
        L.ork_compile_layer.argtypes = [_P(_Spec), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, _f32p, _u8p, _f32p, _f32p, _f32p, _f32p, _f32p, _f64p]
        L.ork_lut_forward.argtypes = [_P(_Art), _f64p, C.c_int64, C.c_int32, C.c_int32, _f64p, _u64p]
        L.ork_lut_model_forward.argtypes = [_P(_Art), C.c_int32, _f64p, C.c_int64, C.c_int32, C.c_int32,
                                            _f64p, _u64p]
        L.ork_spline_forward.argtypes = [_P(_Spec), _f64p, C.c_int64, C.c_int32, C.c_int32, _f64p]
        L.ork_coords.argtypes = [_P(_Art), _f64p, C.c_int64, _u8p, _f64p, _i32p, _i32p, _i32p, _f64p]
        L.ork_gen_layer.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _f64p, _f64p, _f64p,
                                    _f64p, _f64p]
        L.ork_gen_inputs.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, _f64p]
        L.ork_artifact_save.argtypes = [_P(_Art), C.c_char_p]
        L.ork_artifact_load_resave.argtypes = [C.c_char_p, C.c_char_p]
        L.ork_eval_accuracy.argtypes = [_P(_Spec), _P(_Art), _f64p, C.c_int64, C.c_int32, _f64p, _u64p, _i32p]
        L.ork_eval_value.argtypes = [_P(_Art), C.c_int32, C.c_double, _f64p, _i32p]
        L.ork_eval_phi.argtypes = [_P(_Art), C.c_int32, C.c_double, _f64p]
        L.ork_basis_values.argtypes = [_f64p, C.c_int32, C.c_int32, C.c_double, _f64p]
        L.ork_quantize_segment.argtypes = [_f64p, C.c_int32, C.c_int32, _i32p, _f64p, _f64p]
        L.ork_f32_to_f16_bits.argtypes = [C.c_float]
        L.ork_f32_to_f16_bits.restype = C.c_uint16
        L.ork_f16_bits_to_f32.argtypes = [C.c_uint16]
        L.ork_f16_bits_to_f32.restype = C.c_float
        L.ork_rng_uniform.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.ork_rng_normal.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.ork_recipe_layer.argtypes = [C.c_int32, C.c_int32, _f64p, _f64p, _f64p, _f64p, _f64p]
        L.ork_recipe_inputs.argtypes = [C.c_int32, C.c_int64, C.c_int64, _f32p]

    def _chk(self, st):
        if st != 0:
            raise OracleError(st, self.lib.ork_last_error().decode())

    # --------------------------------------------------------------- compile
    def compile_layer(self, spec: Spec, L: int = 64, scheme: int = 0, value_repr: int = 1,
                      param_dtype: int = 0, boundary_mode: int = 1, oob_policy: int = 0,
                      keep_float: bool = False) -> Artifact:
        E, K = spec.in_dim * spec.out_dim, spec.K
        knots = np.zeros(K + 1, np.float32)
        q = np.zeros(E * K * L, np.uint8)
        sc = np.zeros(E * K, np.float32)
        ym = np.zeros(E * K, np.float32)
        gains = [np.zeros(E, np.float32) for _ in range(3)] if value_repr == 1 else [None] * 3
        ft = np.zeros(E * K * L, np.float64) if keep_float else None
        cs = spec._c()
        self._chk(self.lib.ork_compile_layer(C.byref(cs), L, scheme, value_repr, param_dtype, boundary_mode,
                                             oob_policy, _ptr(knots, _f32p), _ptr(q, _u8p), _ptr(sc, _f32p),
                                             _ptr(ym, _f32p), *[_ptr(g, _f32p) for g in gains], _ptr(ft, _f64p)))
        return Artifact(spec.in_dim, spec.out_dim, L, knots, q, sc, ym, *gains, value_repr=value_repr,
                        scheme=scheme, param_dtype=param_dtype, boundary_mode=boundary_mode,
                        oob_policy=oob_policy, float_table=ft)

    # --------------------------------------------------------------- forward
    def lut_forward(self, a: Artifact, X: np.ndarray, tier: int = 1, nthreads: int = 1):
        X = np.ascontiguousarray(X, np.float64)
        rows = X.shape[0]
        Y = np.zeros((rows, a.out_dim), np.float64)
        st = np.zeros(4, np.uint64)
        ac = a._c()
        self._chk(self.lib.ork_lut_forward(C.byref(ac), _ptr(X, _f64p), rows, tier, nthreads, _ptr(Y, _f64p),
                                           _ptr(st, _u64p)))
        return Y, st

    def lut_model_forward(self, chain: list[Artifact], X: np.ndarray, tier: int = 1, nthreads: int = 1):
        X = np.ascontiguousarray(X, np.float64)
        rows = X.shape[0]
        arr = (_Art * len(chain))(*[a._c() for a in chain])
        Y = np.zeros((rows, chain[-1].out_dim), np.float64)
        st = np.zeros((len(chain), 4), np.uint64)
        self._chk(self.lib.ork_lut_model_forward(arr, len(chain), _ptr(X, _f64p), rows, tier, nthreads,
                                                 _ptr(Y, _f64p), _ptr(st, _u64p)))
        return Y, st

    def chain_session(self, chain: list[Artifact], X: np.ndarray, tier: int = 1, nthreads: int = 1):
        """A prepared chain forward for timing (reference library only; None otherwise): artifacts
        converted and the per-thread Matrix shards cut once, so that ``run()`` times only the threads'
        lut_model_forward_batch calls and the copy of their results."""
        if not hasattr(self.lib, "ork_chain_session_create"):
            return None
        return _ChainSession(self, chain, X, tier, nthreads)

    def spline_forward(self, spec: Spec, X: np.ndarray, tier: int = 1, nthreads: int = 1):
        X = np.ascontiguousarray(X, np.float64)
        Y = np.zeros((X.shape[0], spec.out_dim), np.float64)
        cs = spec._c()
        self._chk(self.lib.ork_spline_forward(C.byref(cs), _ptr(X, _f64p), X.shape[0], tier, nthreads,
                                              _ptr(Y, _f64p)))
        return Y

    def gen_layer(self, seed, d, m, segments, degree=3):
        """gen_layer (model_gen.cpp:7-27) -> Spec."""
        R, E = segments + degree, d * m
        bp, co, bs, ss, os_ = np.zeros(segments + 1), np.zeros(E * R), np.zeros(E), np.zeros(E), np.zeros(E)
        self._chk(self.lib.ork_gen_layer(seed, d, m, segments, degree, *[_ptr(a, _f64p) for a in (bp, co, bs, ss, os_)]))
        return Spec(d, m, bp, co, bs, ss, os_, degree)

    def gen_inputs(self, seed, n, dim, lo, hi, clip):
        X = np.zeros((n, dim))
        self._chk(self.lib.ork_gen_inputs(seed, n, dim, lo, hi, int(clip), _ptr(X, _f64p)))
        return X

    def artifact_save(self, a: Artifact, path) -> None:
        """save_artifact (artifact_io.cpp:206-219); reference library only."""
        ac = a._c()
        self._chk(self.lib.ork_artifact_save(C.byref(ac), os.fsencode(path)))

    def artifact_load_status(self, path, resave_path=None) -> int:
        """load_artifact (artifact_io.cpp:221-300): 0 or the error status (9..15 I/O family);
        resave_path: write the loaded artifact again."""
        return self.lib.ork_artifact_load_resave(os.fsencode(path), os.fsencode(resave_path) if resave_path else None)

    def eval_accuracy(self, spec: Spec, a: Artifact, X: np.ndarray, nthreads: int = 1) -> dict:
        """eval_accuracy + memory_breakdown (metrics.cpp:8-103)."""
        X = np.ascontiguousarray(X, np.float64)
        acc = np.zeros(6)
        cnt = np.zeros(11, np.uint64)
        has = C.c_int32(0)
        cs, ac = spec._c(), a._c()
        self._chk(self.lib.ork_eval_accuracy(C.byref(cs), C.byref(ac), _ptr(X, _f64p), X.shape[0], nthreads,
                                             _ptr(acc, _f64p), _ptr(cnt, _u64p), C.byref(has)))
        keys = ("n_inrange_evals", "n_oob_evals", "n_boundary_evals", "n_oob_samples", "q_table_bytes",
                "scale_bytes", "y_min_bytes", "knots_bytes", "edge_scalar_bytes", "total_bytes", "float_model_bytes")
        r = dict(mae_inrange=acc[0], maxabs_inrange=acc[1], mae_oob=acc[2] if has.value else None,
                 maxabs_oob=acc[3] if has.value else None, oob_any_frac=acc[4], overhead_ratio=acc[5])
        r.update({k: int(v) for k, v in zip(keys, cnt)})
        return r

    def coords(self, a: Artifact, x: np.ndarray):
        x = np.ascontiguousarray(x, np.float64).ravel()
        n = len(x)
        inr = np.zeros(n, np.uint8)
        xc = np.zeros(n)
        k, l0, l1 = (np.zeros(n, np.int32) for _ in range(3))
        w = np.zeros(n)
        ac = a._c()
        self._chk(self.lib.ork_coords(C.byref(ac), _ptr(x, _f64p), n, _ptr(inr, _u8p), _ptr(xc, _f64p),
                                      _ptr(k, _i32p), _ptr(l0, _i32p), _ptr(l1, _i32p), _ptr(w, _f64p)))
        return dict(in_range=inr.astype(bool), x_clip=xc, k=k, l0=l0, l1=l1, w=w)

    def eval_value(self, a: Artifact, e: int, x: float):
        v, o = C.c_double(), C.c_int32()
        ac = a._c()
        self._chk(self.lib.ork_eval_value(C.byref(ac), e, x, C.byref(v), C.byref(o)))
        return v.value, bool(o.value)

    def eval_phi(self, a: Artifact, e: int, x: float):
        v = C.c_double()
        ac = a._c()
        self._chk(self.lib.ork_eval_phi(C.byref(ac), e, x, C.byref(v)))
        return v.value

    # ------------------------------------------------------------------ misc
    def basis_values(self, bp, degree, x):
        bp = np.ascontiguousarray(bp, np.float64)
        out = np.zeros(len(bp) - 1 + degree)
        self._chk(self.lib.ork_basis_values(_ptr(bp, _f64p), len(bp) - 1, degree, x, _ptr(out, _f64p)))
        return out

    def quantize_segment(self, v, scheme):
        v = np.ascontiguousarray(v, np.float64)
        q = np.zeros(len(v), np.int32)
        s, y = C.c_double(), C.c_double()
        self._chk(self.lib.ork_quantize_segment(_ptr(v, _f64p), len(v), scheme, _ptr(q, _i32p), C.byref(s),
                                                C.byref(y)))
        return q, s.value, y.value

    def f16_round(self, f: float) -> float:
        return self.lib.ork_f16_bits_to_f32(self.lib.ork_f32_to_f16_bits(f))

    def f32_to_f16_bits(self, f: float) -> int:
        return self.lib.ork_f32_to_f16_bits(f)

    def rng_uniform(self, seed, n):
        out = np.zeros(n)
        self.lib.ork_rng_uniform(seed, n, _ptr(out, _f64p))
        return out

    def rng_normal(self, seed, n):
        out = np.zeros(n)
        self.lib.ork_rng_normal(seed, n, _ptr(out, _f64p))
        return out

    def recipe_layer(self, cfg: int, layer: int) -> Spec:
        dims = RECIPE_DIMS[cfg]
        G = RECIPE_G[cfg]
        d, m = dims[layer], dims[layer + 1]
        E, R = d * m, G + 3
        bp = np.zeros(G + 1)
        co = np.zeros(E * R)
        bs, ss, os_ = np.zeros(E), np.zeros(E), np.zeros(E)
        self._chk(self.lib.ork_recipe_layer(cfg, layer, *[_ptr(a, _f64p) for a in (bp, co, bs, ss, os_)]))
        return Spec(d, m, bp, co.reshape(E, R), bs, ss, os_)

    def recipe_inputs(self, cfg: int, row0: int, rows: int) -> np.ndarray:
        X = np.zeros((rows, RECIPE_DIMS[cfg][0]), np.float32)
        self._chk(self.lib.ork_recipe_inputs(cfg, row0, rows, _ptr(X, _f32p)))
        return X


RECIPE_DIMS = {1: [2, 5, 1], 2: [78, 16, 2], 3: [64, 64, 1], 4: [1024, 1024, 1024, 10], 5: [4096, 4096, 4096]}
RECIPE_G = {1: 5, 2: 5, 3: 8, 4: 8, 5: 16}
