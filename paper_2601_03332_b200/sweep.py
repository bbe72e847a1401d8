"""Sweep driver, result collection and the same-backend honest bench on the GPU engine.

SURVEY §8f rank 4: the reference's experiment driver (proj/core/src/sweep.cpp), its benchmark
protocol (bench.cpp) and report files (artifact_io.cpp:361-460), with every cell compiled,
evaluated and timed by this engine's kernels instead of the single-threaded CPU library:

  * `SweepConfig`, `parse_sweep_config`, `load_sweep_config`   sweep.hpp:17-40, sweep.cpp:121-176
  * `run_sweep` (cells, resume, error reports)                 sweep.cpp:67-118, 178-213
  * `collect_results` (accuracy / oob / memory / speed CSVs)   sweep.cpp:215-417
  * `BenchOptions`, `BenchReport`, `run_honest_bench`          bench.hpp, bench.cpp:16-149
  * `save_eval_report` / `load_eval_report`, `save_bench_report` / `load_bench_report`,
    `read_report_kind`                                         artifact_io.cpp:361-460

A cell directory holds the files the reference writes, in the same formats: config.json,
artifact.lut (byte-identical to the reference's save_artifact), manifest.json, bench_<tier>.json
and report.json (written last: its presence marks the cell complete, so reruns resume). JSON is
printed as nlohmann::json::dump(2) prints it (sorted keys, 2-space indent, shortest round-trip
floats), so config.json and manifest.json are byte-identical to the reference's and the CSVs of
`collect_results` are byte-identical to the reference's collect_results over the same reports.

Differences (all documented): evaluation runs on the GPU (eval.cu, f64; sums by atomics differ from
the reference's sequential sums by ~1e-15 relative); the honest bench times the spline and LUT
KERNELS of this engine on device-resident inputs with CUDA events (the paper's same-backend
comparison), one sample = `inner_repeats` launches, so `Tier` selects nothing (one backend) and
only the optimized tier is timed unless `tiers` says otherwise.
"""
from __future__ import annotations

import json
import math
import os
import statistics
from dataclasses import dataclass, field

import numpy as np

from . import lutkan as _lk
from .lutkan import (BoundaryMode, ConfigError, CorruptBlobError, DimensionError, Dtype, IoError,
                     MemoryBreakdown, MissingKeyError, OobConfig, OobPolicy, ParamDtype, QuantConfig, Scheme,
                     ShapeError, Tier, ValueRepr)

INPUT_SEED_SALT = 0x5EED5EED5EED5EED  # sweep.cpp:25

_NAMES = {
    "scheme": {Scheme.Symmetric: "symmetric", Scheme.Asymmetric: "asymmetric"},
    "dtype": {Dtype.Int8: "int8", Dtype.Uint8: "uint8"},
    "value_repr": {ValueRepr.Phi: "phi", ValueRepr.SplineComponent: "spline_component"},
    "boundary_mode": {BoundaryMode.HalfOpen: "half_open", BoundaryMode.Closed: "closed"},
    "oob_policy": {OobPolicy.ClipX: "clip_x", OobPolicy.ZeroSpline: "zero_spline"},
    "param_dtype": {ParamDtype.F32: "f32", ParamDtype.F16: "f16"},
    "tier": {Tier.Scalar: "scalar", Tier.Optimized: "optimized"},
}
BENCH_MODES = ("steady", "cold_start")  # types.cpp:37-39


def to_string(field_name: str, v) -> str:
    """to_string of types.cpp:5-39."""
    return _NAMES[field_name][v]


# ------------------------------------------------------------------ JSON as nlohmann dump(2)
def _num(v: float) -> str:
    """A double as nlohmann's serializer prints it: shortest round-trip digits, fixed notation for
    decimal exponents in (-4, 15], else d[.ddd]e+XX; non-finite values print as null."""
    if not math.isfinite(v):
        return "null"
    r = repr(float(v))
    if "e" not in r and "E" not in r:
        mant, _, frac = r.lstrip("-").partition(".")
        digits = (mant + frac).lstrip("0")
        n = len(mant.lstrip("0")) if mant.strip("0") else -(len(frac) - len(frac.lstrip("0")))
        if digits and n > 15:  # Python keeps 16-digit integers fixed; nlohmann switches at 1e15
            sign = "-" if r.startswith("-") else ""
            d = (mant + frac).lstrip("0").rstrip("0") or "0"
            return f"{sign}{d[0]}{'.' + d[1:] if len(d) > 1 else ''}e+{n - 1:02d}"
    return r


def dumps(obj, indent: int = 2, _level: int = 0) -> str:
    """nlohmann::json::dump(2) of a dict / list / scalar tree (std::map key order; arrays inline, as
    the nlohmann/json 3.11.3 copy the reference is built with here prints them: "shape": [12,5,32])."""
    pad, inner = " " * (indent * _level), " " * (indent * (_level + 1))
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [f"{inner}{json.dumps(str(k))}: {dumps(obj[k], indent, _level + 1)}" for k in sorted(obj)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(obj, (list, tuple)):  # inline, as the nlohmann copy the reference is built with prints them
        return "[" + ",".join(dumps(v, indent, _level + 1) for v in obj) + "]"
    if isinstance(obj, bool):
        return "true" if obj else "false"
    if obj is None:
        return "null"
    if isinstance(obj, (int, np.integer)):
        return str(int(obj))
    if isinstance(obj, (float, np.floating)):
        return _num(float(obj))
    return json.dumps(obj)


def _write_atomic(path: str, text: str) -> None:
    """write_text_atomic (sweep.cpp:27-36): temp file, then rename."""
    tmp = path + ".tmp"
    try:
        with open(tmp, "w", newline="") as f:
            f.write(text)
    except OSError as e:
        raise IoError(f"cannot write file: {tmp}") from e
    os.replace(tmp, path)


# ------------------------------------------------------------------ reports (artifact_io.cpp:361-460)
def _quant_json(q: QuantConfig) -> dict:
    return {"L": q.samples_per_segment, "scheme": to_string("scheme", q.scheme), "dtype": to_string("dtype", q.dtype),
            "value_repr": to_string("value_repr", q.value_repr), "interp": "linear",
            "param_dtype": to_string("param_dtype", q.param_dtype)}


def _oob_json(o: OobConfig) -> dict:
    return {"boundary_mode": to_string("boundary_mode", o.boundary_mode),
            "oob_policy": to_string("oob_policy", o.oob_policy)}


def _memory_json(m: MemoryBreakdown) -> dict:
    return {"q_table_bytes": m.q_table_bytes, "scale_bytes": m.scale_bytes, "y_min_bytes": m.y_min_bytes,
            "knots_bytes": m.knots_bytes, "edge_scalar_bytes": m.edge_scalar_bytes, "total_bytes": m.total_bytes,
            "float_model_bytes": m.float_model_bytes, "overhead_ratio": float(m.overhead_ratio)}


def _req(j: dict, key: str, where: str):
    if key not in j:
        raise MissingKeyError(f'{where}: missing key "{key}"')
    return j[key]


def _enum(j: dict, key: str, where: str):
    v = _req(j, key, where)
    if not isinstance(v, str):
        raise ShapeError(f'{where}: "{key}" must be a string')
    return _lk.parse_enum(key, v)


def _quant_from(j: dict, where: str) -> QuantConfig:
    L = _req(j, "L", where)
    return QuantConfig(int(L), _enum(j, "scheme", where), _enum(j, "dtype", where), _enum(j, "value_repr", where),
                       _enum(j, "interp", where), _enum(j, "param_dtype", where))


def _oob_from(j: dict, where: str) -> OobConfig:
    return OobConfig(_enum(j, "boundary_mode", where), _enum(j, "oob_policy", where))


def _memory_from(j: dict) -> MemoryBreakdown:
    return MemoryBreakdown(*(int(j.get(k, 0)) for k in ("q_table_bytes", "scale_bytes", "y_min_bytes", "knots_bytes",
                                                         "edge_scalar_bytes", "total_bytes", "float_model_bytes")),
                           float(j.get("overhead_ratio", 0.0)))


def _load_report_json(path: str, expect_kind: str) -> dict:
    """load_report_json (artifact_io.cpp:346-354)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoError(f"cannot open file: {path}") from e
    try:
        j = json.loads(raw)
    except ValueError:
        j = None
    if not isinstance(j, dict):
        raise CorruptBlobError("report is not a JSON object")
    kind = _req(j, "kind", "report")
    if not isinstance(kind, str):
        raise ShapeError('report: "kind" must be a string')
    if kind != expect_kind:
        raise ShapeError(f'report kind is "{kind}", expected "{expect_kind}"')
    return j


def eval_report_json(r: "_lk.EvalReport") -> str:
    m = {"mae_inrange": float(r.mae_inrange), "maxabs_inrange": float(r.maxabs_inrange),
         "oob_any_frac": float(r.oob_any_frac), "n_inrange_evals": int(r.n_inrange_evals),
         "n_oob_evals": int(r.n_oob_evals), "n_boundary_evals": int(r.n_boundary_evals)}
    if r.mae_oob is not None:
        m["mae_oob"] = float(r.mae_oob)
    if r.maxabs_oob is not None:
        m["maxabs_oob"] = float(r.maxabs_oob)
    return dumps({"kind": "eval", "seed": int(r.seed), "n_samples": int(r.n_samples), "quant": _quant_json(r.quant),
                  "oob": _oob_json(r.oob), "metrics": m, "memory": _memory_json(r.memory)})


def save_eval_report(r: "_lk.EvalReport", path) -> None:
    """save_eval_report (artifact_io.cpp:361-381)."""
    with open(path, "w", newline="") as f:
        f.write(eval_report_json(r))


def load_eval_report(path) -> "_lk.EvalReport":
    """load_eval_report (artifact_io.cpp:383-403)."""
    j = _load_report_json(os.fspath(path), "eval")
    m = _req(j, "metrics", "report")
    r = _lk.EvalReport(_quant_from(_req(j, "quant", "report"), "report quant"),
                       _oob_from(_req(j, "oob", "report"), "report oob"))
    r.seed, r.n_samples = int(_req(j, "seed", "report")), int(_req(j, "n_samples", "report"))
    r.mae_inrange = float(_req(m, "mae_inrange", "metrics"))
    r.maxabs_inrange = float(_req(m, "maxabs_inrange", "metrics"))
    r.mae_oob = float(m["mae_oob"]) if "mae_oob" in m else None
    r.maxabs_oob = float(m["maxabs_oob"]) if "maxabs_oob" in m else None
    r.oob_any_frac = float(_req(m, "oob_any_frac", "metrics"))
    r.n_inrange_evals, r.n_oob_evals = int(m.get("n_inrange_evals", 0)), int(m.get("n_oob_evals", 0))
    r.n_boundary_evals = int(m.get("n_boundary_evals", 0))
    if "memory" in j:
        r.memory = _memory_from(j["memory"])
    return r


@dataclass
class BenchOptions:
    """bench.hpp:14-20 (50 warm-up + 200 timed iterations per side)."""
    warmup_iters: int = 50
    timed_iters: int = 200
    tier: Tier = Tier.Optimized
    mode: str = "steady"
    threads: int = 1
    seed: int = 0


@dataclass
class BenchReport:
    """metrics.hpp:72-98."""
    quant: QuantConfig = field(default_factory=QuantConfig)
    oob: OobConfig = field(default_factory=OobConfig)
    tier: Tier = Tier.Optimized
    mode: str = "steady"
    seed: int = 0
    batch: int = 0
    warmup_iters: int = 0
    timed_iters: int = 0
    inner_repeats: int = 1
    threads: int = 1
    spline_ms_mean: float = 0.0
    spline_ms_std: float = 0.0
    spline_ms_median: float = 0.0
    lut_ms_mean: float = 0.0
    lut_ms_std: float = 0.0
    lut_ms_median: float = 0.0
    spline_ms_per_sample: float = 0.0
    lut_ms_per_sample: float = 0.0
    speedup: float = 0.0
    speedup_median: float = 0.0
    memory: MemoryBreakdown = field(default_factory=MemoryBreakdown)


def bench_report_json(r: BenchReport) -> str:
    t = {k: float(getattr(r, k)) for k in ("spline_ms_mean", "spline_ms_std", "spline_ms_median", "lut_ms_mean",
                                           "lut_ms_std", "lut_ms_median", "spline_ms_per_sample",
                                           "lut_ms_per_sample", "speedup", "speedup_median")}
    return dumps({"kind": "bench", "seed": int(r.seed), "tier": to_string("tier", r.tier), "mode": r.mode,
                  "batch": int(r.batch), "warmup_iters": int(r.warmup_iters), "timed_iters": int(r.timed_iters),
                  "inner_repeats": int(r.inner_repeats), "threads": int(r.threads), "quant": _quant_json(r.quant),
                  "oob": _oob_json(r.oob), "timing": t, "memory": _memory_json(r.memory)})


def save_bench_report(r: BenchReport, path) -> None:
    """save_bench_report (artifact_io.cpp:405-432)."""
    with open(path, "w", newline="") as f:
        f.write(bench_report_json(r))


def load_bench_report(path) -> BenchReport:
    """load_bench_report (artifact_io.cpp:434-458)."""
    j = _load_report_json(os.fspath(path), "bench")
    r = BenchReport()
    r.seed = int(_req(j, "seed", "report"))
    r.tier = _enum(j, "tier", "report")
    mode = _req(j, "mode", "report")
    if mode not in BENCH_MODES:
        raise ConfigError(f'unknown mode value: "{mode}"')
    r.mode = mode
    r.batch = int(_req(j, "batch", "report"))
    r.warmup_iters, r.timed_iters = int(j.get("warmup_iters", 0)), int(j.get("timed_iters", 0))
    r.inner_repeats, r.threads = int(j.get("inner_repeats", 1)), int(j.get("threads", 1))
    r.quant = _quant_from(_req(j, "quant", "report"), "report quant")
    r.oob = _oob_from(_req(j, "oob", "report"), "report oob")
    t = _req(j, "timing", "report")
    r.spline_ms_mean = float(_req(t, "spline_ms_mean", "timing"))
    r.lut_ms_mean = float(_req(t, "lut_ms_mean", "timing"))
    r.speedup = float(_req(t, "speedup", "timing"))
    for k in ("spline_ms_std", "spline_ms_median", "lut_ms_std", "lut_ms_median", "spline_ms_per_sample",
              "lut_ms_per_sample", "speedup_median"):
        setattr(r, k, float(t.get(k, 0.0)))
    if "memory" in j:
        r.memory = _memory_from(j["memory"])
    return r


def read_report_kind(path) -> str:
    """read_report_kind (artifact_io.cpp:460-470)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise IoError(f"cannot open file: {path}") from e
    try:
        j = json.loads(raw)
    except ValueError:
        j = None
    if not isinstance(j, dict):
        raise CorruptBlobError("report is not a JSON object")
    kind = _req(j, "kind", "report")
    if not isinstance(kind, str):
        raise ShapeError('report: "kind" must be a string')
    return kind


# ------------------------------------------------------------------ honest bench (bench.cpp) on the GPU
def _summarize(xs: list[float]) -> tuple[float, float, float]:
    """summarize (bench.cpp:46-58): mean, population std, median."""
    if not xs:
        return 0.0, 0.0, 0.0
    mean = sum(xs) / len(xs)
    return mean, math.sqrt(sum((x - mean) ** 2 for x in xs) / len(xs)), statistics.median(xs)


def run_honest_bench(layer: "_lk.KanLayerSpec", artifact_path, X, opts: BenchOptions | None = None,
                     engine: "_lk.Engine | None" = None) -> BenchReport:
    """run_honest_bench (bench.cpp:71-149) on the GPU: the spline kernel (layer_forward_batch) against
    the LUT kernel (lut_layer_forward_batch of the artifact loaded from `artifact_path`) on the same
    device-resident batch. Each sample is one CUDA-event-timed region of `inner_repeats` forwards
    (the reference's calibrate_repeats rule: the smallest power of 4 whose region reaches 2 us);
    cold_start puts the artifact load (file -> device layer) inside every LUT forward."""
    import ctypes as C

    import torch
    opts = opts or BenchOptions()
    if opts.threads != 1:
        raise ConfigError(f"benchmark requires threads == 1, got {opts.threads}")
    if opts.timed_iters < 1:
        raise ConfigError("timed_iters must be at least 1")
    if opts.warmup_iters < 0:
        raise ConfigError("warmup_iters must be non-negative")
    if opts.mode not in BENCH_MODES:
        raise ConfigError(f'unknown mode value: "{opts.mode}"')
    X = np.asarray(X)
    if X.ndim != 2 or X.shape[0] == 0:
        raise DimensionError("benchmark input batch is empty")
    if X.shape[1] != layer.in_dim:
        raise DimensionError(f"benchmark input has {X.shape[1]} columns, layer takes {layer.in_dim}")
    eng = engine or _lk.default_engine()
    art = _lk.load_artifact(artifact_path, engine=eng)
    if art.in_dim != layer.in_dim or art.out_dim != layer.out_dim:
        raise DimensionError("artifact shape does not match the layer")
    lib = _lk.lib()
    rows = X.shape[0]
    dev = torch.device("cuda", eng.device) if hasattr(eng, "device") else torch.device("cuda")
    Xd = torch.from_numpy(np.ascontiguousarray(X, np.float32)).to(dev)
    Yd = torch.empty((rows, layer.out_dim), dtype=torch.float32, device=dev)
    spec, dl = layer.device(eng), art.device(eng)
    path = os.fsencode(os.fspath(artifact_path))

    def spline_fn():
        _lk.check(lib.lkg_spline_forward(eng.handle, spec.handle, C.c_void_p(Xd.data_ptr()), rows,
                                         C.c_void_p(Yd.data_ptr())))

    def lut_steady_fn():
        _lk.check(lib.lkg_layer_forward(eng.handle, dl.handle, C.c_void_p(Xd.data_ptr()), rows,
                                        C.c_void_p(Yd.data_ptr()), None))

    def lut_cold_fn():
        h = C.c_void_p()
        _lk.check(lib.lkg_artifact_load(eng.handle, path, C.byref(h)))
        fresh = _lk.DeviceLayer(h)
        _lk.check(lib.lkg_layer_forward(eng.handle, fresh.handle, C.c_void_p(Xd.data_ptr()), rows,
                                        C.c_void_p(Yd.data_ptr()), None))
        eng.synchronize()
        del fresh

    stream = torch.cuda.ExternalStream(eng.stream) if eng.stream else torch.cuda.current_stream(dev)

    def region_ms(fn, repeats: int) -> float:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.synchronize()
        e0.record(stream)
        for _ in range(repeats):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    def calibrate(fn) -> int:  # bench.cpp:30-38
        repeats = 1
        while repeats < (1 << 20):
            if region_ms(fn, repeats) >= 2e-3:
                break
            repeats *= 4
        return repeats

    lut_fn = lut_cold_fn if opts.mode == "cold_start" else lut_steady_fn
    repeats = max(calibrate(spline_fn), calibrate(lut_fn))

    def run_side(fn) -> list[float]:  # bench.cpp:60-67
        for _ in range(opts.warmup_iters):
            fn()
        return [region_ms(fn, repeats) / repeats for _ in range(opts.timed_iters)]

    ss, ls = _summarize(run_side(spline_fn)), _summarize(run_side(lut_fn))
    eng.collect(1)
    r = BenchReport(QuantConfig(art.L, art.scheme, art.dtype, art.value_repr, art.interp, art.param_dtype), art.oob,
                    opts.tier, opts.mode, opts.seed, rows, opts.warmup_iters, opts.timed_iters, repeats, opts.threads)
    r.spline_ms_mean, r.spline_ms_std, r.spline_ms_median = ss
    r.lut_ms_mean, r.lut_ms_std, r.lut_ms_median = ls
    r.spline_ms_per_sample, r.lut_ms_per_sample = ss[0] / rows, ls[0] / rows
    r.speedup = ss[0] / ls[0] if ls[0] > 0 else 0.0
    r.speedup_median = ss[2] / ls[2] if ls[2] > 0 else 0.0
    r.memory = _lk.memory_breakdown(art, layer)
    return r


# ------------------------------------------------------------------ sweep (sweep.hpp / sweep.cpp)
@dataclass
class SweepConfig:
    """sweep.hpp:17-34 (the reference's defaults)."""
    Ls: list = field(default_factory=lambda: [16, 32, 64, 128])
    schemes: list = field(default_factory=lambda: [Scheme.Symmetric, Scheme.Asymmetric])
    boundary_modes: list = field(default_factory=lambda: [BoundaryMode.HalfOpen, BoundaryMode.Closed])
    oob_policies: list = field(default_factory=lambda: [OobPolicy.ClipX, OobPolicy.ZeroSpline])
    seeds: list = field(default_factory=lambda: [0, 1, 2, 3, 4])
    n_samples: int = 4096
    value_repr: ValueRepr = ValueRepr.SplineComponent
    param_dtype: ParamDtype = ParamDtype.F32
    in_dim: int = 10
    out_dim: int = 8
    segments: int = 8
    degree: int = 3
    with_speed: bool = True
    bench_batch: int = 1024
    bench_warmup_iters: int = 50
    bench_timed_iters: int = 200


_SWEEP_KEYS = ("Ls", "schemes", "boundary_modes", "oob_policies", "seeds", "n_samples", "value_repr", "param_dtype",
               "in_dim", "out_dim", "segments", "degree", "with_speed", "bench_batch", "bench_warmup_iters",
               "bench_timed_iters")


def parse_sweep_config(json_text: str) -> SweepConfig:
    """parse_sweep_config (sweep.cpp:121-171): keys mirror the fields, missing keys keep their
    defaults, unknown keys and empty axes are ConfigErrors. (A value of the wrong JSON type is a
    ConfigError here; the reference lets nlohmann's type_error escape.)"""
    try:
        j = json.loads(json_text)
    except ValueError:
        j = None
    if not isinstance(j, dict):
        raise ConfigError("sweep config is not a JSON object")
    for k in j:
        if k not in _SWEEP_KEYS:
            raise ConfigError(f"unknown sweep config key: {k}")
    c = SweepConfig()

    def ints(k, lo=None):
        v = j[k]
        if not isinstance(v, list) or not all(isinstance(x, int) and not isinstance(x, bool) for x in v) or \
                (lo is not None and any(x < lo for x in v)):
            raise ConfigError(f"sweep config key {k} must be a list of integers")
        return list(v)

    def integer(k, lo=None):
        v = j[k]
        if not isinstance(v, int) or isinstance(v, bool) or (lo is not None and v < lo):
            raise ConfigError(f"sweep config key {k} must be an integer")
        return v

    def enums(k, fname):
        v = j[k]
        if not isinstance(v, list) or not all(isinstance(x, str) for x in v):
            raise ConfigError(f"sweep config key {k} must be a list of strings")
        return [_lk.parse_enum(fname, x) for x in v]

    def enum1(k):
        if not isinstance(j[k], str):
            raise ConfigError(f"sweep config key {k} must be a string")
        return _lk.parse_enum(k, j[k])

    if "Ls" in j:
        c.Ls = ints("Ls")
    if "schemes" in j:
        c.schemes = enums("schemes", "scheme")
    if "boundary_modes" in j:
        c.boundary_modes = enums("boundary_modes", "boundary_mode")
    if "oob_policies" in j:
        c.oob_policies = enums("oob_policies", "oob_policy")
    if "seeds" in j:
        c.seeds = ints("seeds", 0)
    for k in ("n_samples", "bench_batch"):
        if k in j:
            setattr(c, k, integer(k, 0))
    if "value_repr" in j:
        c.value_repr = enum1("value_repr")
    if "param_dtype" in j:
        c.param_dtype = enum1("param_dtype")
    for k in ("in_dim", "out_dim", "segments", "degree", "bench_warmup_iters", "bench_timed_iters"):
        if k in j:
            setattr(c, k, integer(k))
    if "with_speed" in j:
        if not isinstance(j["with_speed"], bool):
            raise ConfigError("sweep config key with_speed must be a boolean")
        c.with_speed = j["with_speed"]
    if not (c.Ls and c.schemes and c.boundary_modes and c.oob_policies and c.seeds):
        raise ConfigError("sweep config has an empty axis")
    return c


def load_sweep_config(path) -> SweepConfig:
    """load_sweep_config (sweep.cpp:173-176)."""
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError as e:
        raise IoError(f"cannot open file: {path}") from e
    return parse_sweep_config(text)


@dataclass
class SweepSummary:
    """sweep.hpp:42-47."""
    n_total: int = 0
    n_run: int = 0
    n_skipped: int = 0
    n_failed: int = 0


def cell_dir_name(L: int, scheme, boundary, policy) -> str:
    """cell_dir_name (sweep.cpp:38-42)."""
    return (f"L{L}_{to_string('scheme', scheme)}_{to_string('boundary_mode', boundary)}_"
            f"{to_string('oob_policy', policy)}")


def cell_config_json(cfg: SweepConfig, L: int, scheme, boundary, policy, seed: int) -> str:
    """cell_config_json (sweep.cpp:44-65), printed as config.json."""
    return dumps({"L": L, "scheme": to_string("scheme", scheme), "boundary_mode": to_string("boundary_mode", boundary),
                  "oob_policy": to_string("oob_policy", policy),
                  "dtype": "int8" if scheme == Scheme.Symmetric else "uint8",
                  "value_repr": to_string("value_repr", cfg.value_repr),
                  "param_dtype": to_string("param_dtype", cfg.param_dtype), "seed": seed,
                  "input_seed": seed ^ INPUT_SEED_SALT, "n_samples": cfg.n_samples, "in_dim": cfg.in_dim,
                  "out_dim": cfg.out_dim, "segments": cfg.segments, "degree": cfg.degree,
                  "with_speed": cfg.with_speed, "bench_batch": cfg.bench_batch,
                  "bench_warmup_iters": cfg.bench_warmup_iters, "bench_timed_iters": cfg.bench_timed_iters})


def run_cell(cfg: SweepConfig, d: str, L: int, scheme, boundary, policy, seed: int, engine,
             tiers=(Tier.Optimized,)) -> None:
    """run_cell (sweep.cpp:67-118) on the GPU engine."""
    layer = _lk.gen_layer(seed, cfg.in_dim, cfg.out_dim, cfg.segments, cfg.degree)
    q = QuantConfig(L, Scheme(scheme), Dtype.Int8 if scheme == Scheme.Symmetric else Dtype.Uint8,
                    cfg.value_repr, _lk.Interp.Linear, cfg.param_dtype)
    art = _lk.compile_layer(layer, q, OobConfig(boundary, policy), engine=engine)
    apath = os.path.join(d, "artifact.lut")
    _lk.save_artifact(art, apath + ".tmp", engine=engine)
    os.replace(apath + ".tmp", apath)
    _write_atomic(os.path.join(d, "manifest.json"), _lk.artifact_manifest_json(art))
    _write_atomic(os.path.join(d, "config.json"), cell_config_json(cfg, L, scheme, boundary, policy, seed))
    input_seed = seed ^ INPUT_SEED_SALT
    lo, hi = float(layer.grid.breakpoints[0]), float(layer.grid.breakpoints[-1])
    X = _lk.gen_inputs(input_seed, cfg.n_samples, cfg.in_dim, lo, hi, True)
    report = _lk.eval_accuracy(layer, art, X, engine=engine)  # f64 inputs, evaluated unrounded
    report.seed = seed
    if cfg.with_speed:
        Xb = _lk.gen_inputs(input_seed, cfg.bench_batch, cfg.in_dim, lo, hi, True)
        for tier in tiers:
            b = run_honest_bench(layer, apath, Xb, BenchOptions(cfg.bench_warmup_iters, cfg.bench_timed_iters, tier,
                                                                 "steady", 1, seed), engine=engine)
            bpath = os.path.join(d, f"bench_{to_string('tier', tier)}.json")
            save_bench_report(b, bpath + ".tmp")
            os.replace(bpath + ".tmp", bpath)
    rpath = os.path.join(d, "report.json")  # written last: the cell's completion marker
    save_eval_report(report, rpath + ".tmp")
    os.replace(rpath + ".tmp", rpath)


def run_sweep(cfg: SweepConfig, root, log=None, engine=None, tiers=(Tier.Optimized,)) -> SweepSummary:
    """run_sweep (sweep.cpp:178-213): every (L, scheme, boundary, policy, seed) cell under
    root/<cell>/seed<N>/; cells with a report.json are skipped (resume); a failing cell writes an
    {"kind": "error", ...} report and the sweep moves on."""
    root = os.fspath(root)
    os.makedirs(root, exist_ok=True)
    eng = engine or _lk.default_engine()
    s = SweepSummary()
    for L in cfg.Ls:
        for scheme in cfg.schemes:
            for boundary in cfg.boundary_modes:
                for policy in cfg.oob_policies:
                    for seed in cfg.seeds:
                        s.n_total += 1
                        d = os.path.join(root, cell_dir_name(L, scheme, boundary, policy), f"seed{seed}")
                        if os.path.exists(os.path.join(d, "report.json")):
                            s.n_skipped += 1
                            continue
                        os.makedirs(d, exist_ok=True)
                        try:
                            run_cell(cfg, d, L, scheme, boundary, policy, seed, eng, tiers)
                            s.n_run += 1
                            if log:
                                log.write(f"ok   {d}\n")
                        except _lk.CudaError:
                            raise  # a device fault is not a cell result
                        except Exception as e:  # noqa: BLE001 — the reference catches std::exception
                            _write_atomic(os.path.join(d, "report.json"), dumps({
                                "kind": "error", "message": str(e), "seed": seed,
                                "cell": {"L": L, "scheme": to_string("scheme", scheme),
                                         "boundary_mode": to_string("boundary_mode", boundary),
                                         "oob_policy": to_string("oob_policy", policy)}}))
                            s.n_failed += 1
                            if log:
                                log.write(f"FAIL {d}: {e}\n")
    return s


def _fmt(v: float) -> str:
    return "%.12g" % v  # sweep.cpp:244-248


def _agg(xs: list[float]) -> str:
    """append_agg (sweep.cpp:277-283) of aggregate (sweep.cpp:255-275): mean,std,min,max."""
    if not xs:
        return ",,,,"
    mean = 0.0
    for x in xs:
        mean += x
    mean /= len(xs)
    ss = 0.0
    for x in xs:
        ss += (x - mean) * (x - mean)
    return "," + ",".join(_fmt(v) for v in (mean, math.sqrt(ss / len(xs)), min(xs), max(xs)))


def _mean(xs: list[float]) -> float:
    m = 0.0
    for x in xs:
        m += x
    return m / len(xs) if xs else 0.0


def collect_results(root, out_dir) -> None:
    """collect_results (sweep.cpp:285-417): per-cell aggregates (seeds collapse to mean / population
    std / min / max) of every eval report and bench report under root, sorted by (L, scheme,
    boundary_mode, oob_policy) — accuracy.csv, oob_matrix.csv, memory.csv, speed_scalar.csv,
    speed_optimized.csv, formatted deterministically (%.12g)."""
    root, out_dir = os.fspath(root), os.fspath(out_dir)
    cells: dict = {}
    if os.path.isdir(root):
        for cell in os.listdir(root):
            cdir = os.path.join(root, cell)
            if not os.path.isdir(cdir):
                continue
            for seed in os.listdir(cdir):
                d = os.path.join(cdir, seed)
                cp, rp = os.path.join(d, "config.json"), os.path.join(d, "report.json")
                if not os.path.isdir(d) or not os.path.exists(cp) or not os.path.exists(rp):
                    continue
                try:
                    with open(cp, "rb") as f:
                        cj = json.loads(f.read())
                    key = (int(cj["L"]), str(cj["scheme"]), str(cj["boundary_mode"]), str(cj["oob_policy"]))
                except Exception:  # noqa: BLE001 — unreadable config: skipped, as the reference does
                    continue
                try:
                    if read_report_kind(rp) != "eval":
                        continue
                    r = load_eval_report(rp)
                    a = cells.setdefault(key, {"mae_in": [], "max_in": [], "oob_any": [], "mae_oob": [],
                                               "max_oob": [], "memory": None,
                                               Tier.Scalar: ([], [], [], []), Tier.Optimized: ([], [], [], [])})
                    a["mae_in"].append(r.mae_inrange)
                    a["max_in"].append(r.maxabs_inrange)
                    a["oob_any"].append(r.oob_any_frac)
                    if r.mae_oob is not None:
                        a["mae_oob"].append(r.mae_oob)
                    if r.maxabs_oob is not None:
                        a["max_oob"].append(r.maxabs_oob)
                    if a["memory"] is None:
                        a["memory"] = r.memory
                    for tier in (Tier.Scalar, Tier.Optimized):
                        bp = os.path.join(d, f"bench_{to_string('tier', tier)}.json")
                        if not os.path.exists(bp):
                            continue
                        b = load_bench_report(bp)
                        for lst, v in zip(a[tier], (b.speedup, b.speedup_median, b.spline_ms_per_sample,
                                                    b.lut_ms_per_sample)):
                            lst.append(v)
                except Exception:  # noqa: BLE001
                    continue
    os.makedirs(out_dir, exist_ok=True)
    keys = sorted(cells)

    def prefix(k):
        return f"{k[0]},{k[1]},{k[2]},{k[3]}"

    rows = ["L,scheme,boundary_mode,oob_policy,n_seeds,mae_inrange_mean,mae_inrange_std,mae_inrange_min,"
            "mae_inrange_max,maxabs_inrange_mean,maxabs_inrange_std,maxabs_inrange_min,maxabs_inrange_max"]
    for k in keys:
        a = cells[k]
        rows.append(f"{prefix(k)},{len(a['mae_in'])}" + _agg(a["mae_in"]) + _agg(a["max_in"]))
    _write_atomic(os.path.join(out_dir, "accuracy.csv"), "\n".join(rows) + "\n")

    rows = ["L,scheme,boundary_mode,oob_policy,n_seeds,oob_any_frac_mean,mae_oob_mean,mae_oob_std,mae_oob_min,"
            "mae_oob_max,maxabs_oob_mean,maxabs_oob_std,maxabs_oob_min,maxabs_oob_max"]
    for k in keys:
        a = cells[k]
        rows.append(f"{prefix(k)},{len(a['oob_any'])},{_fmt(_mean(a['oob_any']))}" + _agg(a["mae_oob"]) +
                    _agg(a["max_oob"]))
    _write_atomic(os.path.join(out_dir, "oob_matrix.csv"), "\n".join(rows) + "\n")

    rows = ["L,scheme,boundary_mode,oob_policy,q_table_bytes,scale_bytes,y_min_bytes,knots_bytes,"
            "edge_scalar_bytes,total_bytes,float_model_bytes,q_table_frac,overhead_ratio"]
    for k in keys:
        m = cells[k]["memory"]
        if m is None:
            rows.append(prefix(k) + ",,,,,,,,,")
        else:
            rows.append(f"{prefix(k)},{m.q_table_bytes},{m.scale_bytes},{m.y_min_bytes},{m.knots_bytes},"
                        f"{m.edge_scalar_bytes},{m.total_bytes},{m.float_model_bytes},{_fmt(m.q_table_frac())},"
                        f"{_fmt(m.overhead_ratio)}")
    _write_atomic(os.path.join(out_dir, "memory.csv"), "\n".join(rows) + "\n")

    for tier in (Tier.Scalar, Tier.Optimized):
        rows = ["L,scheme,boundary_mode,oob_policy,n_seeds,speedup_mean,speedup_std,speedup_min,speedup_max,"
                "speedup_median_mean,spline_ms_per_sample_mean,lut_ms_per_sample_mean"]
        for k in keys:
            sp, med, sps, lps = cells[k][tier]
            row = f"{prefix(k)},{len(sp)}" + _agg(sp)
            row += ",,," if not sp else f",{_fmt(_mean(med))},{_fmt(_mean(sps))},{_fmt(_mean(lps))}"
            rows.append(row)
        _write_atomic(os.path.join(out_dir, f"speed_{to_string('tier', tier)}.csv"), "\n".join(rows) + "\n")


def main(argv=None) -> int:
    """`python -m paper_2601_03332_b200.sweep <config.json> <root> [csv_dir]` — the `lutkan sweep` +
    `lutkan collect` pair (lutkan_main.cpp:210-235) on the GPU engine."""
    import sys
    argv = sys.argv[1:] if argv is None else argv
    if len(argv) not in (2, 3):
        print("usage: python -m paper_2601_03332_b200.sweep <config.json> <root> [csv_dir]", file=sys.stderr)
        return 2
    s = run_sweep(load_sweep_config(argv[0]), argv[1], log=sys.stderr)
    if len(argv) == 3:
        collect_results(argv[1], argv[2])
    print(json.dumps(s.__dict__))
    return 0 if s.n_failed == 0 else 1


if __name__ == "__main__":
    raise SystemExit(main())
