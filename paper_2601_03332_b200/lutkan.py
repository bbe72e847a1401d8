"""Host-side mirror of the reference ``lutkan`` core API over the CUDA C-ABI.

Same names, argument meaning and error behaviour as the reference hot path
(/root/reference/proj/core/include/lutkan):

* types: ``KnotGrid``, ``KanLayerSpec``, ``EdgeParams``-free packed arrays (spline.hpp:15-74),
  ``QuantConfig`` (compiler.hpp:15-24), ``OobConfig`` / ``LutLayerArtifact`` / ``OobStats``
  (runtime.hpp:19-120), the enums of types.hpp:41-49 and the exception taxonomy
  ``ConfigError`` / ``DimensionError`` / ``NonFiniteError`` / ``UnsupportedBaseError``
  (types.hpp:11-39);
* compile: ``compile_layer``, ``compile_model``, ``compile_layer_debug_float`` (compiler.hpp:67-77);
* forward: ``lut_layer_forward_batch``, ``lut_layer_forward``, ``lut_model_forward_batch``,
  ``lut_model_forward`` (runtime.hpp:126-148);
* honest baseline: ``layer_forward_batch`` (spline.hpp:100-101).

All arithmetic runs in liblutkan_b200.so on the GPU. Batches may be numpy arrays
(host; copied in and out inside the call) or torch CUDA tensors (device; no copies).
Differences from the reference, by design: activations are fp32 on the device and
results come back as fp32; ``tier`` is accepted and ignored (one backend).
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import lib


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """lutkan::Error (types.hpp:11-14)."""


class ConfigError(Error):
    pass


class DimensionError(Error):
    pass


class NonFiniteError(Error):
    pass


class UnsupportedBaseError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


class IoError(Error):
    """artifact_io.hpp:11-52: the container error family."""


class CorruptArchiveError(IoError):
    pass


class CorruptBlobError(IoError):
    pass


class MissingKeyError(IoError):
    pass


class ShapeError(IoError):
    pass


class VersionError(IoError):
    pass


class EnumError(IoError):
    pass


_ERRORS = {_capi.ERR_IO: IoError, _capi.ERR_CORRUPT_ARCHIVE: CorruptArchiveError,
           _capi.ERR_CORRUPT_BLOB: CorruptBlobError, _capi.ERR_MISSING_KEY: MissingKeyError,
           _capi.ERR_SHAPE: ShapeError, _capi.ERR_VERSION: VersionError, _capi.ERR_ENUM: EnumError,
           _capi.ERR_CONFIG: ConfigError, _capi.ERR_DIMENSION: DimensionError,
           _capi.ERR_NON_FINITE: NonFiniteError, _capi.ERR_UNSUPPORTED_BASE: UnsupportedBaseError,
           _capi.ERR_CUDA: CudaError, _capi.ERR_NCCL: NcclError, _capi.ERR_OOM: CudaError,
           _capi.ERR_INVALID_ARG: ValueError}


def check(status: int) -> None:
    if status != _capi.OK:
        msg = lib().lkg_last_error().decode()
        raise _ERRORS.get(status, Error)(msg)


# ------------------------------------------------------------------- enums
class Scheme(enum.IntEnum):
    Symmetric = 0
    Asymmetric = 1


class Dtype(enum.IntEnum):
    Int8 = 0
    Uint8 = 1


class ValueRepr(enum.IntEnum):
    Phi = 0
    SplineComponent = 1


class Interp(enum.IntEnum):
    Linear = 0


class BoundaryMode(enum.IntEnum):
    HalfOpen = 0
    Closed = 1


class OobPolicy(enum.IntEnum):
    ClipX = 0
    ZeroSpline = 1


class ParamDtype(enum.IntEnum):
    F32 = 0
    F16 = 1


class Tier(enum.IntEnum):
    Scalar = 0
    Optimized = 1


_PARSE = {
    "scheme": {"symmetric": Scheme.Symmetric, "asymmetric": Scheme.Asymmetric},
    "dtype": {"int8": Dtype.Int8, "uint8": Dtype.Uint8},
    "value_repr": {"phi": ValueRepr.Phi, "spline_component": ValueRepr.SplineComponent},
    "interp": {"linear": Interp.Linear},
    "boundary_mode": {"half_open": BoundaryMode.HalfOpen, "closed": BoundaryMode.Closed},
    "oob_policy": {"clip_x": OobPolicy.ClipX, "zero_spline": OobPolicy.ZeroSpline},
    "param_dtype": {"f32": ParamDtype.F32, "f16": ParamDtype.F16},
    "tier": {"scalar": Tier.Scalar, "optimized": Tier.Optimized},
}


def parse_enum(field_name: str, s: str):
    """parse_* of types.cpp: ConfigError naming the field on unknown strings."""
    try:
        return _PARSE[field_name][s]
    except KeyError:
        raise ConfigError(f'unknown {field_name} value: "{s}"') from None


# ------------------------------------------------------------------ configs
@dataclass
class QuantConfig:
    """compiler.hpp:15-24 (defaults: L=64, symmetric int8, spline_component, f32 params)."""
    samples_per_segment: int = 64
    scheme: Scheme = Scheme.Symmetric
    dtype: Dtype = Dtype.Int8
    value_repr: ValueRepr = ValueRepr.SplineComponent
    interp: Interp = Interp.Linear
    param_dtype: ParamDtype = ParamDtype.F32

    def validate(self) -> None:
        if self.samples_per_segment < 2:
            raise ConfigError("samples_per_segment must be >= 2")
        if self.scheme == Scheme.Symmetric and self.dtype != Dtype.Int8:
            raise ConfigError("symmetric scheme requires int8")
        if self.scheme == Scheme.Asymmetric and self.dtype != Dtype.Uint8:
            raise ConfigError("asymmetric scheme requires uint8")

    def _c(self):
        return _capi.QuantCfg(self.samples_per_segment, int(self.scheme), int(self.dtype), int(self.value_repr),
                              int(self.interp), int(self.param_dtype))


@dataclass
class OobConfig:
    """runtime.hpp:19-22 (default closed + clip_x)."""
    boundary_mode: BoundaryMode = BoundaryMode.Closed
    oob_policy: OobPolicy = OobPolicy.ClipX


@dataclass
class OobStats:
    """runtime.hpp:105-120."""
    n_samples: int = 0
    n_oob_samples: int = 0
    n_inputs: int = 0
    n_oob_inputs: int = 0

    def oob_any_frac(self) -> float:
        return 0.0 if self.n_samples == 0 else self.n_oob_samples / self.n_samples

    def merge(self, o: "OobStats") -> None:
        self.n_samples += o.n_samples
        self.n_oob_samples += o.n_oob_samples
        self.n_inputs += o.n_inputs
        self.n_oob_inputs += o.n_oob_inputs

    @staticmethod
    def _from(c: _capi.OobStatsC) -> "OobStats":
        return OobStats(c.n_samples, c.n_oob_samples, c.n_inputs, c.n_oob_inputs)


# ------------------------------------------------------------------ engine
class Engine:
    """A CUDA context + stream of the library (lkg_ctx). ``stream`` is a cudaStream_t
    handle (e.g. ``torch.cuda.current_stream().cuda_stream``) or None for a private one."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        # None -> private stream; 0 (the legacy default stream) -> cudaStreamLegacy (0x1)
        s = None if stream is None else C.c_void_p(stream if stream != 0 else 1)
        check(lib().lkg_ctx_create(device, s, C.byref(h)))
        self.handle, self.device = h, device

    def close(self):
        if self.handle:
            lib().lkg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        check(lib().lkg_ctx_synchronize(self.handle))

    @property
    def stream(self) -> int:
        return lib().lkg_ctx_stream(self.handle) or 0

    @property
    def launch_count(self) -> int:
        return lib().lkg_ctx_launch_count(self.handle)

    @property
    def workspace_bytes(self) -> int:
        """Device workspace held between calls (hidden activations, transposed inputs / coordinate
        records, gather and staging buffers)."""
        return lib().lkg_ctx_workspace_bytes(self.handle)

    def trim(self) -> None:
        """Synchronize and free the workspace (it regrows on demand)."""
        check(lib().lkg_ctx_trim(self.handle))

    def collect(self, n_layers: int) -> list[OobStats]:
        arr = (_capi.OobStatsC * n_layers)()
        check(lib().lkg_ctx_collect(self.handle, arr, n_layers))
        return [OobStats._from(s) for s in arr]

    def set_spline_kernel(self, kind: str) -> None:
        """'auto' (tensor-core GEMM form where eligible) or 'simt' (the SIMT spline kernels)."""
        check(lib().lkg_ctx_set_spline_kernel(self.handle, {"auto": 0, "simt": 1}[kind]))

    def init_nccl(self, uid: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(lib().lkg_ctx_init_nccl(self.handle, buf, nranks, rank))


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().lkg_nccl_unique_id(buf))
    return bytes(buf)


_default: dict[int, Engine] = {}


def default_engine(device: int = 0) -> Engine:
    if device not in _default:
        _default[device] = Engine(device)
    return _default[device]


# ------------------------------------------------------------------- specs
@dataclass
class KnotGrid:
    """spline.hpp:15-31 (validation happens in the C-ABI, spline.cpp:8-27)."""
    breakpoints: np.ndarray
    degree: int = 3

    @property
    def K(self) -> int:
        return len(self.breakpoints) - 1

    def segment_count(self) -> int:
        return self.K

    def basis_count(self) -> int:
        return self.K + self.degree


@dataclass
class KanLayerSpec:
    """spline.hpp:35-74 with packed arrays: coeffs [E, R], gains [E]; edges e = i*out_dim + j."""
    in_dim: int
    out_dim: int
    grid: KnotGrid
    coeffs: np.ndarray
    base_scale: np.ndarray
    spline_scale: np.ndarray
    out_scale: np.ndarray
    base_kind: str = "silu"
    # column-shard placement: this spec holds columns [col0, col0 + out_dim) of a layer whose
    # full width is full_out_dim (0 = not a shard)
    col0: int = 0
    full_out_dim: int = 0
    _dev: dict = field(default_factory=dict, repr=False)

    def edge_count(self) -> int:
        return self.in_dim * self.out_dim

    def _desc(self):
        keep = [np.ascontiguousarray(a, np.float64) for a in
                (self.grid.breakpoints, self.coeffs, self.base_scale, self.spline_scale, self.out_scale)]
        p = [a.ctypes.data_as(_capi.f64p) for a in keep]
        d = _capi.SpecDesc(self.in_dim, self.out_dim, self.grid.K, self.grid.degree, self.base_kind.encode(), *p)
        return d, keep

    def device(self, engine: Engine, col0: int = 0, col1: int = 0) -> "DeviceSpec":
        key = (engine.device, col0, col1)
        if key not in self._dev:
            d, keep = self._desc()
            h = C.c_void_p()
            if col1 > col0:
                check(lib().lkg_spec_upload_columns(engine.handle, C.byref(d), col0, col1, C.byref(h)))
            elif self.full_out_dim:
                check(lib().lkg_spec_upload_shard(engine.handle, C.byref(d), self.col0, self.full_out_dim, C.byref(h)))
            else:
                check(lib().lkg_spec_upload(engine.handle, C.byref(d), C.byref(h)))
            self._dev[key] = DeviceSpec(h, self.in_dim, (col1 - col0) if col1 > col0 else self.out_dim)
        return self._dev[key]


class DeviceSpec:
    def __init__(self, h, in_dim, out_dim):
        self.handle, self.in_dim, self.out_dim = h, in_dim, out_dim

    def __del__(self):
        try:
            if self.handle:
                lib().lkg_spec_free(self.handle)
        except Exception:
            pass


class DeviceLayer:
    """Device-resident artifact (lkg_layer)."""

    def __init__(self, h):
        self.handle = h
        info = _capi.LayerInfo()
        check(lib().lkg_layer_info_get(h, C.byref(info)))
        self.info = info

    def __del__(self):
        try:
            if self.handle:
                lib().lkg_layer_free(self.handle)
        except Exception:
            pass


# ---------------------------------------------------------------- artifacts
class LutLayerArtifact:
    """runtime.hpp:31-63. Host arrays are materialised lazily from the device copy
    for compiled artifacts (a C5 layer never needs its 34 GB downloaded)."""

    _HOST = ("knots", "q_table", "scale", "y_min", "edge_base_scale", "edge_spline_scale", "edge_out_scale",
             "float_table")

    def __init__(self, in_dim=0, out_dim=0, L=0, value_repr=ValueRepr.SplineComponent, scheme=Scheme.Symmetric,
                 dtype=Dtype.Int8, param_dtype=ParamDtype.F32, oob: OobConfig | None = None, base_kind="silu",
                 interp=Interp.Linear, **arrays):
        self.in_dim, self.out_dim, self.L = in_dim, out_dim, L
        self.value_repr, self.scheme, self.dtype = ValueRepr(value_repr), Scheme(scheme), Dtype(dtype)
        self.param_dtype, self.interp = ParamDtype(param_dtype), Interp(interp)
        self.oob = oob or OobConfig()
        self.base_kind = base_kind
        self._host = {k: arrays.get(k) for k in self._HOST}
        self._dev: dict = {}
        self._origin: DeviceLayer | None = None
        self._origin_engine: Engine | None = None

    # host arrays (lazy download for compiled artifacts)
    def __getattr__(self, name):
        if name in LutLayerArtifact._HOST:
            h = self.__dict__["_host"]
            if h.get(name) is None and self.__dict__.get("_origin") is not None:
                self._download()
            return h.get(name)
        raise AttributeError(name)

    def __setattr__(self, name, value):
        if name in LutLayerArtifact._HOST:
            self._host[name] = value
            self._dev.clear()
        else:
            object.__setattr__(self, name, value)

    def edge_count(self) -> int:
        return self.in_dim * self.out_dim

    def segment_count(self) -> int:
        return len(self.knots) - 1

    @property
    def K(self) -> int:
        return self.segment_count()

    def _download(self):
        o, eng = self._origin, self._origin_engine
        E, K, L = self.in_dim * self.out_dim, o.info.K, self.L
        knots = np.zeros(K + 1, np.float32)
        q = np.zeros(E * K * L, np.uint8)
        sc, ym = np.zeros(E * K, np.float32), np.zeros(E * K, np.float32)
        sr = self.value_repr == ValueRepr.SplineComponent
        g = [np.zeros(E, np.float32) for _ in range(3)] if sr else [None] * 3
        ft = np.zeros(E * K * L, np.float64) if o.info.has_float_table else None
        ptr = lambda a, t: None if a is None else a.ctypes.data_as(t)
        check(lib().lkg_layer_download(eng.handle, o.handle, ptr(knots, _capi.f32p), ptr(q, _capi.u8p),
                                       ptr(sc, _capi.f32p), ptr(ym, _capi.f32p), *[ptr(x, _capi.f32p) for x in g],
                                       ptr(ft, _capi.f64p)))
        self._host.update(knots=knots, q_table=q, scale=sc, y_min=ym, edge_base_scale=g[0], edge_spline_scale=g[1],
                          edge_out_scale=g[2], float_table=ft)

    def _desc(self):
        conv = lambda a, t: None if a is None else np.ascontiguousarray(a, t)
        h = self._host
        keep = [conv(h["knots"], np.float32), conv(h["q_table"], np.uint8), conv(h["scale"], np.float32),
                conv(h["y_min"], np.float32), conv(h["edge_base_scale"], np.float32),
                conv(h["edge_spline_scale"], np.float32), conv(h["edge_out_scale"], np.float32),
                conv(h["float_table"], np.float64)]
        for name, a in zip(("knots", "q_table", "scale", "y_min"), keep[:4]):
            if a is None:
                raise DimensionError(f"artifact has no {name}")
        # array sizes against the declared shape (LutLayerArtifact::finalize, runtime.cpp:24-39)
        if len(keep[0]) < 2:
            raise ConfigError("artifact needs at least 2 knots")
        E, K = self.in_dim * self.out_dim, len(keep[0]) - 1
        if self.in_dim < 1 or self.out_dim < 1:
            raise ConfigError("artifact dims must be >= 1")
        if self.L < 2:
            raise ConfigError("samples per segment must be >= 2")
        if keep[1].size != E * K * self.L:
            raise DimensionError("q_table size does not match [E, K, L]")
        if keep[2].size != E * K:
            raise DimensionError("scale size does not match [E, K]")
        if keep[3].size != E * K:
            raise DimensionError("y_min size does not match [E, K]")
        for g in keep[4:7]:
            if g is not None and g.size != E:
                raise DimensionError("edge scale arrays must have one entry per edge")
        if keep[7] is not None and keep[7].size != keep[1].size:
            raise DimensionError("float_table size does not match q_table")
        types = [_capi.f32p, _capi.u8p, _capi.f32p, _capi.f32p, _capi.f32p, _capi.f32p, _capi.f32p, _capi.f64p]
        ptrs = [None if a is None else a.ctypes.data_as(t) for a, t in zip(keep, types)]
        n_k = len(keep[0]) - 1
        d = _capi.LayerDesc(self.in_dim, self.out_dim, n_k, self.L, int(self.value_repr), int(self.interp),
                            int(self.scheme), int(self.dtype), int(self.param_dtype), int(self.oob.boundary_mode),
                            int(self.oob.oob_policy), (self.base_kind or "").encode(), *ptrs)
        return d, keep

    def finalize(self) -> None:
        """Validate like LutLayerArtifact::finalize by uploading (runtime.cpp:11-43)."""
        self.device(default_engine())

    def device(self, engine: Engine, col0: int = 0, col1: int = 0) -> DeviceLayer:
        key = (engine.device, col0, col1)
        if key in self._dev:
            return self._dev[key]
        if self._origin is not None and self._origin_engine is not None and \
                self._origin_engine.device == engine.device and col1 <= col0:
            self._dev[key] = self._origin
            return self._origin
        d, keep = self._desc()
        h = C.c_void_p()
        if col1 > col0:
            check(lib().lkg_layer_upload_columns(engine.handle, C.byref(d), col0, col1, C.byref(h)))
        else:
            check(lib().lkg_layer_upload(engine.handle, C.byref(d), C.byref(h)))
        self._dev[key] = DeviceLayer(h)
        return self._dev[key]


# ------------------------------------------------------------------ compile
def compile_layer(layer: KanLayerSpec, config: QuantConfig | None = None, oob: OobConfig | None = None,
                  engine: Engine | None = None, _keep_float: bool = False, col0: int = 0,
                  col1: int = 0) -> LutLayerArtifact:
    """compiler.cpp:213-216 on the GPU (bytes bit-exact with the reference)."""
    config = config or QuantConfig()
    oob = oob or OobConfig()
    config.validate()
    eng = engine or default_engine()
    spec = layer.device(eng, col0, col1)
    h = C.c_void_p()
    qc = config._c()
    oc = _capi.OobCfg(int(oob.boundary_mode), int(oob.oob_policy))
    check(lib().lkg_compile_layer(eng.handle, spec.handle, C.byref(qc), C.byref(oc), int(_keep_float), C.byref(h)))
    dl = DeviceLayer(h)
    a = LutLayerArtifact(layer.in_dim, dl.info.out_dim, config.samples_per_segment, config.value_repr,
                         config.scheme, config.dtype, config.param_dtype, OobConfig(oob.boundary_mode, oob.oob_policy),
                         layer.base_kind if config.value_repr == ValueRepr.SplineComponent else "", config.interp)
    a._origin, a._origin_engine = dl, eng
    return a


def compile_layer_debug_float(layer, config=None, oob=None, engine=None) -> LutLayerArtifact:
    """compiler.cpp:230-233: also keeps the unquantized f64 table."""
    return compile_layer(layer, config, oob, engine, _keep_float=True)


def compile_model(layers: list[KanLayerSpec], config=None, oob=None, engine=None) -> list[LutLayerArtifact]:
    """compiler.cpp:218-228."""
    if not layers:
        raise ConfigError("model has no layers")
    for l in range(1, len(layers)):
        if layers[l].in_dim != layers[l - 1].out_dim:
            raise DimensionError(f"layer shapes do not chain at position {l}")
    return [compile_layer(s, config, oob, engine) for s in layers]


# ------------------------------------------------------------------ forward
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class ChainBatchResult:
    """runtime.hpp:143-146."""
    Y: object
    per_layer: list


def _torch_enter(eng: Engine, t):
    """Order the engine's stream after torch's current stream on t's device (an X produced by an
    asynchronous torch kernel, or the copy .contiguous().float() just made, is complete before the
    library reads it); returns the engine stream as a torch stream."""
    import torch
    dev = t.device
    ext = torch.cuda.ExternalStream(eng.stream, device=dev) if eng.stream else torch.cuda.default_stream(dev)
    ext.wait_stream(torch.cuda.current_stream(dev))
    return ext


def _torch_exit(ext, *tensors):
    """Order torch's current stream after the engine's work. The tensors the engine read or wrote
    were allocated on that stream, so the caching allocator reuses their memory only after this
    wait (record_stream on the engine's stream is deliberately NOT used: that stream may be
    destroyed with its Engine before the allocator records the tensor's release on it)."""
    import torch
    dev = tensors[0].device
    torch.cuda.current_stream(dev).wait_stream(ext)


def _forward(chain, X, engine: Engine | None):
    eng = engine or default_engine()
    if not chain:
        raise ConfigError("artifact chain is empty")
    layers = [a.device(eng) for a in chain]
    for l in range(1, len(chain)):
        if chain[l].in_dim != chain[l - 1].out_dim:
            raise DimensionError(f"artifact chain dimension mismatch between layers {l - 1} and {l}")
    handles = (C.c_void_p * len(layers))(*[d.handle for d in layers])
    stats = (_capi.OobStatsC * len(layers))()
    m_out = layers[-1].info.out_dim
    if _is_torch(X):
        import torch
        if X.dim() != 2 or X.shape[1] != chain[0].in_dim:
            raise DimensionError("batch column count does not match artifact in_dim")
        X = X.contiguous().float()
        Y = torch.empty((X.shape[0], m_out), device=X.device, dtype=torch.float32)
        ext = _torch_enter(eng, X)
        check(lib().lkg_model_forward(eng.handle, handles, len(layers), C.c_void_p(X.data_ptr()), X.shape[0],
                                      C.c_void_p(Y.data_ptr()), stats))
        _torch_exit(ext, X, Y)
    else:
        X = np.asarray(X)
        if X.ndim != 2 or X.shape[1] != chain[0].in_dim:
            raise DimensionError("batch column count does not match artifact in_dim")
        X = np.ascontiguousarray(X, np.float32)
        Y = np.zeros((X.shape[0], m_out), np.float32)
        check(lib().lkg_model_forward_host(eng.handle, handles, len(layers), X.ctypes.data_as(C.c_void_p),
                                           X.shape[0], Y.ctypes.data_as(C.c_void_p), stats))
    return Y, [OobStats._from(s) for s in stats]


def lut_layer_forward_batch(a: LutLayerArtifact, X, tier: Tier = Tier.Optimized, engine: Engine | None = None):
    """runtime.cpp:250-285 -> (Y, OobStats)."""
    Y, st = _forward([a], X, engine)
    return Y, st[0]


def lut_layer_forward(a: LutLayerArtifact, x, tier: Tier = Tier.Optimized, engine: Engine | None = None):
    """runtime.cpp:287-296 (single row)."""
    x = np.asarray(x, np.float32).reshape(-1)
    if x.shape[0] != a.in_dim:
        raise DimensionError("input size does not match artifact in_dim")
    Y, st = lut_layer_forward_batch(a, x[None, :], tier, engine)
    return Y[0], st


def lut_model_forward_batch(chain: list[LutLayerArtifact], X, tier: Tier = Tier.Optimized,
                            engine: Engine | None = None) -> ChainBatchResult:
    """runtime.cpp:298-314."""
    Y, st = _forward(chain, X, engine)
    return ChainBatchResult(Y, st)


class ChainGraph:
    """A chain forward on fixed device tensors, captured once as a CUDA graph (lkg_graph_create) and
    replayed with one cudaGraphLaunch per call — for small batches served repeatedly, where launch
    overhead dominates. ``X`` and ``Y`` are CUDA tensors bound at capture (write new inputs into
    ``X`` in place); OOB statistics accumulate in the engine (``engine.collect``)."""

    def __init__(self, chain: list["LutLayerArtifact"], X, Y, engine: Engine | None = None):
        if not (_is_torch(X) and X.is_cuda and _is_torch(Y) and Y.is_cuda):
            raise DimensionError("ChainGraph binds CUDA tensors")
        self.engine = eng = engine or default_engine(X.device.index or 0)
        self._dev = [a.device(eng) for a in chain]
        self.X, self.Y = X, Y
        hs = (C.c_void_p * len(chain))(*[d.handle for d in self._dev])
        h = C.c_void_p()
        check(lib().lkg_graph_create(eng.handle, hs, len(chain), C.c_void_p(X.data_ptr()), X.shape[0],
                                     C.c_void_p(Y.data_ptr()), C.byref(h)))
        self.handle = h

    def __call__(self):
        ext = _torch_enter(self.engine, self.X)  # X may have been rewritten in place by torch
        check(lib().lkg_graph_launch(self.handle))
        _torch_exit(ext, self.Y)
        return self.Y

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().lkg_graph_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def lut_model_forward(chain, x, tier: Tier = Tier.Optimized, engine: Engine | None = None):
    """runtime.cpp:316-325 (single row): (y, per_layer)."""
    x = np.asarray(x, np.float32).reshape(1, -1)
    r = lut_model_forward_batch(chain, x, tier, engine)
    return r.Y[0], r.per_layer


def layer_forward_batch(layer: KanLayerSpec, X, tier: Tier = Tier.Optimized, engine: Engine | None = None):
    """spline.cpp:183-187 — the same-backend B-spline forward (honest baseline)."""
    eng = engine or default_engine()
    if layer.base_kind != "silu":
        raise UnsupportedBaseError(f'unsupported base kind: "{layer.base_kind}"')
    spec = layer.device(eng)
    if _is_torch(X):
        import torch
        if X.dim() != 2 or X.shape[1] != layer.in_dim:
            raise DimensionError("batch column count does not match in_dim")
        X = X.contiguous().float()
        Y = torch.empty((X.shape[0], layer.out_dim), device=X.device, dtype=torch.float32)
        ext = _torch_enter(eng, X)
        check(lib().lkg_spline_forward(eng.handle, spec.handle, C.c_void_p(X.data_ptr()), X.shape[0],
                                       C.c_void_p(Y.data_ptr())))
        _torch_exit(ext, X, Y)
        return Y
    X = np.asarray(X)
    if X.ndim != 2 or X.shape[1] != layer.in_dim:
        raise DimensionError("batch column count does not match in_dim")
    X = np.ascontiguousarray(X, np.float32)
    Y = np.zeros((X.shape[0], layer.out_dim), np.float32)
    check(lib().lkg_spline_forward_host(eng.handle, spec.handle, X.ctypes.data_as(C.c_void_p), X.shape[0],
                                        Y.ctypes.data_as(C.c_void_p)))
    return Y


# ------------------------------------------------------------------ element primitives (§8a F7-F13, S2, CM3-CM9)
def _f64(x):
    return np.ascontiguousarray(np.atleast_1d(np.asarray(x, np.float64)))


def lut_coords(a: "LutLayerArtifact", x, engine: Engine | None = None) -> dict:
    """safe_clip / segment_index / interp_coords / in_range (runtime.cpp:45-75) of every x, on the
    device in f64: dict of in_range, x_clip, k, l0, l1, w arrays."""
    eng = engine or default_engine()
    xv = _f64(x)
    n = xv.size
    out = dict(in_range=np.zeros(n, np.uint8), x_clip=np.zeros(n), k=np.zeros(n, np.int32),
               l0=np.zeros(n, np.int32), l1=np.zeros(n, np.int32), w=np.zeros(n))
    check(lib().lkg_lut_coords64(eng.handle, a.device(eng).handle, xv.ctypes.data_as(_capi.f64p), n,
                                 *[out[k].ctypes.data_as(t) for k, t in (("in_range", _capi.u8p), ("x_clip", _capi.f64p),
                                                                         ("k", _capi.i32p), ("l0", _capi.i32p),
                                                                         ("l1", _capi.i32p), ("w", _capi.f64p))]))
    out["in_range"] = out["in_range"].astype(bool)
    return out


def in_range(a: "LutLayerArtifact", x, engine: Engine | None = None):
    """runtime.cpp:71-75."""
    r = lut_coords(a, x, engine)["in_range"]
    return bool(r[0]) if np.isscalar(x) else r


def _lut_eval(a, e, x, engine):
    eng = engine or default_engine()
    xv, ev = _f64(x), np.ascontiguousarray(np.atleast_1d(np.asarray(e, np.int32)))
    ev, xv = np.broadcast_arrays(ev, xv)
    ev, xv = np.ascontiguousarray(ev, np.int32), np.ascontiguousarray(xv, np.float64)
    n = xv.size
    val, oob, phi = np.zeros(n), np.zeros(n, np.uint8), np.zeros(n)
    check(lib().lkg_lut_eval(eng.handle, a.device(eng).handle, ev.ctypes.data_as(_capi.i32p),
                             xv.ctypes.data_as(_capi.f64p), n, val.ctypes.data_as(_capi.f64p),
                             oob.ctypes.data_as(_capi.u8p), phi.ctypes.data_as(_capi.f64p)))
    return val, oob.astype(bool), phi


def lut_eval_value(a: "LutLayerArtifact", e, x, engine: Engine | None = None):
    """runtime.cpp:96-109: (value, was_oob) of edge e at x (scalars or broadcastable arrays)."""
    v, o, _ = _lut_eval(a, e, x, engine)
    return (float(v[0]), bool(o[0])) if np.isscalar(x) and np.isscalar(e) else (v, o)


def lut_eval_phi(a: "LutLayerArtifact", e, x, engine: Engine | None = None):
    """runtime.cpp:111-120."""
    _, _, p = _lut_eval(a, e, x, engine)
    return float(p[0]) if np.isscalar(x) and np.isscalar(e) else p


def basis_values(grid: KnotGrid, x, engine: Engine | None = None):
    """spline.cpp:89-94: the R = K + degree basis values at x ([R], or [n, R] for an array x)."""
    eng = engine or default_engine()
    xv = _f64(x)
    bp = np.ascontiguousarray(grid.breakpoints, np.float64)
    R = grid.K + grid.degree
    out = np.zeros((xv.size, R))
    check(lib().lkg_basis_values(eng.handle, bp.ctypes.data_as(_capi.f64p), grid.K, grid.degree,
                                 xv.ctypes.data_as(_capi.f64p), xv.size, out.ctypes.data_as(_capi.f64p)))
    return out[0] if np.isscalar(x) else out


def eval_spline(grid: KnotGrid, coeffs, x, engine: Engine | None = None):
    """spline.cpp:96-103: sum_r c_r B_r(x), r ascending (the reference's order, element-wise)."""
    c = np.asarray(coeffs, np.float64)
    if c.size != grid.K + grid.degree:
        raise DimensionError("coefficient count does not match basis count")
    b = np.atleast_2d(basis_values(grid, x, engine))
    acc = np.zeros(b.shape[0])
    for r in range(c.size):
        acc = acc + c[r] * b[:, r]
    return float(acc[0]) if np.isscalar(x) else acc


def base_fn(kind: str, x):
    """spline.cpp:105-108."""
    if kind != "silu":
        raise UnsupportedBaseError(f'unsupported base kind: "{kind}"')
    xv = np.asarray(x, np.float64)
    return xv / (1.0 + np.exp(-xv))


def eval_edge_phi(layer: KanLayerSpec, e, x, engine: Engine | None = None):
    """spline.cpp:110-115 for edge e = i*out_dim + j of the layer, on the device in f64."""
    if layer.base_kind != "silu":
        raise UnsupportedBaseError(f'unsupported base kind: "{layer.base_kind}"')
    eng = engine or default_engine()
    xv, ev = _f64(x), np.ascontiguousarray(np.atleast_1d(np.asarray(e, np.int32)))
    ev, xv = np.broadcast_arrays(ev, xv)
    ev, xv = np.ascontiguousarray(ev, np.int32), np.ascontiguousarray(xv, np.float64)
    phi = np.zeros(xv.size)
    check(lib().lkg_edge_phi(eng.handle, layer.device(eng).handle, ev.ctypes.data_as(_capi.i32p),
                             xv.ctypes.data_as(_capi.f64p), xv.size, phi.ctypes.data_as(_capi.f64p)))
    return float(phi[0]) if np.isscalar(x) and np.isscalar(e) else phi


def layer_forward(layer: KanLayerSpec, x, tier: Tier = Tier.Optimized, engine: Engine | None = None):
    """spline.cpp:117-125: one row."""
    x = np.asarray(x, np.float32)
    if x.ndim != 1 or x.size != layer.in_dim:
        raise DimensionError("input size does not match in_dim")
    return layer_forward_batch(layer, x[None, :], tier, engine)[0]


def sample_segment_points(breakpoints, k: int, L: int) -> np.ndarray:
    """compiler.cpp:18-27 (x = t_k + l*step, step = (t_k+1 - t_k)/L, right endpoint excluded)."""
    bp = np.asarray(breakpoints, np.float64)
    if L < 2:
        raise ConfigError("samples_per_segment must be >= 2")
    if k < 0 or k + 1 >= bp.size:
        raise DimensionError("segment index out of range")
    step = (bp[k + 1] - bp[k]) / float(L)
    return bp[k] + np.arange(L, dtype=np.float64) * step


def _quantize(values, scheme: int, engine):
    eng = engine or default_engine()
    v = np.ascontiguousarray(np.asarray(values, np.float64))
    if v.size == 0:
        raise ConfigError("cannot quantize an empty segment")
    q, sc, ym = np.zeros(v.size, np.int32), np.zeros(1), np.zeros(1)
    check(lib().lkg_quantize_segments(eng.handle, v.ctypes.data_as(_capi.f64p), 1, v.size, scheme,
                                      q.ctypes.data_as(_capi.i32p), sc.ctypes.data_as(_capi.f64p),
                                      ym.ctypes.data_as(_capi.f64p)))
    return q, float(sc[0]), float(ym[0])


def quantize_segment_symmetric(values, engine: Engine | None = None):
    """compiler.cpp:105-114: (codes, scale, y_min) with scale = amax/127, y_min = 0."""
    return _quantize(values, int(Scheme.Symmetric), engine)


def quantize_segment_asymmetric(values, engine: Engine | None = None):
    """compiler.cpp:116-128: (codes, scale, y_min) with y_min = min, scale = (max - min)/255."""
    return _quantize(values, int(Scheme.Asymmetric), engine)


def build_float_lut(layer: KanLayerSpec, config: QuantConfig | None = None, engine: Engine | None = None):
    """compiler.cpp:29-73: the unquantized table values [E, K*L] (f64), as compile_layer_debug_float
    produces them on the device."""
    a = compile_layer_debug_float(layer, config, OobConfig(), engine)
    return np.asarray(a.float_table).reshape(layer.in_dim * layer.out_dim, -1)


# ------------------------------------------------------------------ artifact container (artifact_io.hpp)
def save_artifact(artifact: "LutLayerArtifact", path, engine: Engine | None = None, store: bool = False,
                  parallel: bool = False) -> None:
    """artifact_io.cpp:206-219: the `.lut` container, byte-identical to the reference's file (ZIP64
    records only when a blob or offset needs them). store=True writes stored entries; parallel=True
    a deflate stream of independently compressed segments that loads on all host threads (both
    readable by the reference). Device artifacts (compiled / loaded) are written from device
    memory; host-array artifacts need no GPU."""
    mode = 1 if store else (2 if parallel else 0)
    if artifact._origin is None:
        d, keep = artifact._desc()
        check(lib().lkg_artifact_save_desc(C.byref(d), os.fsencode(path), mode))
        return
    eng = engine or artifact._origin_engine or default_engine()
    check(lib().lkg_artifact_save(eng.handle, artifact.device(eng).handle, os.fsencode(path), mode))


def artifact_manifest_json(artifact: "LutLayerArtifact") -> str:
    """artifact_io.cpp:98-124 — the manifest text exactly as save_artifact writes it (host only)."""
    d = _capi.LayerDesc()
    K = artifact._origin.info.K if artifact._origin is not None else artifact.K  # no table download
    d.in_dim, d.out_dim, d.K, d.L = artifact.in_dim, artifact.out_dim, K, artifact.L
    d.value_repr, d.interp, d.scheme = int(artifact.value_repr), 0, int(artifact.scheme)
    d.dtype, d.param_dtype = int(artifact.dtype), int(artifact.param_dtype)
    d.boundary_mode, d.oob_policy = int(artifact.oob.boundary_mode), int(artifact.oob.oob_policy)
    base = (artifact.base_kind or "").encode()
    d.base_kind = base
    n = C.c_size_t()
    check(lib().lkg_artifact_manifest(C.byref(d), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().lkg_artifact_manifest(C.byref(d), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def check_artifact(path) -> None:
    """Every load_artifact check (artifact_io.cpp:221-300 + finalize) without a device upload;
    raises the reference's error class."""
    check(lib().lkg_artifact_check(os.fsencode(path)))


def load_artifact(path, engine: Engine | None = None) -> "LutLayerArtifact":
    """artifact_io.cpp:221-300 straight to device memory; host arrays materialise lazily."""
    eng = engine or default_engine()
    h = C.c_void_p()
    check(lib().lkg_artifact_load(eng.handle, os.fsencode(path), C.byref(h)))
    dl = DeviceLayer(h)
    i = dl.info
    sr = i.value_repr == int(ValueRepr.SplineComponent)
    a = LutLayerArtifact(i.in_dim, i.out_dim, i.L, ValueRepr(i.value_repr), Scheme(i.scheme), Dtype(i.scheme),
                         ParamDtype(i.param_dtype), OobConfig(BoundaryMode(i.boundary_mode), OobPolicy(i.oob_policy)),
                         "silu" if sr else "")
    a._origin, a._origin_engine = dl, eng
    return a


# ------------------------------------------------------------------ accuracy (metrics.hpp)
@dataclass
class MemoryBreakdown:
    """metrics.hpp:17-33 — exact byte accounting of an artifact next to its float model."""
    q_table_bytes: int = 0
    scale_bytes: int = 0
    y_min_bytes: int = 0
    knots_bytes: int = 0
    edge_scalar_bytes: int = 0
    total_bytes: int = 0
    float_model_bytes: int = 0
    overhead_ratio: float = 0.0

    def q_table_frac(self) -> float:
        return 0.0 if self.total_bytes == 0 else self.q_table_bytes / self.total_bytes


def memory_breakdown(artifact: "LutLayerArtifact", layer: KanLayerSpec) -> MemoryBreakdown:
    """metrics.cpp:8-28 (host arithmetic on the shapes; no table is downloaded)."""
    E, K, L = artifact.in_dim * artifact.out_dim, artifact.K, artifact.L
    ps = 2 if artifact.param_dtype == ParamDtype.F16 else 4
    m = MemoryBreakdown()
    m.q_table_bytes = E * K * L
    m.scale_bytes = E * K * ps
    m.y_min_bytes = E * K * ps
    m.knots_bytes = (K + 1) * 4
    m.edge_scalar_bytes = 3 * E * 4 if artifact.value_repr == ValueRepr.SplineComponent else 0
    m.total_bytes = m.q_table_bytes + m.scale_bytes + m.y_min_bytes + m.knots_bytes + m.edge_scalar_bytes
    m.float_model_bytes = 4 * layer.in_dim * layer.out_dim * (layer.grid.K + layer.grid.degree + 3)
    m.overhead_ratio = 0.0 if m.float_model_bytes == 0 else m.total_bytes / m.float_model_bytes
    return m


@dataclass
class EvalReport:
    """metrics.hpp:49-76. mae_oob / maxabs_oob are None when the OOB bucket is empty."""
    quant: QuantConfig
    oob: OobConfig
    seed: int = 0
    n_samples: int = 0
    mae_inrange: float = 0.0
    maxabs_inrange: float = 0.0
    mae_oob: float | None = None
    maxabs_oob: float | None = None
    oob_any_frac: float = 0.0
    n_inrange_evals: int = 0
    n_oob_evals: int = 0
    n_boundary_evals: int = 0
    memory: MemoryBreakdown = field(default_factory=MemoryBreakdown)


def eval_accuracy(layer: KanLayerSpec, artifact: "LutLayerArtifact", X, engine: Engine | None = None) -> EvalReport:
    """metrics.cpp:30-103 on the GPU (csrc/eval.cu): |LUT - spline| per (sample, input, edge) in f64."""
    eng = engine or default_engine()
    if layer.in_dim != artifact.in_dim or layer.out_dim != artifact.out_dim:
        raise DimensionError("layer and artifact shapes differ")
    if layer.base_kind != "silu":
        raise UnsupportedBaseError(f'unsupported base kind: "{layer.base_kind}"')
    spec, dl = layer.device(eng), artifact.device(eng)
    r = _capi.EvalReportC()
    if _is_torch(X):
        if X.dim() != 2 or X.shape[1] != layer.in_dim:
            raise DimensionError("input column count does not match in_dim")
        X = X.contiguous().float()
        check(lib().lkg_eval_accuracy(eng.handle, spec.handle, dl.handle, C.c_void_p(X.data_ptr()), X.shape[0],
                                      C.byref(r)))
    else:
        X = np.asarray(X)
        if X.ndim != 2 or X.shape[1] != layer.in_dim:
            raise DimensionError("input column count does not match in_dim")
        if X.dtype == np.float64:  # the reference's f64 Matrix values, evaluated unrounded
            X = np.ascontiguousarray(X)
            check(lib().lkg_eval_accuracy_host_f64(eng.handle, spec.handle, dl.handle, X.ctypes.data_as(C.c_void_p),
                                                   X.shape[0], C.byref(r)))
        else:
            X = np.ascontiguousarray(X, np.float32)
            check(lib().lkg_eval_accuracy_host(eng.handle, spec.handle, dl.handle, X.ctypes.data_as(C.c_void_p),
                                               X.shape[0], C.byref(r)))
    q = QuantConfig(artifact.L, artifact.scheme, artifact.dtype, artifact.value_repr, artifact.interp,
                    artifact.param_dtype)
    return EvalReport(q, artifact.oob, 0, int(r.n_samples), r.mae_inrange, r.maxabs_inrange,
                      r.mae_oob if r.has_oob else None, r.maxabs_oob if r.has_oob else None, r.oob_any_frac,
                      int(r.n_inrange_evals), int(r.n_oob_evals), int(r.n_boundary_evals),
                      memory_breakdown(artifact, layer))


# ------------------------------------------------------------------ recipes
def gen_layer(seed: int, in_dim: int, out_dim: int, segments: int, degree: int = 3) -> KanLayerSpec:
    """model_gen.cpp:7-27 (the reference's test-model generator)."""
    R, E = segments + degree, in_dim * out_dim
    bp, co = np.zeros(max(segments, 0) + 1), np.zeros(max(E * R, 0))
    bs, ss, os_ = np.zeros(max(E, 0)), np.zeros(max(E, 0)), np.zeros(max(E, 0))
    check(lib().lkg_gen_layer(seed, in_dim, out_dim, segments, degree,
                              *[a.ctypes.data_as(_capi.f64p) for a in (bp, co, bs, ss, os_)]))
    return KanLayerSpec(in_dim, out_dim, KnotGrid(bp, degree), co.reshape(E, R), bs, ss, os_)


def gen_sanity_layer(seed: int) -> KanLayerSpec:
    """model_gen.cpp:29-31."""
    return gen_layer(seed, 10, 8, 8, 3)


def gen_inputs(seed: int, n: int, dim: int, lo: float, hi: float, clip: bool) -> np.ndarray:
    """model_gen.cpp:33-45: [n, dim] f64 standard normals, clamped to [lo, hi] when clip."""
    X = np.zeros((n, dim))
    check(lib().lkg_gen_inputs(seed, n, dim, lo, hi, int(clip), X.ctypes.data_as(_capi.f64p)))
    return X


def recipe_dims(cfg: int):
    nl, G = C.c_int32(), C.c_int32()
    dims = (C.c_int32 * 5)()
    lo, hi = C.c_double(), C.c_double()
    check(lib().lkg_recipe_dims(cfg, C.byref(nl), dims, C.byref(G), C.byref(lo), C.byref(hi)))
    return list(dims[: nl.value + 1]), G.value, lo.value, hi.value


def recipe_layer(cfg: int, layer: int, col0: int = 0, col1: int = 0) -> KanLayerSpec:
    """Layer `layer` of BASELINE config `cfg` (DESIGN.md §3 recipe), optionally a column shard."""
    dims, G, _, _ = recipe_dims(cfg)
    if not 0 <= layer < len(dims) - 1:
        raise DimensionError("layer out of range")
    d, m = dims[layer], dims[layer + 1]
    mc = (col1 - col0) if col1 > col0 else m
    E, R = d * mc, G + 3
    bp, co = np.zeros(G + 1), np.zeros(E * R)
    bs, ss, os_ = np.zeros(E), np.zeros(E), np.zeros(E)
    check(lib().lkg_recipe_layer(cfg, layer, col0, col1, *[a.ctypes.data_as(_capi.f64p) for a in (bp, co, bs, ss, os_)]))
    spec = KanLayerSpec(d, mc, KnotGrid(bp, 3), co.reshape(E, R), bs, ss, os_)
    if col1 > col0:
        spec.col0, spec.full_out_dim = col0, m
    return spec


def recipe_inputs(cfg: int, row0: int, rows: int, out: np.ndarray | None = None) -> np.ndarray:
    dims, _, _, _ = recipe_dims(cfg)
    X = out if out is not None else np.zeros((rows, dims[0]), np.float32)
    check(lib().lkg_recipe_inputs(cfg, row0, rows, X.ctypes.data_as(_capi.f32p)))
    return X
