"""ctypes binding of liblutkan_b200.so (include/lutkan_b200.h).

The CUDA library is the only execution path: importing this module on a machine
without the built library raises, and every call that needs a GPU fails loudly
with the library's own CUDA error — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LKG_LIB") or os.path.join(PKG, "liblutkan_b200.so")  # LKG_LIB: A/B experiments

_P = C.POINTER
f32p, f64p, u8p, i32p = _P(C.c_float), _P(C.c_double), _P(C.c_uint8), _P(C.c_int32)

OK, ERR_CONFIG, ERR_DIMENSION, ERR_NON_FINITE, ERR_UNSUPPORTED_BASE, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_INVALID_ARG = range(9)
# artifact container I/O (artifact_io.hpp:11-52)
ERR_IO, ERR_CORRUPT_ARCHIVE, ERR_CORRUPT_BLOB, ERR_MISSING_KEY, ERR_SHAPE, ERR_VERSION, ERR_ENUM = range(9, 16)


class LayerDesc(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("out_dim", C.c_int32), ("K", C.c_int32), ("L", C.c_int32),
                ("value_repr", C.c_int32), ("interp", C.c_int32), ("scheme", C.c_int32), ("dtype", C.c_int32),
                ("param_dtype", C.c_int32), ("boundary_mode", C.c_int32), ("oob_policy", C.c_int32),
                ("base_kind", C.c_char_p), ("knots", f32p), ("q_table", u8p), ("scale", f32p), ("y_min", f32p),
                ("edge_base_scale", f32p), ("edge_spline_scale", f32p), ("edge_out_scale", f32p),
                ("float_table", f64p)]


class SpecDesc(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("out_dim", C.c_int32), ("K", C.c_int32), ("degree", C.c_int32),
                ("base_kind", C.c_char_p), ("breakpoints", f64p), ("coeffs", f64p), ("base_scale", f64p),
                ("spline_scale", f64p), ("out_scale", f64p)]


class QuantCfg(C.Structure):
    _fields_ = [("L", C.c_int32), ("scheme", C.c_int32), ("dtype", C.c_int32), ("value_repr", C.c_int32),
                ("interp", C.c_int32), ("param_dtype", C.c_int32)]


class OobCfg(C.Structure):
    _fields_ = [("boundary_mode", C.c_int32), ("oob_policy", C.c_int32)]


class OobStatsC(C.Structure):
    _fields_ = [("n_samples", C.c_uint64), ("n_oob_samples", C.c_uint64), ("n_inputs", C.c_uint64),
                ("n_oob_inputs", C.c_uint64)]


class LayerInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("in_dim", "out_dim", "K", "L", "col0", "col1", "full_out_dim",
                                         "value_repr", "scheme", "param_dtype", "boundary_mode", "oob_policy",
                                         "has_float_table")] + [("device_bytes", C.c_uint64)]


class EvalReportC(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("mae_inrange", "maxabs_inrange", "mae_oob", "maxabs_oob", "oob_any_frac")] + \
               [(n, C.c_uint64) for n in ("n_samples", "n_inrange_evals", "n_oob_evals", "n_boundary_evals",
                                          "n_oob_samples")] + [("has_oob", C.c_int32)]


# name -> (restype, argtypes); the exported C-ABI, one entry per declaration in the header.
SIGNATURES = {
    "lkg_last_error": (C.c_char_p, []),
    "lkg_version": (C.c_char_p, []),
    "lkg_ctx_create": (C.c_int, [C.c_int32, C.c_void_p, _P(C.c_void_p)]),
    "lkg_ctx_destroy": (C.c_int, [C.c_void_p]),
    "lkg_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "lkg_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "lkg_ctx_launch_count": (C.c_uint64, [C.c_void_p]),
    "lkg_ctx_workspace_bytes": (C.c_uint64, [C.c_void_p]),
    "lkg_ctx_trim": (C.c_int, [C.c_void_p]),
    "lkg_layer_upload": (C.c_int, [C.c_void_p, _P(LayerDesc), _P(C.c_void_p)]),
    "lkg_layer_upload_columns": (C.c_int, [C.c_void_p, _P(LayerDesc), C.c_int32, C.c_int32, _P(C.c_void_p)]),
    "lkg_layer_info_get": (C.c_int, [C.c_void_p, _P(LayerInfo)]),
    "lkg_layer_base_kind": (C.c_char_p, [C.c_void_p]),
    "lkg_layer_download": (C.c_int, [C.c_void_p, C.c_void_p, f32p, u8p, f32p, f32p, f32p, f32p, f32p, f64p]),
    "lkg_layer_free": (C.c_int, [C.c_void_p]),
    "lkg_spec_upload": (C.c_int, [C.c_void_p, _P(SpecDesc), _P(C.c_void_p)]),
    "lkg_spec_upload_columns": (C.c_int, [C.c_void_p, _P(SpecDesc), C.c_int32, C.c_int32, _P(C.c_void_p)]),
    "lkg_spec_upload_shard": (C.c_int, [C.c_void_p, _P(SpecDesc), C.c_int32, C.c_int32, _P(C.c_void_p)]),
    "lkg_spec_free": (C.c_int, [C.c_void_p]),
    "lkg_compile_layer": (C.c_int, [C.c_void_p, C.c_void_p, _P(QuantCfg), _P(OobCfg), C.c_int32, _P(C.c_void_p)]),
    "lkg_layer_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, _P(OobStatsC)]),
    "lkg_model_forward": (C.c_int, [C.c_void_p, _P(C.c_void_p), C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                    _P(OobStatsC)]),
    "lkg_model_forward_host": (C.c_int, [C.c_void_p, _P(C.c_void_p), C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                         _P(OobStatsC)]),
    "lkg_layer_forward_blocked": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                            _P(OobStatsC)]),
    "lkg_layer_coords": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
    "lkg_ctx_collect": (C.c_int, [C.c_void_p, _P(OobStatsC), C.c_int32]),
    "lkg_spline_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "lkg_ctx_set_spline_kernel": (C.c_int, [C.c_void_p, C.c_int32]),
    "lkg_model_forward_host_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                             C.c_void_p]),
    "lkg_spline_forward_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "lkg_artifact_save": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p, C.c_int32]),
    "lkg_artifact_load": (C.c_int, [C.c_void_p, C.c_char_p, _P(C.c_void_p)]),
    "lkg_artifact_save_desc": (C.c_int, [_P(LayerDesc), C.c_char_p, C.c_int32]),
    "lkg_artifact_check": (C.c_int, [C.c_char_p]),
    "lkg_graph_create": (C.c_int, [C.c_void_p, _P(C.c_void_p), C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                   _P(C.c_void_p)]),
    "lkg_graph_launch": (C.c_int, [C.c_void_p]),
    "lkg_graph_destroy": (C.c_int, [C.c_void_p]),
    "lkg_artifact_manifest": (C.c_int, [_P(LayerDesc), C.c_char_p, C.c_size_t, _P(C.c_size_t)]),
    "lkg_lut_coords64": (C.c_int, [C.c_void_p, C.c_void_p, f64p, C.c_int64, u8p, f64p, i32p, i32p, i32p, f64p]),
    "lkg_lut_eval": (C.c_int, [C.c_void_p, C.c_void_p, i32p, f64p, C.c_int64, f64p, u8p, f64p]),
    "lkg_basis_values": (C.c_int, [C.c_void_p, f64p, C.c_int32, C.c_int32, f64p, C.c_int64, f64p]),
    "lkg_edge_phi": (C.c_int, [C.c_void_p, C.c_void_p, i32p, f64p, C.c_int64, f64p]),
    "lkg_quantize_segments": (C.c_int, [C.c_void_p, f64p, C.c_int64, C.c_int32, C.c_int32, i32p, f64p, f64p]),
    "lkg_eval_accuracy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, _P(EvalReportC)]),
    "lkg_eval_accuracy_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                         _P(EvalReportC)]),
    "lkg_eval_accuracy_host_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                             _P(EvalReportC)]),
    "lkg_nccl_unique_id": (C.c_int, [_P(C.c_uint8)]),
    "lkg_ctx_init_nccl": (C.c_int, [C.c_void_p, _P(C.c_uint8), C.c_int32, C.c_int32]),
    "lkg_model_forward_sharded": (C.c_int, [C.c_void_p, _P(C.c_void_p), C.c_int32, C.c_void_p, C.c_int64,
                                            C.c_void_p, _P(OobStatsC)]),
    "lkg_recipe_dims": (C.c_int, [C.c_int32, i32p, i32p, i32p, f64p, f64p]),
    "lkg_recipe_layer": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, f64p, f64p, f64p, f64p, f64p]),
    "lkg_gen_layer": (C.c_int, [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, f64p, f64p, f64p, f64p,
                                f64p]),
    "lkg_gen_inputs": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32, f64p]),
    "lkg_recipe_inputs": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, f32p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree CUDA library (built by paper_2601_03332_b200.build); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib
