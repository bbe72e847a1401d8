"""B200-native LUT-KAN inference engine (arXiv 2601.03332 hot path).

Drop-in for the reference ``lutkan`` core hot path: LUT compile, LUT layer/model
forward and the same-backend B-spline forward, executed by hand-written sm_100a
CUDA kernels in ``liblutkan_b200.so`` behind the C-ABI ``include/lutkan_b200.h``.
"""
from .lutkan import (  # noqa: F401
    BoundaryMode, ChainBatchResult, ChainGraph, ConfigError, CudaError, DimensionError, Dtype, Engine, Error, EvalReport,
    Interp, KanLayerSpec, MemoryBreakdown, eval_accuracy, memory_breakdown, IoError, CorruptArchiveError,
    CorruptBlobError, MissingKeyError, ShapeError, VersionError, EnumError, save_artifact, load_artifact, check_artifact, artifact_manifest_json, lut_coords, in_range,
    lut_eval_value, lut_eval_phi, basis_values, eval_spline, base_fn, eval_edge_phi, layer_forward,
    sample_segment_points, quantize_segment_symmetric, quantize_segment_asymmetric, build_float_lut,
    gen_layer, gen_sanity_layer, gen_inputs, KnotGrid, LutLayerArtifact, NcclError, NonFiniteError, OobConfig, OobPolicy, OobStats,
    ParamDtype, QuantConfig, Scheme, Tier, UnsupportedBaseError, ValueRepr, compile_layer,
    compile_layer_debug_float, compile_model, default_engine, layer_forward_batch, lut_layer_forward,
    lut_layer_forward_batch, lut_model_forward, lut_model_forward_batch, nccl_unique_id, parse_enum,
    recipe_dims, recipe_inputs, recipe_layer)

__all__ = [n for n in dir() if not n.startswith("_")]
