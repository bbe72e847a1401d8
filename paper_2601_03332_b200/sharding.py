"""Multi-GPU partitioning of the LUT-KAN forward, one process per GPU.

* Batch sharding (configs[3], "C4"): rank g evaluates rows [g*B/G, (g+1)*B/G) against a full
  replica of the LUT; no collective. Results are bit-identical to one GPU because every row is
  computed by exactly the same kernel arithmetic.
* Output-column sharding (configs[4], "C5"): rank g holds the edges (i, j) with j in
  J_g = [g*m/G, (g+1)*m/G) of every layer — for each input row i one contiguous run of the
  reference q_table (e = i*m + j, spline.hpp:43). Layer l writes y[:, J_g]; an NCCL all-gather
  over NVLink gives every rank the full hidden activations in rank-major blocks
  [G][rows][m/G], which the next layer's kernel reads in place (x_blk = m/G). Column sharding
  does not change any per-(row, j) sum, so results are again identical to one GPU.

The exchange runs inside the C-ABI (lkg_model_forward_sharded: ncclAllGather on the context's
stream); this module holds the plan and the host plumbing (NCCL id broadcast over
torch.distributed).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import lib
from .lutkan import (ConfigError, DimensionError, Engine, KanLayerSpec, LutLayerArtifact, OobConfig, OobStats,
                     QuantConfig, _torch_enter, _torch_exit, check, compile_layer)


ROW_ALIGN = 64  # csrc/lkg_internal.h kRowAlign: shard starts keep every row's lane phase


def batch_bounds(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of `rank` under batch sharding: contiguous, balanced to within ROW_ALIGN rows,
    every shard starting at a multiple of ROW_ALIGN so each row's result is bit-identical to the
    1-GPU run."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")

    def start(r):
        return min(rows, (rows * r // world + ROW_ALIGN - 1) // ROW_ALIGN * ROW_ALIGN)
    return start(rank), (rows if rank == world - 1 else start(rank + 1))


def column_bounds(m: int, world: int, rank: int) -> tuple[int, int]:
    """Output columns [c0, c1) of `rank` under column sharding (equal shards, rank order)."""
    if m % world:
        raise DimensionError(f"out_dim {m} is not divisible by {world} ranks")
    w = m // world
    return rank * w, (rank + 1) * w


def blocked_to_rowmajor(buf: np.ndarray, rows: int, world: int, blk: int) -> np.ndarray:
    """Rank-major all-gather layout [world][rows][blk] -> row-major [rows][world*blk]."""
    return np.ascontiguousarray(np.asarray(buf).reshape(world, rows, blk).transpose(1, 0, 2).reshape(rows, world * blk))


def rowmajor_to_blocked(x: np.ndarray, world: int) -> np.ndarray:
    """Row-major [rows][world*blk] -> rank-major blocks [world][rows][blk] (what all-gather produces)."""
    rows, m = x.shape
    return np.ascontiguousarray(x.reshape(rows, world, m // world).transpose(1, 0, 2))


def init_nccl(engine: Engine, dist) -> None:
    """Create the engine's NCCL communicator over an initialised torch.distributed group."""
    import torch
    from .lutkan import nccl_unique_id
    world, rank = dist.get_world_size(), dist.get_rank()
    if world == 1:
        engine.init_nccl(nccl_unique_id(), 1, 0)
        return
    uid = nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0)
    engine.init_nccl(bytes(t.cpu().tolist()), world, rank)


@dataclass
class ColumnShardedChain:
    """A chain whose every layer is column-sharded over the ranks of `engine`'s communicator."""
    layers: list  # per layer: LutLayerArtifact holding this rank's columns (device-compiled)
    world: int
    rank: int
    engine: Engine

    @staticmethod
    def compile(specs_for_rank: list[KanLayerSpec], full_out_dims: list[int], config: QuantConfig,
                oob: OobConfig, engine: Engine, world: int, rank: int) -> "ColumnShardedChain":
        """specs_for_rank[l] holds this rank's columns of layer l (see recipe_layer(col0, col1));
        each is compiled on this rank's GPU (bit-exact with the reference's compile of those edges)."""
        if len(specs_for_rank) != len(full_out_dims):
            raise ConfigError("one spec per layer")
        for s, m in zip(specs_for_rank, full_out_dims):
            if s.out_dim * world != m:
                raise DimensionError("each rank must hold an equal column shard")
        c0s = [column_bounds(m, world, rank)[0] for m in full_out_dims]
        for s, c0, m in zip(specs_for_rank, c0s, full_out_dims):
            if s.full_out_dim and (s.full_out_dim, s.col0) != (m, c0):
                raise DimensionError("spec shard does not match this rank's columns")
            s.col0, s.full_out_dim = c0, m
        arts = [compile_layer(s, config, oob, engine=engine) for s in specs_for_rank]
        return ColumnShardedChain(arts, world, rank, engine)

    def forward(self, X, Y=None) -> tuple[object, list[OobStats]]:
        """X: torch CUDA tensor [rows, in_dim] (replicated). Returns this rank's columns of the
        last layer [rows, out_dim/world] and per-layer OOB stats (identical on every rank)."""
        import torch
        devs = [a.device(self.engine) for a in self.layers]
        handles = (C.c_void_p * len(devs))(*[d.handle for d in devs])
        X = _cuda_input(X, self.layers[0].in_dim)
        rows = X.shape[0]
        m_out = devs[-1].info.out_dim
        if Y is None:
            Y = torch.empty((rows, m_out), device=X.device, dtype=torch.float32)
        _check_output(Y, X, rows, m_out)
        stats = (_capi.OobStatsC * len(devs))()
        ext = _torch_enter(self.engine, X)
        check(lib().lkg_model_forward_sharded(self.engine.handle, handles, len(devs), C.c_void_p(X.data_ptr()), rows,
                                              C.c_void_p(Y.data_ptr()), stats))
        _torch_exit(ext, X, Y)
        return Y, [OobStats._from(s) for s in stats]


def _cuda_input(X, in_dim: int):
    """A CUDA [rows, in_dim] tensor as the contiguous fp32 the C-ABI reads (as lutkan._forward)."""
    if not (type(X).__module__.startswith("torch") and X.is_cuda):
        raise DimensionError("sharded forwards take CUDA tensors")
    if X.dim() != 2 or X.shape[1] != in_dim:
        raise DimensionError("batch column count does not match artifact in_dim")
    return X.contiguous().float()


def _check_output(Y, X, rows: int, cols: int) -> None:
    import torch
    if not (isinstance(Y, torch.Tensor) and Y.is_cuda and Y.device == X.device and Y.dtype == torch.float32
            and Y.is_contiguous() and tuple(Y.shape) == (rows, cols)):
        raise DimensionError(f"Y must be a contiguous float32 CUDA tensor of shape ({rows}, {cols}) on {X.device}")


def layer_forward_blocked(art: LutLayerArtifact, X, x_blk: int, engine: Engine):
    """One layer on input in the rank-major all-gather layout (torch CUDA tensors)."""
    import torch
    d = art.device(engine)
    if not (isinstance(X, torch.Tensor) and X.is_cuda):
        raise DimensionError("layer_forward_blocked takes a CUDA tensor")
    if x_blk <= 0 or art.in_dim % x_blk or X.numel() % art.in_dim:
        raise DimensionError("blocked input: x_blk must divide in_dim and X must hold rows x in_dim values")
    X = X.contiguous().float()
    rows = X.numel() // art.in_dim
    Y = torch.empty((rows, d.info.out_dim), device=X.device, dtype=torch.float32)
    st = _capi.OobStatsC()
    ext = _torch_enter(engine, X)
    check(lib().lkg_layer_forward_blocked(engine.handle, d.handle, C.c_void_p(X.data_ptr()), rows, x_blk,
                                          C.c_void_p(Y.data_ptr()), C.byref(st)))
    _torch_exit(ext, X, Y)
    return Y, OobStats._from(st)
