"""Multi-GPU partitioning.

CPU (gloo, world_size 2): the column-shard plan and the rank-major all-gather layout are
checked end to end with the oracle doing each rank's arithmetic — every rank evaluates only its
own output columns, the shards are exchanged with a real all_gather, the next layer consumes the
gathered blocks, and the result equals the unsharded chain bit for bit. Batch sharding likewise.

GPU (-m gpu, one B200): the same layouts through the CUDA path — column shards compiled and
evaluated separately reproduce the full layer exactly, the blocked-input entry point
(lkg_layer_forward_blocked) consumes the all-gather layout, and the NCCL column-sharded chain
(lkg_model_forward_sharded, 1-rank communicator here) equals the unsharded chain.
"""
import os
import socket

import numpy as np
import pytest

from helpers import assert_close, to_oracle_spec, to_product_artifact


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _model(seed=3):
    from oracle.pyoracle import Spec
    rng = np.random.default_rng(seed)
    dims = [6, 8, 4]
    bp = np.linspace(-1.0, 1.0, 6)
    specs = []
    for l in range(2):
        E = dims[l] * dims[l + 1]
        specs.append(Spec(dims[l], dims[l + 1], bp, rng.normal(0, 0.1, (E, 8)), rng.uniform(-1, 1, E), np.ones(E),
                          np.ones(E)))
    X = rng.uniform(-1.2, 1.2, (40, dims[0])).astype(np.float32).astype(np.float64)
    return specs, X


def _col_spec(spec, c0, c1):
    from oracle.pyoracle import Spec
    m = spec.out_dim
    idx = (np.arange(spec.in_dim)[:, None] * m + np.arange(c0, c1)[None, :]).ravel()
    return Spec(spec.in_dim, c1 - c0, spec.breakpoints, spec.coeffs[idx], spec.base_scale[idx],
                spec.spline_scale[idx], spec.out_scale[idx], spec.degree)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import Oracle
        from paper_2601_03332_b200.sharding import batch_bounds, blocked_to_rowmajor, column_bounds
        o = Oracle("auto")
        specs, X = _model()
        rows = X.shape[0]
        cur = X
        for l, spec in enumerate(specs):
            c0, c1 = column_bounds(spec.out_dim, world, rank)
            art = o.compile_layer(_col_spec(spec, c0, c1), 16, 1, 1, 0, 1, 1)  # this rank's edges only
            y_local, _ = o.lut_forward(art, cur)
            t = torch.from_numpy(np.ascontiguousarray(y_local))
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)                       # rank-major blocks [world][rows][m/world]
            gathered = torch.stack(parts).numpy()
            cur = blocked_to_rowmajor(gathered, rows, world, c1 - c0)
        full = [o.compile_layer(s, 16, 1, 1, 0, 1, 1) for s in specs]
        ref, _ = o.lut_model_forward(full, X)
        ok_cols = bool(np.array_equal(cur, ref))
        # batch sharding: each rank its rows, gathered back in order
        r0, r1 = batch_bounds(rows, world, rank)
        yb, st = o.lut_model_forward(full, X[r0:r1])
        parts = [None] * world
        dist.all_gather_object(parts, (r0, yb))
        yall = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
        ok_rows = bool(np.array_equal(yall, ref))
        q.put((rank, ok_cols, ok_rows))
    finally:
        dist.destroy_process_group()


def test_column_and_batch_sharding_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert res == [(0, True, True), (1, True, True)]


def test_shard_plan_and_layout_helpers():
    from paper_2601_03332_b200.sharding import (batch_bounds, blocked_to_rowmajor, column_bounds,
                                                rowmajor_to_blocked)
    import paper_2601_03332_b200 as lk
    assert [column_bounds(4096, 8, g) for g in (0, 7)] == [(0, 512), (3584, 4096)]
    with pytest.raises(lk.DimensionError):
        column_bounds(10, 4, 0)
    b = [batch_bounds(1_048_576, 8, g) for g in range(8)]
    assert b[0][0] == 0 and b[-1][1] == 1_048_576 and all(b[g][1] == b[g + 1][0] for g in range(7))
    x = np.arange(5 * 12, dtype=np.float32).reshape(5, 12)
    blk = rowmajor_to_blocked(x, 3)
    assert blk.shape == (3, 5, 4)
    assert np.array_equal(blocked_to_rowmajor(blk, 5, 3, 4), x)


# ------------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_column_shards_and_blocked_input_gpu(lk, oracle, engine):
    import torch
    from paper_2601_03332_b200.sharding import layer_forward_blocked, rowmajor_to_blocked
    qc = lk.QuantConfig(32)
    oob = lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX)
    full0 = lk.compile_layer(lk.recipe_layer(3, 0), qc, oob, engine=engine)
    shards = [lk.compile_layer(lk.recipe_layer(3, 0, c0, c0 + 32), qc, oob, engine=engine) for c0 in (0, 32)]
    layer1 = lk.compile_layer(lk.recipe_layer(3, 1), qc, oob, engine=engine)
    X = torch.from_numpy(lk.recipe_inputs(3, 0, 3000)).cuda()
    Yfull, _ = lk.lut_layer_forward_batch(full0, X, engine=engine)
    parts = [lk.lut_layer_forward_batch(s, X, engine=engine)[0] for s in shards]
    assert torch.equal(torch.cat(parts, dim=1), Yfull)       # column shards == the full layer, bit for bit
    gathered = torch.stack(parts).contiguous()                 # the all-gather layout [2][rows][32]
    Yb, st = layer_forward_blocked(layer1, gathered, 32, engine)
    Yr, st_r = lk.lut_layer_forward_batch(layer1, Yfull, engine=engine)
    assert torch.equal(Yb, Yr)
    assert (st.n_oob_inputs, st.n_oob_samples) == (st_r.n_oob_inputs, st_r.n_oob_samples)
    H = Yfull.cpu().numpy()
    o1 = oracle.compile_layer(to_oracle_spec(lk.recipe_layer(3, 1)), 32, 0, 1, 0, 0, 0)
    Yo, _ = oracle.lut_forward(o1, H.astype(np.float64))
    assert_close(Yb.cpu().numpy(), Yo, "blocked layer 1")
    assert np.array_equal(rowmajor_to_blocked(H, 2), gathered.cpu().numpy())


@pytest.mark.gpu
def test_blocked_input_into_record_walk_gpu(lk, engine):
    """Wide layers of a column-sharded chain read the all-gathered activations in rank-major blocks:
    the coordinate-record / transposed-input passes take that layout directly, so such layers keep
    the record walk (and its bits) behind an all-gather. A 64 -> 64 layer (4 j-blocks, fp32) from 2
    blocks of 32 and a 1024 -> 256 layer (16 j-blocks, f64 TMEM) from 4 blocks of 256, both against the
    row-major call."""
    import torch
    from paper_2601_03332_b200.sharding import layer_forward_blocked, rowmajor_to_blocked
    oob = lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX)
    for spec, rows, world in ((lk.recipe_layer(3, 0), 3001, 2), (lk.gen_layer(9, 1024, 256, 8), 2048, 4)):
        art = lk.compile_layer(spec, lk.QuantConfig(64), oob, engine=engine)
        X = np.random.default_rng(rows).uniform(-1.2, 1.2, (rows, spec.in_dim)).astype(np.float32)
        Yr, st_r = lk.lut_layer_forward_batch(art, torch.from_numpy(X).cuda(), engine=engine)
        blk = torch.from_numpy(rowmajor_to_blocked(X, world)).cuda()
        Yb, st_b = layer_forward_blocked(art, blk, spec.in_dim // world, engine)
        assert torch.equal(Yb, Yr)
        assert (st_b.n_oob_inputs, st_b.n_oob_samples) == (st_r.n_oob_inputs, st_r.n_oob_samples)


@pytest.mark.gpu
def test_nccl_sharded_chain_one_rank(lk, engine):
    import torch
    from paper_2601_03332_b200.sharding import ColumnShardedChain
    eng = lk.Engine(0)
    eng.init_nccl(lk.nccl_unique_id(), 1, 0)
    qc = lk.QuantConfig(64)
    oob = lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX)
    specs = [lk.recipe_layer(3, l) for l in range(2)]
    chain = ColumnShardedChain.compile(specs, [64, 1], qc, oob, eng, 1, 0)
    X = torch.from_numpy(lk.recipe_inputs(3, 0, 5000)).cuda()
    Y, st = chain.forward(X)
    ref = lk.lut_model_forward_batch(chain.layers, X, engine=eng)
    assert torch.equal(Y, ref.Y)
    assert [(s.n_oob_inputs, s.n_oob_samples) for s in st] == [(s.n_oob_inputs, s.n_oob_samples) for s in ref.per_layer]


@pytest.mark.gpu
def test_nccl_sharded_chain_row_chunks_overlap(tmp_path):
    """The row-chunked pipeline of the column-sharded chain (all-gather of chunk c on the
    communication stream while the next chunk computes; LKG_SHARD_CHUNKS=3, 1-rank NCCL, a
    3-layer C4-shaped chain so a long-reduction layer consumes the gathered blocks) equals the
    unsharded chain bit for bit, stats included."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import paper_2601_03332_b200 as lk\n"
        "from paper_2601_03332_b200.sharding import ColumnShardedChain\n"
        "eng = lk.Engine(0); eng.init_nccl(lk.nccl_unique_id(), 1, 0)\n"
        "specs = [lk.recipe_layer(4, l) for l in range(3)]\n"
        "chain = ColumnShardedChain.compile(specs, [1024, 1024, 10], lk.QuantConfig(64), lk.OobConfig(), eng, 1, 0)\n"
        "X = torch.from_numpy(lk.recipe_inputs(4, 0, 3001)).cuda()\n"
        "Y, st = chain.forward(X)\n"
        "ref = lk.lut_model_forward_batch(chain.layers, X, engine=eng)\n"
        "assert torch.equal(Y, ref.Y), (Y - ref.Y).abs().max()\n"
        "assert [(s.n_oob_inputs, s.n_oob_samples) for s in st] == "
        "[(s.n_oob_inputs, s.n_oob_samples) for s in ref.per_layer]\n"
        "print('ok')\n") % root
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LKG_SHARD_CHUNKS="3"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])


@pytest.mark.gpu
def test_nccl_sharded_chain_row_chunks_widening(tmp_path):
    """Row-chunked column-sharded chain whose hidden width GROWS ([64, 32, 64, 48, 2]): chunk c
    of every layer owns a fixed region of the scratch and gather buffers (sized by the widest
    layer), so a wider layer l+1 never writes over layer l's chunks c+1.. while their gathers are
    in flight on the communication stream (LKG_SHARD_CHUNKS=3, 1-rank NCCL). Equal bit for bit to
    the unsharded chain, stats included."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import paper_2601_03332_b200 as lk\n"
        "from paper_2601_03332_b200.sharding import ColumnShardedChain\n"
        "eng = lk.Engine(0); eng.init_nccl(lk.nccl_unique_id(), 1, 0)\n"
        "dims = [64, 32, 64, 48, 2]\n"
        "specs = [lk.gen_layer(11 + l, dims[l], dims[l + 1], 8) for l in range(4)]\n"
        "chain = ColumnShardedChain.compile(specs, dims[1:], lk.QuantConfig(64), lk.OobConfig(), eng, 1, 0)\n"
        "for rows in (70001, 9000):\n"
        "    X = torch.empty((rows, 64), device='cuda').uniform_(-1.2, 1.2)\n"
        "    for _ in range(3):\n"
        "        Y, st = chain.forward(X)\n"
        "        ref = lk.lut_model_forward_batch(chain.layers, X, engine=eng)\n"
        "        assert torch.equal(Y, ref.Y), (Y - ref.Y).abs().max()\n"
        "        assert [(s.n_oob_inputs, s.n_oob_samples) for s in st] == "
        "[(s.n_oob_inputs, s.n_oob_samples) for s in ref.per_layer]\n"
        "print('ok')\n") % root
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LKG_SHARD_CHUNKS="3"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])


@pytest.mark.gpu
def test_batch_shards_and_host_chunks_bit_identical(lk):
    """Batch shards (batch_bounds: 64-row aligned starts) and the host path's row chunks give
    every row exactly the bits of one whole-batch launch (bit-identical to 1 GPU)."""
    import torch
    from paper_2601_03332_b200.sharding import batch_bounds
    for cfg, layer, rows in ((3, 0, 5000), (4, 1, 3001), (2, 1, 4099)):
        spec = lk.recipe_layer(cfg, layer)
        a = lk.compile_layer(spec, lk.QuantConfig(64), lk.OobConfig())
        X = torch.empty((rows, spec.in_dim), device="cuda").uniform_(-1.3, 1.3)
        Y, _ = lk.lut_layer_forward_batch(a, X)
        for world in (2, 3, 8):
            parts = []
            for r in range(world):
                r0, r1 = batch_bounds(rows, world, r)
                if r1 > r0:
                    parts.append(lk.lut_layer_forward_batch(a, X[r0:r1].contiguous())[0])
            assert torch.equal(torch.cat(parts), Y), (cfg, layer, world)
    spec = lk.recipe_layer(2, 0)
    a = lk.compile_layer(spec, lk.QuantConfig(64), lk.OobConfig())
    X = lk.recipe_inputs(2, 0, 250000)              # > 2 host-path chunks of X
    Yh, sh = lk.lut_layer_forward_batch(a, X)
    Yd, sd = lk.lut_layer_forward_batch(a, torch.from_numpy(X).cuda())
    assert np.array_equal(Yh, Yd.cpu().numpy()) and sh.n_oob_inputs == sd.n_oob_inputs
