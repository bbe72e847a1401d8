"""GPU parity through the C-ABI (liblutkan_b200.so) against the CPU oracle.

Bars (BASELINE.json north_star): LUT bytes / scales / y_mins, segment indices, OOB masks,
OOB counts and argmax classes bit-exact; float outputs within max-abs 1e-5 (relative
1e-5 where |y| > 1), per layer on identical fp32 inputs (the compiled table
is discontinuous at knots, so chains are compared per layer plus argmax).
"""
import numpy as np
import pytest

from helpers import assert_close, hidden_inputs, stats_list, to_oracle_spec, to_product_artifact, to_product_spec
from kat import HAND_CLOSED_CLIPX, HAND_CLOSED_ZS, hand_artifact_arrays

pytestmark = pytest.mark.gpu


def _bytes_equal(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


def _compile_both(lk, oracle, cfg, layer, L, scheme, vr=1, pd=0, bm=1, op=0, keep_float=False):
    spec = lk.recipe_layer(cfg, layer)
    qc = lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme), lk.ValueRepr(vr), lk.Interp.Linear, lk.ParamDtype(pd))
    oob = lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op))
    g = lk.compile_layer_debug_float(spec, qc, oob) if keep_float else lk.compile_layer(spec, qc, oob)
    o = oracle.compile_layer(to_oracle_spec(spec), L, scheme, vr, pd, bm, op, keep_float=keep_float)
    return spec, g, o


# ------------------------------------------------------------------ compile
@pytest.mark.parametrize("cfg,layer,L,scheme", [(1, 0, 64, 0), (1, 1, 64, 0), (2, 0, 64, 0), (2, 0, 64, 1),
                                                (2, 1, 64, 1), (3, 0, 16, 0), (3, 0, 32, 1), (3, 0, 64, 0),
                                                (3, 0, 128, 1), (3, 1, 128, 0)])
def test_compile_bit_exact(lk, oracle, cfg, layer, L, scheme):
    _, g, o = _compile_both(lk, oracle, cfg, layer, L, scheme)
    assert _bytes_equal(g.q_table, o.q)
    assert _bytes_equal(g.scale, o.scale) and _bytes_equal(g.y_min, o.y_min)
    assert _bytes_equal(g.knots, o.knots)
    for a, b in ((g.edge_base_scale, o.base_scale), (g.edge_spline_scale, o.spline_scale), (g.edge_out_scale, o.out_scale)):
        assert _bytes_equal(a, b)


@pytest.mark.parametrize("vr,pd", [(0, 0), (0, 1), (1, 1)])
def test_compile_phi_and_f16_bit_exact(lk, oracle, vr, pd):
    for scheme in (0, 1):
        _, g, o = _compile_both(lk, oracle, 2, 0, 32, scheme, vr, pd, keep_float=True)
        assert _bytes_equal(g.q_table, o.q) and _bytes_equal(g.scale, o.scale) and _bytes_equal(g.y_min, o.y_min)
        assert _bytes_equal(g.float_table, o.float_table)
        if vr == 0:
            assert g.edge_base_scale is None and g.base_kind == ""


def test_compile_large_edge_slices(lk, oracle):
    """C4 (1024x1024, K=8, L=64) compiled whole on the GPU; the oracle compiles per-input-row
    edge slices, which are exactly the matching byte ranges."""
    spec = lk.recipe_layer(4, 0)
    g = lk.compile_layer(spec, lk.QuantConfig(64), lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX))
    os_ = to_oracle_spec(spec)
    m, K, L = 1024, 8, 64
    for i in (0, 1, 511, 1023):
        o = oracle.compile_layer(os_.edge_slice(i, i + 1), 64, 0, 1, 0, 0, 0)
        assert _bytes_equal(g.q_table[i * m * K * L:(i + 1) * m * K * L], o.q)
        assert _bytes_equal(g.scale[i * m * K:(i + 1) * m * K], o.scale)


def test_compile_tiles_only_download(lk, oracle, monkeypatch):
    """Large layers keep their codes only in the forward tiles (the reference-layout copy is
    freed); download rebuilds q_table from the tiles byte for byte. Forced here on a C3 layer."""
    monkeypatch.setenv("LKG_TILE_ONLY_BYTES", "0")
    for scheme, L in ((0, 64), (1, 128)):
        spec = lk.recipe_layer(3, 0)
        g = lk.compile_layer(spec, lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme)), lk.OobConfig())
        o = oracle.compile_layer(to_oracle_spec(spec), L, scheme, 1, 0, 1, 0)
        assert _bytes_equal(g.q_table, o.q)
        X = oracle.recipe_inputs(3, 0, 2000)
        Y, _ = lk.lut_layer_forward_batch(g, X)
        Yo, _ = oracle.lut_forward(o, X.astype(np.float64))
        assert_close(Y, Yo, f"tiles-only L{L}")


def test_compile_c5_column_shard(lk, oracle):
    """C5 geometry (G=16 on [-2,2], L=128, uint8 asym): a column shard compiled on the GPU
    matches the oracle's compile of the same edges."""
    cols = (1024, 1088)
    spec = lk.recipe_layer(5, 0, *cols)
    g = lk.compile_layer(spec, lk.QuantConfig(128, lk.Scheme.Asymmetric, lk.Dtype.Uint8),
                         lk.OobConfig(lk.BoundaryMode.Closed, lk.OobPolicy.ZeroSpline))
    mc, K, L = cols[1] - cols[0], 16, 128
    for i in (0, 4095):
        o = oracle.compile_layer(to_oracle_spec(spec).edge_slice(i, i + 1), 128, 1, 1, 0, 1, 1)
        assert _bytes_equal(g.q_table[i * mc * K * L:(i + 1) * mc * K * L], o.q)
        assert _bytes_equal(g.y_min[i * mc * K:(i + 1) * mc * K], o.y_min)


# ------------------------------------------------------------------ coordinates
@pytest.mark.parametrize("bm", [0, 1])
def test_segment_index_and_mask_bit_exact(lk, oracle, engine, bm):
    import ctypes as C
    import torch
    from paper_2601_03332_b200._capi import lib
    for cfg, L in ((2, 64), (3, 16), (4, 64), (5, 128)):
        spec = lk.recipe_layer(cfg, 0, 0, 1)
        g = lk.compile_layer(spec, lk.QuantConfig(L),
                             lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy.ZeroSpline))
        knots = g.knots
        adv = [knots, np.nextafter(knots, np.float32(np.inf)), np.nextafter(knots, np.float32(-np.inf))]
        # every sample node z = l of every segment (f64 position rounded to f32) and 3 ulps either
        # side: where floor(z) in fp32 can disagree with the reference's f64 z
        kd64 = knots.astype(np.float64)
        nodes = (kd64[:-1, None] + np.arange(L)[None, :] / (L - 1) * np.diff(kd64)[:, None]).ravel().astype(np.float32)
        for _ in range(3):
            adv += [nodes := np.nextafter(nodes, np.float32(np.inf))]
        nodes = (kd64[:-1, None] + np.arange(L)[None, :] / (L - 1) * np.diff(kd64)[:, None]).ravel().astype(np.float32)
        adv.append(nodes)
        for _ in range(3):
            adv += [nodes := np.nextafter(nodes, np.float32(-np.inf))]
        rng = np.random.default_rng(5)
        x = np.concatenate(adv + [rng.uniform(knots[0] * 1.3, knots[-1] * 1.3, 200000).astype(np.float32)])
        x = x.astype(np.float32)
        xd = torch.from_numpy(x).cuda()
        ind, kd, l0d = (torch.zeros(len(x), dtype=torch.int32, device="cuda") for _ in range(3))
        dl = g.device(engine)
        torch.cuda.synchronize()
        lk.lutkan.check(lib().lkg_layer_coords(engine.handle, dl.handle, C.c_void_p(xd.data_ptr()), len(x),
                                               C.c_void_p(ind.data_ptr()), C.c_void_p(kd.data_ptr()),
                                               C.c_void_p(l0d.data_ptr())))
        from oracle.pyoracle import Artifact
        oa = Artifact(1, 1, g.L, g.knots, g.q_table, g.scale, g.y_min, g.edge_base_scale, g.edge_spline_scale,
                      g.edge_out_scale, 1, 0, 0, bm, 1)
        c = oracle.coords(oa, x.astype(np.float64))
        assert np.array_equal(ind.cpu().numpy().astype(bool), c["in_range"])
        assert np.array_equal(kd.cpu().numpy(), c["k"])
        l0_mis = np.mean(l0d.cpu().numpy() != c["l0"])
        assert l0_mis == 0.0, l0_mis


# ------------------------------------------------------------------ forward
def _layer_parity(lk, oracle, art_o, X, what):
    a = to_product_artifact(lk, art_o)
    Y, st = lk.lut_layer_forward_batch(a, X)
    Yo, sto = oracle.lut_forward(art_o, X.astype(np.float64))
    err = assert_close(Y, Yo, what)
    assert stats_list(st) == [int(v) for v in sto], what
    return err


@pytest.mark.parametrize("cfg,rows", [(1, 4096), (2, 20000)])
def test_forward_layers_c1_c2(lk, oracle, cfg, rows):
    for scheme in (0, 1):
        contract = (0, 0) if cfg == 1 else (1, 0)
        for layer in (0, 1):
            spec = oracle.recipe_layer(cfg, layer)
            art = oracle.compile_layer(spec, 64, scheme, 1, 0, *contract)
            X = oracle.recipe_inputs(cfg, 0, rows) if layer == 0 else hidden_inputs(cfg, layer, rows, spec.in_dim)
            _layer_parity(lk, oracle, art, X, f"C{cfg} layer {layer} scheme {scheme}")


@pytest.mark.parametrize("L", [16, 32, 64, 128])
@pytest.mark.parametrize("scheme", [0, 1])
def test_forward_c3_cells(lk, oracle, L, scheme):
    """All 32 cells of C3's resolution x quantization x OOB sweep (layer 0, 64->64)."""
    spec = oracle.recipe_layer(3, 0)
    X = oracle.recipe_inputs(3, 0, 4096)
    for bm in (0, 1):
        for op in (0, 1):
            art = oracle.compile_layer(spec, L, scheme, 1, 0, bm, op)
            _layer_parity(lk, oracle, art, X, f"C3 L{L} s{scheme} bm{bm} op{op}")


def test_forward_phi_and_float_table(lk, oracle):
    spec = oracle.recipe_layer(2, 0)
    X = oracle.recipe_inputs(2, 0, 3000)
    for op in (0, 1):
        art = oracle.compile_layer(spec, 32, 1, 0, 0, 0, op)
        _layer_parity(lk, oracle, art, X, f"phi op{op}")
        art = oracle.compile_layer(spec, 32, 0, 1, 0, 0, op, keep_float=True)
        _layer_parity(lk, oracle, art, X, f"float_table op{op}")


def test_forward_c4_layer_rows(lk, oracle):
    spec = oracle.recipe_layer(4, 0)
    art = oracle.compile_layer(spec, 64, 0, 1, 0, 0, 0)
    X = oracle.recipe_inputs(4, 0, 48)
    _layer_parity(lk, oracle, art, X, "C4 layer 0")
    spec = oracle.recipe_layer(4, 2)   # 1024 -> 10
    art = oracle.compile_layer(spec, 64, 0, 1, 0, 0, 0)
    _layer_parity(lk, oracle, art, hidden_inputs(4, 2, 512, 1024), "C4 layer 2")


def test_forward_c5_column_shard(lk, oracle):
    """C5 contract (L=128 uint8 asym, closed, zero_spline, d=4096): a column shard."""
    cols = (0, 48)
    spec = lk.recipe_layer(5, 0, *cols)
    art = oracle.compile_layer(to_oracle_spec(spec), 128, 1, 1, 0, 1, 1)
    X = lk.recipe_inputs(5, 0, 24)
    _layer_parity(lk, oracle, art, X, "C5 shard")


def test_chain_argmax_c2(lk, oracle):
    """C2 end to end: argmax classes of the GPU chain vs the f64 oracle chain."""
    rows = 50000
    X = oracle.recipe_inputs(2, 0, rows)
    for scheme in (0, 1):
        chain_o = [oracle.compile_layer(oracle.recipe_layer(2, l), 64, scheme, 1, 0, 1, 0) for l in range(2)]
        r = lk.lut_model_forward_batch([to_product_artifact(lk, a) for a in chain_o], X)
        Yo, sto = oracle.lut_model_forward(chain_o, X.astype(np.float64))
        agree = np.argmax(r.Y, 1) == np.argmax(Yo, 1)
        # any disagreement must be a near-tie of the two logits
        gap = np.abs(Yo[:, 0] - Yo[:, 1])
        assert np.all(agree | (gap < 1e-4)), (np.sum(~agree), gap[~agree].max())
        assert [stats_list(s) for s in r.per_layer] == sto.astype(int).tolist()
        # layer 2 per layer on the GPU's own hidden values
        chain = [to_product_artifact(lk, a) for a in chain_o]
        H, _ = lk.lut_layer_forward_batch(chain[0], X[:5000])
        Y2o, _ = oracle.lut_forward(chain_o[1], H.astype(np.float64))
        assert_close(r.Y[:5000], Y2o, "C2 layer 2")


def test_chain_fused_epilogue(tmp_path):
    """The epilogue-fused chain (LKG_FUSE=1: layer 2 evaluated in layer 1's epilogue, off by
    default) gives the unfused chain's outputs and stats, in a fresh process."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = (
        "import sys, numpy as np; sys.path[:0] = [%r, %r]\n"
        "import paper_2601_03332_b200 as lk\n"
        "X = lk.recipe_inputs(2, 0, 20000)\n"
        "for s in (0, 1):\n"
        "    ch = lk.compile_model([lk.recipe_layer(2, l) for l in range(2)], lk.QuantConfig(64, lk.Scheme(s), lk.Dtype(s)),"
        " lk.OobConfig())\n"
        "    r = lk.lut_model_forward_batch(ch, X)\n"
        "    np.save(%r + '/y%%d.npy' %% s, r.Y); np.save(%r + '/s%%d.npy' %% s, np.array([[x.n_oob_samples, x.n_oob_inputs]"
        " for x in r.per_layer]))\n") % (os.path.dirname(here), here, str(tmp_path), str(tmp_path))
    outs = {}
    for fuse in ("0", "1"):
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LKG_FUSE=fuse), check=True)
        outs[fuse] = [(np.load(tmp_path / f"y{s}.npy"), np.load(tmp_path / f"s{s}.npy")) for s in (0, 1)]
    for (y0, s0), (y1, s1) in zip(outs["0"], outs["1"]):
        assert np.array_equal(s0, s1)
        assert np.max(np.abs(y0 - y1)) <= 1e-6


def test_chain_c1(lk, oracle):
    X = oracle.recipe_inputs(1, 0, 4096)
    chain_o = [oracle.compile_layer(oracle.recipe_layer(1, l), 64, 0, 1, 0, 0, 0) for l in range(2)]
    chain = [to_product_artifact(lk, a) for a in chain_o]
    r = lk.lut_model_forward_batch(chain, X)
    # per-layer parity on the GPU's own hidden activations
    H, _ = lk.lut_layer_forward_batch(chain[0], X)
    _layer_parity(lk, oracle, chain_o[1], H, "C1 layer 1 on GPU hidden")
    Y2, _ = lk.lut_layer_forward_batch(chain[1], H)
    assert np.array_equal(r.Y, Y2)


def test_input_split_items(lk, oracle, tmp_path):
    """f64-accumulating layers with too few (row tile, j-block) items to fill the SMs split each
    item's inputs S ways (split-K): a split writes its f64 sums to a plane, a reduce kernel adds the
    planes in f64 in split order and rounds once. Forced S = 2, 4, 8 (LKG_KSPLIT) against S = 1:
    identical OobStats (OOB rows counted once through row flags) and the same outputs up to f64
    reassociation before the one f32 rounding (at most a stray last-bit difference); repeat launches
    bit-identical; the automatic choice against the reference."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = (
        "import sys, numpy as np, torch; sys.path[:0] = [%r, %r]\n"
        "import paper_2601_03332_b200 as lk\n"
        "for t, (d, m, rows, s) in enumerate(((1024, 512, 2048, 0), (256, 64, 1000, 1), (512, 48, 3000, 0))):\n"
        "    a = lk.compile_layer(lk.gen_layer(40 + t, d, m, 8), lk.QuantConfig(64, lk.Scheme(s), lk.Dtype(s)),"
        " lk.OobConfig(lk.BoundaryMode.Closed, lk.OobPolicy(s)))\n"
        "    X = torch.from_numpy(np.random.default_rng(t).uniform(-1.3, 1.3, (rows, d)).astype(np.float32)).cuda()\n"
        "    Y, st = lk.lut_layer_forward_batch(a, X)\n"
        "    Y2, st2 = lk.lut_layer_forward_batch(a, X)\n"
        "    assert torch.equal(Y, Y2) and st.n_oob_samples == st2.n_oob_samples\n"
        "    np.save(%r + '/y%%d.npy' %% t, Y.cpu().numpy())\n"
        "    np.save(%r + '/s%%d.npy' %% t, np.array([st.n_oob_samples, st.n_oob_inputs, st.n_samples, st.n_inputs]))\n"
    ) % (os.path.dirname(here), here, str(tmp_path), str(tmp_path))
    outs = {}
    for S in ("1", "2", "4", "8"):
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LKG_KSPLIT=S), check=True)
        outs[S] = [(np.load(tmp_path / f"y{t}.npy"), np.load(tmp_path / f"s{t}.npy")) for t in range(3)]
    for S in ("2", "4", "8"):
        for (y1, s1), (yS, sS) in zip(outs["1"], outs[S]):
            assert np.array_equal(s1, sS)
            diff = y1 != yS
            assert np.count_nonzero(diff) <= 2 and np.all(np.abs(y1 - yS) <= 1.2e-7 * np.maximum(1.0, np.abs(y1)))
    # the automatic choice (64 items on 148 SMs: split) against the reference
    so = oracle.gen_layer(40, 1024, 512, 8)
    art = oracle.compile_layer(so, 64, 0, 1, 0, 1, 0)
    X = np.random.default_rng(0).uniform(-1.3, 1.3, (2048, 1024)).astype(np.float32)
    _layer_parity(lk, oracle, art, X, "split-K 1024->512")


def test_workspace_report_and_trim(lk):
    """The context reports the device workspace it keeps between calls (hidden activations, the
    coordinate-record buffer of the wide-layer walk) and frees it on request; it regrows on demand."""
    eng = lk.Engine(0)
    chain = lk.compile_model([lk.recipe_layer(3, l) for l in range(2)], lk.QuantConfig(64), lk.OobConfig(), engine=eng)
    X = lk.recipe_inputs(3, 0, 3000)
    assert eng.workspace_bytes == 0
    r0 = lk.lut_model_forward_batch(chain, X, engine=eng)
    # records + silu of the 64 -> 64 layer (2 x rows x 64 x 4 B) and the two hidden buffers (+ host staging)
    assert eng.workspace_bytes >= 2 * 3000 * 64 * 4 + 2 * 3000 * 64 * 4
    eng.trim()
    assert eng.workspace_bytes == 0
    r1 = lk.lut_model_forward_batch(chain, X, engine=eng)
    assert np.array_equal(r0.Y, r1.Y)


def test_gc_pair_entries_bit_identical(tmp_path):
    """Codes-in-global layers on the integer-lerp walk can store pair entries (one 256-bit load per
    (row, input), chosen for tiles beyond L1: configs[4]); forced here (LKG_GCPAIR=1) on the C3 L=128
    layer in both schemes: the same output bits and OobStats as the code lines (LKG_GCPAIR=0), and the
    reference-layout q_table rebuilt from the pair entries byte for byte (tiles-only download)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = (
        "import sys, numpy as np; sys.path[:0] = [%r, %r]\n"
        "import paper_2601_03332_b200 as lk\n"
        "X = lk.recipe_inputs(3, 0, 3001)\n"
        "for s in (0, 1):\n"
        "    a = lk.compile_layer(lk.recipe_layer(3, 0), lk.QuantConfig(128, lk.Scheme(s), lk.Dtype(s)),"
        " lk.OobConfig(lk.BoundaryMode.Closed, lk.OobPolicy(s)))\n"
        "    Y, st = lk.lut_layer_forward_batch(a, X)\n"
        "    np.save(%r + '/y%%d.npy' %% s, Y); np.save(%r + '/q%%d.npy' %% s, a.q_table)\n"
        "    np.save(%r + '/s%%d.npy' %% s, np.array([st.n_oob_samples, st.n_oob_inputs]))\n"
    ) % (os.path.dirname(here), here, str(tmp_path), str(tmp_path), str(tmp_path))
    outs = {}
    for pair in ("1", "0"):
        subprocess.run([sys.executable, "-c", code], check=True,
                       env=dict(os.environ, LKG_GCPAIR=pair, LKG_TILE_ONLY_BYTES="0"))
        outs[pair] = [[np.load(tmp_path / f"{n}{s}.npy") for n in "yqs"] for s in (0, 1)]
    for s in (0, 1):
        for a, b in zip(outs["1"][s], outs["0"][s]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("dims,rows,scheme,bm,op", [((2, 5, 1), 4096, 0, 0, 0), ((7, 8, 3, 2), 4097, 1, 1, 1),
                                                    ((30, 4, 8, 4, 1), 63, 0, 1, 0), ((2, 5, 1), 1, 0, 0, 1),
                                                    ((12, 6, 2), 400_000, 1, 0, 0)])
def test_fused_small_chain(lk, oracle, dims, rows, scheme, bm, op):
    """Chains whose every layer is a small value-table layer run as ONE launch (forward_chain.cu,
    SURVEY §8f rank 3; the reference chain runtime.cpp:298-314): outputs and per-layer OobStats are
    bit-identical to the layer-by-layer launches, the last layer is within the bar of the reference
    on the GPU's own hidden values, and a non-finite hidden or input value raises NonFiniteError."""
    eng = lk.Engine(0)
    specs_o = [oracle.gen_layer(100 + l + sum(dims), dims[l], dims[l + 1], 5 + l) for l in range(len(dims) - 1)]
    Ls = 64 if dims[0] == 2 else 16   # (all the value tables must fit shared memory together)
    chain_o = [oracle.compile_layer(s, Ls, scheme, 1, 0, bm, op) for s in specs_o]
    chain = [to_product_artifact(lk, a) for a in chain_o]
    X = np.random.default_rng(rows).uniform(-1.3, 1.3, (rows, dims[0])).astype(np.float32)
    lk.lut_model_forward_batch(chain, X[:1], engine=eng)        # (uploads the artifacts)
    n0 = eng.launch_count
    r = lk.lut_model_forward_batch(chain, X, engine=eng)
    assert eng.launch_count - n0 == 1                          # one kernel for the whole chain
    H, per_layer = X, []
    for l, a in enumerate(chain):                              # layer by layer: never fused
        Hn, st = lk.lut_layer_forward_batch(a, H, engine=eng)
        per_layer.append(stats_list(st))
        if l == len(chain) - 1:
            Yo, _ = oracle.lut_forward(chain_o[l], H.astype(np.float64))
            assert_close(r.Y, Yo, f"fused chain {dims} last layer")
        H = Hn
    assert np.array_equal(r.Y, H)
    assert [stats_list(s) for s in r.per_layer] == per_layer
    Xn = X.copy()
    Xn[rows // 2, 0] = np.nan
    with pytest.raises(lk.NonFiniteError):
        lk.lut_model_forward_batch(chain, Xn, engine=eng)


# ------------------------------------------------------------------ spline
@pytest.mark.parametrize("cfg,layer,rows", [(1, 0, 4096), (2, 0, 4000), (3, 0, 2000), (4, 2, 256)])
def test_spline_forward(lk, oracle, cfg, layer, rows):
    spec = lk.recipe_layer(cfg, layer)
    X = oracle.recipe_inputs(cfg, 0, rows) if layer == 0 else hidden_inputs(cfg, layer, rows, spec.in_dim, -2.5, 2.5)
    Y = lk.layer_forward_batch(spec, X)
    Yo = oracle.spline_forward(to_oracle_spec(spec), X.astype(np.float64))
    assert_close(Y, Yo, f"spline C{cfg}")


def _spline_edge_inputs(spec, rows, seed):
    """Uniform draws plus every extended knot, its fp32 neighbours and far-outside values."""
    bp = np.asarray(spec.grid.breakpoints, np.float64)
    p, hl, hr = spec.grid.degree, bp[1] - bp[0], bp[-1] - bp[-2]
    ext = np.concatenate([bp[0] - hl * np.arange(p, 0, -1), bp, bp[-1] + hr * np.arange(1, p + 1)]).astype(np.float32)
    special = np.concatenate([ext, np.nextafter(ext, np.float32(-np.inf)), np.nextafter(ext, np.float32(np.inf)),
                              np.float32([0.0, -0.0, 1e3, -1e3, 20.0, -20.0])])
    rng = np.random.default_rng(seed)
    X = rng.uniform(ext[0] - hl, ext[-1] + hr, size=(rows, spec.in_dim)).astype(np.float32)
    X.ravel()[: special.size * 7 : 7] = np.resize(special, X.ravel()[: special.size * 7 : 7].size)
    return X


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_spline_forward_knot_edges(lk, oracle, cfg):
    """Tiled uniform-cubic path at every extended knot and outside the domain (basis 0, silu kept)."""
    spec = lk.recipe_layer(cfg, 0)
    X = _spline_edge_inputs(spec, 3000, 50 + cfg)
    Y = lk.layer_forward_batch(spec, X)
    Yo = oracle.spline_forward(to_oracle_spec(spec), X.astype(np.float64))
    assert_close(Y, Yo, f"spline edges C{cfg}")


@pytest.mark.parametrize("kind", ["nonuniform", "degree2", "degree5"])
def test_spline_forward_generic(lk, oracle, kind):
    """Grids outside the tiled kernel's domain (non-uniform knots, degree != 3): generic kernel."""
    import dataclasses
    base = lk.recipe_layer(1, 0)
    rng = np.random.default_rng(7)
    bp = np.asarray(base.grid.breakpoints, np.float64).copy()
    deg = {"nonuniform": 3, "degree2": 2, "degree5": 5}[kind]
    if kind == "nonuniform":
        bp[1:-1] += rng.uniform(-0.3, 0.3, bp.size - 2) * (bp[1] - bp[0])
    E, R = base.in_dim * base.out_dim, bp.size - 1 + deg
    spec = dataclasses.replace(base, grid=lk.KnotGrid(bp, deg), coeffs=rng.normal(0, 0.5, (E, R)), _dev={})
    X = _spline_edge_inputs(spec, 2000, 60 + deg)
    Y = lk.layer_forward_batch(spec, X)
    Yo = oracle.spline_forward(to_oracle_spec(spec), X.astype(np.float64))
    assert_close(Y, Yo, f"spline {kind}")


# ------------------------------------------------------------------ eval_accuracy (§8f)
def _eval_match(r, ro, what):
    """Counts and fractions exact; maxima to f64 rounding; means to summation order."""
    for k in ("n_inrange_evals", "n_oob_evals", "n_boundary_evals"):
        assert getattr(r, k) == ro[k], (what, k, getattr(r, k), ro[k])
    assert r.oob_any_frac == ro["oob_any_frac"], what
    assert (r.mae_oob is None) == (ro["mae_oob"] is None), what
    pairs = [(r.maxabs_inrange, ro["maxabs_inrange"]), (r.mae_inrange, ro["mae_inrange"])]
    if ro["mae_oob"] is not None:
        pairs += [(r.maxabs_oob, ro["maxabs_oob"]), (r.mae_oob, ro["mae_oob"])]
    for g, o in pairs:
        assert abs(g - o) <= 1e-15 + 1e-9 * abs(o), (what, g, o)
    m = r.memory
    assert [m.q_table_bytes, m.scale_bytes, m.y_min_bytes, m.knots_bytes, m.edge_scalar_bytes, m.total_bytes,
            m.float_model_bytes] == [ro[k] for k in ("q_table_bytes", "scale_bytes", "y_min_bytes", "knots_bytes",
                                                     "edge_scalar_bytes", "total_bytes", "float_model_bytes")], what
    assert m.overhead_ratio == ro["overhead_ratio"], what


@pytest.mark.parametrize("cfg,L,scheme,bm,op,vr,pd,rows", [
    (1, 64, 0, 0, 0, 1, 0, 4096), (1, 16, 1, 1, 1, 1, 0, 4096), (1, 64, 0, 1, 0, 0, 0, 4096),
    (2, 64, 0, 1, 0, 1, 0, 3000), (2, 64, 1, 1, 0, 1, 1, 3000),
    (3, 16, 0, 1, 0, 1, 0, 2000), (3, 128, 1, 0, 1, 1, 0, 2000), (3, 32, 1, 1, 1, 0, 1, 2000)])
def test_eval_accuracy_gpu(lk, oracle, cfg, L, scheme, bm, op, vr, pd, rows):
    """GPU eval_accuracy (csrc/eval.cu) vs the reference's metrics.cpp:30-103 on the same inputs
    (C3 inputs include exact knot values: boundary bucket under closed mode)."""
    spec = lk.recipe_layer(cfg, 0)
    so = to_oracle_spec(spec)
    ao = oracle.compile_layer(so, L, scheme, vr, pd, bm, op)
    X = oracle.recipe_inputs(cfg, 0, rows)
    r = lk.eval_accuracy(spec, to_product_artifact(lk, ao), X)
    ro = oracle.eval_accuracy(so, ao, X.astype(np.float64), nthreads=8)
    _eval_match(r, ro, f"eval C{cfg} L{L} s{scheme} bm{bm} op{op} vr{vr} pd{pd}")
    assert r.n_samples == rows and r.quant.samples_per_segment == L


def test_eval_accuracy_gpu_float_table_and_errors(lk, oracle):
    """Debug float_table artifacts (fetch_cell reads the f64 table), hidden-layer inputs,
    shape mismatch (DimensionError) and non-finite inputs (NonFiniteError)."""
    spec = lk.recipe_layer(2, 1)
    so = to_oracle_spec(spec)
    ao = oracle.compile_layer(so, 32, 0, 1, 0, 1, 1, keep_float=True)
    X = hidden_inputs(2, 1, 5000, spec.in_dim, -1.6, 1.6)
    _eval_match(lk.eval_accuracy(spec, to_product_artifact(lk, ao), X),
                oracle.eval_accuracy(so, ao, X.astype(np.float64), nthreads=8), "float_table")
    a = to_product_artifact(lk, ao)
    with pytest.raises(lk.DimensionError):
        lk.eval_accuracy(lk.recipe_layer(2, 0), a, X)
    X[3, 2] = np.nan
    with pytest.raises(lk.NonFiniteError):
        lk.eval_accuracy(spec, a, X)
    r = lk.eval_accuracy(spec, a, X[:0])
    assert r.n_samples == 0 and r.n_inrange_evals == 0 and r.mae_oob is None


# ------------------------------------------------------------------ KATs / errors
def _hand(lk, bm, op):
    h = hand_artifact_arrays(bm, op)
    return lk.LutLayerArtifact(1, 1, 4, lk.ValueRepr.Phi, lk.Scheme.Asymmetric, lk.Dtype.Uint8, lk.ParamDtype.F32,
                               lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op)), "",
                               knots=h["knots"], q_table=h["q"], scale=h["scale"], y_min=h["y_min"])


def test_kat_hand_table_gpu(lk):
    a = _hand(lk, 1, 0)
    xs = np.array([[x] for x, _, _ in HAND_CLOSED_CLIPX], np.float32)
    Y, st = lk.lut_layer_forward_batch(a, xs)
    assert np.allclose(Y[:, 0], [v for _, v, _ in HAND_CLOSED_CLIPX], rtol=1e-6, atol=0)
    assert st.n_oob_inputs == sum(o for _, _, o in HAND_CLOSED_CLIPX)
    Y, _ = lk.lut_layer_forward_batch(a, np.array([[0.0], [1.0], [2.0]], np.float32))
    assert Y[:, 0].tolist() == [0.0, 40.0, 70.0]    # segment starts are exact
    a = _hand(lk, 1, 1)
    Y, _ = lk.lut_layer_forward_batch(a, np.array([[x] for x, _, _ in HAND_CLOSED_ZS], np.float32))
    assert Y[:, 0].tolist() == [v for _, v, _ in HAND_CLOSED_ZS]
    a = _hand(lk, 0, 1)    # half_open masks the top knot
    Y, st = lk.lut_layer_forward_batch(a, np.array([[2.0], [1.9999]], np.float32))
    assert Y[0, 0] == 0.0 and st.n_oob_inputs == 1


def test_oob_stats_gpu(lk, oracle):
    spec = oracle.recipe_layer(1, 0)
    art = oracle.compile_layer(spec, 8, 0, 1, 0, 0, 0)
    a = to_product_artifact(lk, art)
    tK = float(spec.breakpoints[-1])
    X = np.array([[0.0, 0.0], [tK, 0.0], [tK, tK + 5.0]], np.float32)
    _, st = lk.lut_layer_forward_batch(a, X)
    assert stats_list(st) == [3, 2, 6, 3]
    assert st.oob_any_frac() == pytest.approx(2 / 3)


def test_errors_and_edges_gpu(lk, oracle):
    a = _hand(lk, 1, 0)
    with pytest.raises(lk.NonFiniteError):
        lk.lut_layer_forward_batch(a, np.array([[np.nan]], np.float32))
    with pytest.raises(lk.NonFiniteError):
        lk.lut_layer_forward_batch(a, np.array([[0.5], [-np.inf]], np.float32))
    Y, st = lk.lut_layer_forward_batch(a, np.array([[0.5]], np.float32))   # context recovers after an error
    assert Y[0, 0] == pytest.approx(15.0)
    with pytest.raises(lk.DimensionError):
        lk.lut_layer_forward_batch(a, np.zeros((2, 3), np.float32))
    with pytest.raises(lk.ConfigError):
        lk.lut_model_forward_batch([], np.zeros((1, 1), np.float32))
    spec = oracle.recipe_layer(1, 0)
    art = to_product_artifact(lk, oracle.compile_layer(spec, 8, 0, 1, 0, 0, 0))
    with pytest.raises(lk.DimensionError):
        lk.lut_model_forward_batch([art, art], np.zeros((1, 2), np.float32))
    Y, st = lk.lut_layer_forward_batch(art, np.zeros((0, 2), np.float32))     # empty batch
    assert Y.shape == (0, 5) and stats_list(st) == [0, 0, 0, 0]
    bad = _hand(lk, 1, 0)
    bad.dtype = lk.Dtype.Int8       # asymmetric requires uint8 (runtime.cpp:21-22)
    with pytest.raises(lk.ConfigError):
        bad.finalize()
    bad = _hand(lk, 1, 0)
    bad.knots = np.array([0, 2, 1], np.float32)
    with pytest.raises(lk.ConfigError):
        bad.finalize()
    bad = _hand(lk, 1, 0)
    bad.scale = np.ones(3, np.float32)
    with pytest.raises(lk.DimensionError):
        bad.finalize()
    s = lk.recipe_layer(1, 0)
    s.base_kind = "tanh"
    with pytest.raises(lk.UnsupportedBaseError):
        lk.layer_forward_batch(s, np.zeros((1, 2), np.float32))
    with pytest.raises(lk.ConfigError):
        lk.compile_layer(lk.recipe_layer(1, 0), lk.QuantConfig(1))


# ------------------------------------------------------------------ edge cases / maximum sizes
def _special_values(knots):
    k = np.asarray(knots, np.float32)
    lo, hi = k[0], k[-1]
    inf, ninf = np.float32(np.inf), np.float32(-np.inf)
    vals = [0.0, -0.0, 1e-40, -1e-40, 1e-38, 1e30, -1e30, lo, hi,
            np.nextafter(lo, ninf), np.nextafter(lo, inf), np.nextafter(hi, ninf), np.nextafter(hi, inf)]
    vals += list(k) + list(np.nextafter(k, inf)) + list(np.nextafter(k, ninf))
    return np.array(vals, np.float32)


@pytest.mark.parametrize("cfg,layer,scheme", [(2, 0, 0), (2, 1, 1), (3, 0, 1), (4, 2, 0)])
@pytest.mark.parametrize("bm,op", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_forward_special_values_ragged_rows(lk, oracle, cfg, layer, scheme, bm, op):
    """Every knot ±1 ulp, t_0/t_K and their neighbours, ±0, subnormals, ±1e30, ±3e38, scattered
    through ragged row counts (1, 31, 33, 1025, 2049: partial warps, tiles and row tiles), all
    four boundary/OOB contracts, tiled (m=16/64/1024) and small (m=2/10) layouts."""
    spec = oracle.recipe_layer(cfg, layer)
    art = oracle.compile_layer(spec, 32, scheme, 1, 0, bm, op)
    sv = _special_values(art.knots)
    rng = np.random.default_rng(cfg * 100 + layer * 10 + bm * 2 + op)
    for rows in (1, 31, 33, 1025, 2049):
        X = rng.uniform(-1.6, 1.6, (rows, spec.in_dim)).astype(np.float32)
        pos = rng.choice(X.size, size=min(X.size, 3 * sv.size), replace=False)
        X.ravel()[pos] = np.resize(sv, pos.size)
        _layer_parity(lk, oracle, art, X, f"C{cfg} l{layer} s{scheme} bm{bm} op{op} rows{rows}")


def test_empty_and_single_row_everywhere(lk, oracle):
    """rows = 0 and rows = 1 through every entry point (forward, chain, spline, eval, coords)."""
    chain_o = [oracle.compile_layer(oracle.recipe_layer(2, l), 64, 0, 1, 0, 1, 0) for l in range(2)]
    chain = [to_product_artifact(lk, a) for a in chain_o]
    spec = lk.recipe_layer(2, 0)
    for rows in (0, 1):
        X = oracle.recipe_inputs(2, 0, max(rows, 1))[:rows]
        Y, st = lk.lut_layer_forward_batch(chain[0], X)
        assert Y.shape == (rows, 16) and st.n_samples == rows and st.n_inputs == rows * 78
        r = lk.lut_model_forward_batch(chain, X)
        assert r.Y.shape == (rows, 2) and len(r.per_layer) == 2
        assert lk.layer_forward_batch(spec, X).shape == (rows, 16)
        rep = lk.eval_accuracy(spec, chain[0], X)
        assert rep.n_samples == rows
        if rows:
            Yo, sto = oracle.lut_model_forward(chain_o, X.astype(np.float64))
            assert_close(r.Y, Yo, "single-row chain")
            assert [stats_list(s) for s in r.per_layer] == sto.astype(int).tolist()


def test_forward_c5_full_layer_row_subsample(lk, oracle):
    """Maximum size: the whole C5 layer 0 (4096 x 4096 edges, K=16, L=128, uint8 asym, closed,
    zero_spline: 68.7 GB of codes, stored tiles-only) compiled and evaluated on one GPU; 48 rows,
    checked on column slices against the reference compiled on exactly those edges."""
    spec = lk.recipe_layer(5, 0)
    g = lk.compile_layer(spec, lk.QuantConfig(128, lk.Scheme.Asymmetric, lk.Dtype.Uint8),
                         lk.OobConfig(lk.BoundaryMode.Closed, lk.OobPolicy.ZeroSpline))
    X = lk.recipe_inputs(5, 0, 48)
    Y, st = lk.lut_layer_forward_batch(g, X)
    del g
    for c0, c1 in ((0, 8), (2044, 2052), (4088, 4096)):
        so = to_oracle_spec(lk.recipe_layer(5, 0, c0, c1))
        ao = oracle.compile_layer(so, 128, 1, 1, 0, 1, 1)
        Yo, sto = oracle.lut_forward(ao, X.astype(np.float64), nthreads=8)
        assert_close(Y[:, c0:c1], Yo, f"C5 full layer cols {c0}:{c1}")
        assert stats_list(st) == [int(v) for v in sto]  # OOB stats count inputs, not edges


# ------------------------------------------------------------------ element primitives (§8a)
def _adversarial_x(knots, L, rng, n=3000):
    k64 = np.asarray(knots, np.float64)
    nodes = (k64[:-1, None] + np.arange(L)[None, :] / (L - 1) * np.diff(k64)[:, None]).ravel()
    xs = [k64, nodes, np.nextafter(k64, np.inf), np.nextafter(k64, -np.inf),
          np.nextafter(nodes, np.inf), np.nextafter(nodes, -np.inf),
          rng.uniform(k64[0] - 1, k64[-1] + 1, n), [0.0, -0.0, 1e300, -1e300, 5e-324]]
    return np.concatenate([np.asarray(v, np.float64) for v in xs])


@pytest.mark.parametrize("bm,op,scheme,vr", [(0, 0, 0, 1), (1, 1, 1, 1), (1, 0, 1, 0), (0, 1, 0, 0)])
def test_element_primitives_lut(lk, oracle, bm, op, scheme, vr):
    """lut_coords (safe_clip / segment_index / interp_coords / in_range), lut_eval_value and
    lut_eval_phi on the device equal the reference's scalar functions (f64 inputs, including
    every sample node and knot ±1 ulp): coordinates and values bit-exact, phi to exp() ulps."""
    ao = oracle.compile_layer(oracle.recipe_layer(1, 0), 16, scheme, vr, 0, bm, op)
    a = to_product_artifact(lk, ao)
    rng = np.random.default_rng(bm * 4 + op)
    x = _adversarial_x(ao.knots, 16, rng)
    c = lk.lut_coords(a, x)
    co = oracle.coords(ao, x)
    for key in ("in_range", "x_clip", "k", "l0", "l1", "w"):
        assert np.array_equal(c[key], co[key]), key
    E = ao.in_dim * ao.out_dim
    e = rng.integers(0, E, x.size).astype(np.int32)
    v, oob = lk.lut_eval_value(a, e, x)
    phi = lk.lut_eval_phi(a, e, x)
    for t in range(0, x.size, 7):
        vo, oo = oracle.eval_value(ao, int(e[t]), float(x[t]))
        assert v[t] == vo and oob[t] == oo, t
        po = oracle.eval_phi(ao, int(e[t]), float(x[t]))
        assert abs(phi[t] - po) <= 4e-16 * max(1.0, abs(po)), (t, phi[t], po)
    with pytest.raises(lk.NonFiniteError):
        lk.lut_eval_phi(a, 0, np.nan)
    with pytest.raises(lk.DimensionError):
        lk.lut_eval_value(a, E, 0.5)


def test_element_primitives_spline_and_quantize(lk, oracle):
    """basis_values, eval_spline, eval_edge_phi, sample_segment_points and
    quantize_segment_symmetric / _asymmetric on the device equal the reference's."""
    rng = np.random.default_rng(9)
    spec = lk.recipe_layer(3, 0)
    so = to_oracle_spec(spec)
    for bp, deg in ((spec.grid.breakpoints, 3), (np.cumsum(rng.uniform(0.1, 1, 7)) - 2, 2),
                    (np.cumsum(rng.uniform(0.1, 1, 5)) - 1, 5)):
        grid = lk.KnotGrid(np.asarray(bp, np.float64), deg)
        x = _adversarial_x(bp, 8, rng, 500)
        B = lk.basis_values(grid, x)
        for t in range(0, x.size, 5):
            assert np.array_equal(B[t], oracle.basis_values(bp, deg, float(x[t]))), t
    x = _adversarial_x(spec.grid.breakpoints, 8, rng, 2000)
    E = spec.in_dim * spec.out_dim
    e = rng.integers(0, E, x.size).astype(np.int32)
    phi = lk.eval_edge_phi(spec, e, x)
    R = spec.grid.K + spec.grid.degree
    coeffs = np.asarray(so.coeffs, np.float64).reshape(E, R)
    for t in range(0, x.size, 11):
        b = oracle.basis_values(spec.grid.breakpoints, 3, float(x[t]))
        sp = 0.0
        for r in range(R):
            sp += float(coeffs[e[t], r]) * b[r]
        ref = so.out_scale[e[t]] * (so.base_scale[e[t]] * (x[t] / (1.0 + np.exp(-x[t]))) + so.spline_scale[e[t]] * sp)
        assert abs(phi[t] - ref) <= 4e-16 * max(1.0, abs(ref)), (t, phi[t], ref)
        assert lk.eval_spline(spec.grid, spec.coeffs[e[t]], float(x[t])) == sp
    for k in range(spec.grid.K):
        pts = lk.sample_segment_points(spec.grid.breakpoints, k, 64)
        step = (spec.grid.breakpoints[k + 1] - spec.grid.breakpoints[k]) / 64.0
        assert np.array_equal(pts, [spec.grid.breakpoints[k] + l * step for l in range(64)])
    for trial in range(40):
        vals = rng.normal(0, rng.uniform(1e-3, 2), int(rng.integers(2, 130)))
        if trial % 5 == 0:
            vals[:] = vals[0]                      # degenerate (constant) segment
        if trial % 7 == 0:
            vals[::3] = -vals[0]                   # ties of |v| with opposite signs (amax / min / max)
        for scheme, fn in ((0, lk.quantize_segment_symmetric), (1, lk.quantize_segment_asymmetric)):
            q, s, y = fn(vals)
            qo, so_, yo = oracle.quantize_segment(vals, scheme)
            assert np.array_equal(q, qo) and s == so_ and y == yo, (trial, scheme)
    with pytest.raises(lk.NonFiniteError):
        lk.quantize_segment_symmetric([1.0, np.inf])
    with pytest.raises(lk.ConfigError):
        lk.quantize_segment_asymmetric([])


# ------------------------------------------------------------------ randomized shapes
# (LKG_FUZZ_SEEDS widens the campaign: profiles/r02g/fuzz_1000.log is a 1000-seed run)
@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("LKG_FUZZ_SEEDS", "80"))))
def test_fuzz_compile_and_forward(lk, oracle, seed):
    """Random layer shapes, grids and contracts (d, m off the 8/16 tile multiples; K up to 40;
    L from 2 to 160; uneven knots; phi and spline_component; f16 params; all boundary/OOB
    contracts; ragged rows): compile byte-identical, forward within the bar, stats exact."""
    from oracle.pyoracle import Spec
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.choice([1, 3, 7, 9, 17, 33, 70, 130, 300]))
    m = int(rng.choice([1, 2, 5, 8, 9, 15, 16, 17, 40]))
    K = int(rng.integers(1, 41))
    deg = int(rng.integers(1, 4))
    L = int(rng.choice([2, 3, 16, 33, 64, 100, 160]))
    uniform = rng.random() < 0.7
    lo, hi = sorted(rng.uniform(-3, 3, 2)) if rng.random() < 0.5 else (-1.0, 1.0)
    if hi - lo < 0.5:
        hi = lo + 0.5
    bp = np.linspace(lo, hi, K + 1) if uniform else np.cumsum(rng.uniform(0.2, 1.0, K + 1)) * (hi - lo) / (K + 1) + lo
    E, R = d * m, K + deg
    so = Spec(d, m, bp, rng.normal(0, 0.3, (E, R)), rng.uniform(-1, 1, E), rng.uniform(0.5, 1.5, E),
              rng.uniform(0.5, 1.5, E), deg)
    scheme, vr, pd = int(rng.integers(0, 2)), int(rng.random() < 0.8), int(rng.random() < 0.25)
    bm, op = int(rng.integers(0, 2)), int(rng.integers(0, 2))
    ao = oracle.compile_layer(so, L, scheme, vr, pd, bm, op)
    spec = to_product_spec(lk, so)
    qc = lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme), lk.ValueRepr(vr), lk.Interp.Linear, lk.ParamDtype(pd))
    g = lk.compile_layer(spec, qc, lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op)))
    assert _bytes_equal(g.q_table, ao.q) and _bytes_equal(g.scale, ao.scale) and _bytes_equal(g.y_min, ao.y_min)
    rows = int(rng.choice([1, 37, 1000, 2500]))
    X = rng.uniform(lo - 0.3 * (hi - lo), hi + 0.3 * (hi - lo), (rows, d)).astype(np.float32)
    X.ravel()[:: max(1, X.size // 50)] = np.asarray(ao.knots)[rng.integers(0, K + 1, X.ravel()[:: max(1, X.size // 50)].size)]
    _layer_parity(lk, oracle, ao, X, f"fuzz {seed}: d{d} m{m} K{K} deg{deg} L{L} s{scheme} vr{vr} pd{pd} bm{bm} op{op}")


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("LKG_FUZZ_SPLINE_SEEDS", "30"))))
def test_fuzz_spline_forward(lk, oracle, seed):
    """Random spline layers through layer_forward_batch (tiled kernel on uniform cubic grids,
    generic kernel otherwise) against the reference's spline forward."""
    import dataclasses
    from oracle.pyoracle import Spec
    rng = np.random.default_rng(5000 + seed)
    d = int(rng.choice([1, 5, 8, 13, 64, 300]))
    m = int(rng.choice([1, 3, 16, 17, 33]))
    K = int(rng.integers(1, 30))
    deg = 3 if rng.random() < 0.6 else int(rng.integers(0, 6))
    uniform = rng.random() < 0.7
    bp = np.linspace(-1.5, 2.0, K + 1) if uniform else np.cumsum(rng.uniform(0.1, 1.0, K + 1)) - 1.0
    E, R = d * m, K + deg
    so = Spec(d, m, bp, rng.normal(0, 0.4, (E, R)), rng.uniform(-1, 1, E), rng.uniform(0.5, 1.5, E),
              rng.uniform(0.5, 1.5, E), deg)
    spec = to_product_spec(lk, so)
    rows = int(rng.choice([1, 40, 700, 2100]))
    X = rng.uniform(bp[0] - 1.0, bp[-1] + 1.0, (rows, d)).astype(np.float32)
    Y = lk.layer_forward_batch(spec, X)
    Yo = oracle.spline_forward(so, X.astype(np.float64))
    assert_close(Y, Yo, f"spline fuzz {seed}: d{d} m{m} K{K} deg{deg} uniform{uniform}")


@pytest.mark.gpu
def test_chain_graph_replay_matches_direct(lk):
    """lkg_graph_create / _launch (CUDA-graph replay of a chain forward) == lkg_model_forward bit for
    bit, OOB statistics accumulate per replay, in-place input updates are seen by the replay."""
    import torch
    for cfg, rows in ((1, 4096), (2, 20000)):
        dims, _, _, _ = lk.recipe_dims(cfg)
        eng = lk.Engine(0)
        chain = [lk.compile_layer(lk.recipe_layer(cfg, l), lk.QuantConfig(64), lk.OobConfig(), engine=eng)
                 for l in range(len(dims) - 1)]
        X = torch.from_numpy(lk.recipe_inputs(cfg, 0, rows)).cuda()
        res = lk.lut_model_forward_batch(chain, X, engine=eng)
        Y = torch.empty((rows, dims[-1]), device="cuda")
        g = lk.ChainGraph(chain, X, Y, engine=eng)
        eng.collect(len(chain))                      # drop what creation ran
        for _ in range(3):
            g()
        eng.synchronize()
        assert torch.equal(Y, res.Y if hasattr(res.Y, "device") else torch.from_numpy(res.Y).cuda())
        st = eng.collect(len(chain))
        for s_g, s_d in zip(st, res.per_layer):
            assert s_g.n_samples == 3 * s_d.n_samples and s_g.n_oob_inputs == 3 * s_d.n_oob_inputs
            assert s_g.n_oob_samples == 3 * s_d.n_oob_samples and s_g.n_inputs == 3 * s_d.n_inputs
        X2 = torch.from_numpy(lk.recipe_inputs(cfg, rows, rows)).cuda()
        X.copy_(X2)                                   # new batch in place, same graph
        g()
        eng.synchronize()
        ref2 = lk.lut_model_forward_batch(chain, X2, engine=eng).Y
        assert torch.equal(Y, ref2 if hasattr(ref2, "device") else torch.from_numpy(ref2).cuda())
        del g
    with pytest.raises(lk.DimensionError):
        lk.ChainGraph(chain, X.cpu(), Y)


@pytest.mark.gpu
def test_chain_graph_owns_its_buffers(lk):
    """A captured graph keeps working after the same engine ran larger or wider forwards (which
    grow, i.e. free and reallocate, the engine's scratch and transposed-input buffers): the graph
    owns its own. Layer 0 (256 -> 256, 16 j-blocks, 1024-row batch) takes the XT walk,
    whose tensor map is baked into the captured launch."""
    import torch
    eng = lk.Engine(0)
    specs = [lk.gen_layer(21, 256, 256, 8), lk.gen_layer(22, 256, 4, 8)]
    chain = lk.compile_model(specs, lk.QuantConfig(64), lk.OobConfig(), engine=eng)
    X = torch.empty((1024, 256), device="cuda").uniform_(-1.2, 1.2)
    want = lk.lut_model_forward_batch(chain, X, engine=eng).Y.clone()
    Y = torch.empty((1024, 4), device="cuda")
    g = lk.ChainGraph(chain, X, Y, engine=eng)
    big = torch.empty((16384, 256), device="cuda").uniform_(-1.2, 1.2)
    wide = [lk.compile_layer(lk.gen_layer(23, 256, 1024, 8), lk.QuantConfig(64), lk.OobConfig(), engine=eng),
            lk.compile_layer(lk.gen_layer(24, 1024, 4, 8), lk.QuantConfig(64), lk.OobConfig(), engine=eng)]
    for _ in range(2):
        lk.lut_model_forward_batch(chain, big, engine=eng)   # scratch and xt grow (reallocated)
        lk.lut_model_forward_batch(wide, big, engine=eng)
        Y.zero_()
        g()
        torch.cuda.synchronize()
        assert torch.equal(Y, want)
    eng.collect(2)
    del g


@pytest.mark.gpu
def test_chain_graph_with_input_split(lk):
    """A captured chain whose wide layer splits its inputs (1024 -> 512 on 2048 rows: 64 items on 148
    SMs) replays the walk, the row-flag reset and the reduce kernel; the graph owns the planes of
    partial sums, so larger split forwards on the same engine in between do not disturb it, and the
    OobStats of each replay are the direct call's."""
    import torch
    eng = lk.Engine(0)
    chain = lk.compile_model([lk.gen_layer(31, 1024, 512, 8), lk.gen_layer(32, 512, 4, 8)], lk.QuantConfig(64),
                             lk.OobConfig(), engine=eng)
    X = torch.empty((2048, 1024), device="cuda").uniform_(-1.3, 1.3)
    ref = lk.lut_model_forward_batch(chain, X, engine=eng)
    want = ref.Y.clone()
    Y = torch.empty((2048, 4), device="cuda")
    g = lk.ChainGraph(chain, X, Y, engine=eng)
    big = torch.empty((6144, 1024), device="cuda").uniform_(-1.3, 1.3)
    for _ in range(2):
        lk.lut_model_forward_batch(chain, big, engine=eng)      # grows the engine's own planes
        Y.zero_()
        g()
        torch.cuda.synchronize()
        assert torch.equal(Y, want)
        st = eng.collect(2)
        assert [(s.n_oob_samples, s.n_oob_inputs) for s in st] == \
            [(s.n_oob_samples, s.n_oob_inputs) for s in ref.per_layer]
    del g


@pytest.mark.gpu
def test_torch_inputs_are_stream_ordered(lk):
    """A torch input still being written on torch's current stream (delayed by a long-running
    kernel) is read only after that write: the engine's private stream waits on torch's stream
    (ADVICE r1), for the LUT chain, the spline forward and graph replay."""
    import torch
    eng = lk.Engine(0)
    spec = lk.recipe_layer(3, 0)
    a = lk.compile_layer(spec, lk.QuantConfig(64), lk.OobConfig(), engine=eng)
    X2 = torch.from_numpy(lk.recipe_inputs(3, 0, 65536)).cuda()
    want = lk.lut_layer_forward_batch(a, X2, engine=eng)[0].clone()
    want_s = lk.layer_forward_batch(spec, X2, engine=eng).clone()
    X = torch.zeros_like(X2)
    for fn, ref in ((lambda: lk.lut_layer_forward_batch(a, X, engine=eng)[0], want),
                    (lambda: lk.layer_forward_batch(spec, X, engine=eng), want_s)):
        X.zero_()
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000_000)   # ~0.1 s on torch's stream before the new batch lands
        X.copy_(X2)
        Y = fn()
        assert torch.equal(Y, ref)
    Y = torch.empty((65536, 64), device="cuda")
    g = lk.ChainGraph([a], X, Y, engine=eng)
    X.zero_()
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)
    X.copy_(X2)
    out = g()
    assert torch.equal(out, want)
    eng.collect(1)
    del g


@pytest.mark.gpu
def test_balanced_rows_small_batches_bit_identical(lk, oracle):
    """One-j-block layers split any batch over every SM in 64-aligned row ranges: prefixes of a batch
    (1 .. 5000 rows, odd sizes, fewer rows than SMs x 64) reproduce the full launch bit for bit, and
    match the oracle within the north-star bar."""
    for scheme in (0, 1):
        spec = lk.recipe_layer(2, 0)
        a = lk.compile_layer(spec, lk.QuantConfig(64, lk.Scheme(scheme), lk.Dtype(scheme)), lk.OobConfig())
        X = lk.recipe_inputs(2, 0, 9471)
        Yfull, sfull = lk.lut_layer_forward_batch(a, X)
        for n in (1, 2, 63, 64, 65, 127, 1000, 5000, 9470):
            Y, st = lk.lut_layer_forward_batch(a, X[:n])
            assert np.array_equal(Y, Yfull[:n]), (scheme, n)
            assert st.n_samples == n
        so = to_oracle_spec(spec)
        ao = oracle.compile_layer(so, 64, scheme, 1, 0, 1, 0)
        Yo, cnt = oracle.lut_forward(ao, X[:3000].astype(np.float64))
        assert_close(Yfull[:3000], Yo, f"balanced rows scheme {scheme}")
        assert sfull.n_samples == 9471


@pytest.mark.gpu
def test_transposed_input_walk_bit_identical(lk, oracle):
    """Layers with many j-blocks (>= 16) take their input transposed through 2D TMA boxes when the
    batch is whole 1024-row tiles (XT mode): same bits as the row-major path (a batch one row short
    takes that path), OOB counts equal, and the oracle's outputs within the north-star bar."""
    import torch
    spec = lk.recipe_layer(4, 1)                  # 1024 -> 1024, 64 j-blocks, f64 accumulators
    a = lk.compile_layer(spec, lk.QuantConfig(64), lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX))
    g = torch.Generator().manual_seed(7)
    X = (torch.rand((2048, 1024), generator=g) * 2.6 - 1.3).numpy().astype(np.float32)
    Yt, st = lk.lut_layer_forward_batch(a, torch.from_numpy(X).cuda())       # XT
    Yr, sr = lk.lut_layer_forward_batch(a, torch.from_numpy(X[:2047]).cuda())  # row-major path
    Yt, Yr = Yt.cpu().numpy(), Yr.cpu().numpy()
    assert np.array_equal(Yt[:2047], Yr)
    assert st.n_samples == 2048 and sr.n_samples == 2047
    assert st.n_oob_inputs >= sr.n_oob_inputs and st.n_oob_inputs - sr.n_oob_inputs <= 1024
    ao = oracle.compile_layer(to_oracle_spec(spec), 64, 0, 1, 0, 0, 0)
    Yo, cnt = oracle.lut_forward(ao, X[2000:2048].astype(np.float64))
    assert_close(Yt[2000:2048], Yo, "XT walk vs oracle")


def test_transposed_input_walk_codes_in_l2_bit_identical(lk, oracle):
    """C5 geometry (L=128 uint8 asym, codes read from L2: the GC kernel) on 1024 output columns
    (>= 16 j-blocks): whole 1024-row tiles take the transposed-input (XT) walk, a batch one row short
    the row-major one; the same bits, and the oracle on a column slice within the north-star bar."""
    import torch
    spec = lk.recipe_layer(5, 0, 0, 1024)
    g = lk.compile_layer(spec, lk.QuantConfig(128, lk.Scheme.Asymmetric, lk.Dtype.Uint8),
                         lk.OobConfig(lk.BoundaryMode.Closed, lk.OobPolicy.ZeroSpline))
    X = lk.recipe_inputs(5, 0, 2048)
    Yt, st = lk.lut_layer_forward_batch(g, torch.from_numpy(X).cuda())
    Yr, sr = lk.lut_layer_forward_batch(g, torch.from_numpy(X[:2047]).cuda())
    del g
    Yt, Yr = Yt.cpu().numpy(), Yr.cpu().numpy()
    assert np.array_equal(Yt[:2047], Yr)
    assert st.n_samples == 2048 and sr.n_samples == 2047
    c0, c1 = 1016, 1024
    ao = oracle.compile_layer(to_oracle_spec(lk.recipe_layer(5, 0, c0, c1)), 128, 1, 1, 0, 1, 1)
    Yo, _ = oracle.lut_forward(ao, X[2016:2048].astype(np.float64), nthreads=8)
    assert_close(Yt[2016:2048, c0:c1], Yo, "GC XT walk vs oracle")


@pytest.mark.gpu
def test_coordinate_record_walk(lk, oracle, tmp_path):
    """Layers with >= 4 j-blocks on the integer-lerp walk take their coordinates once per input
    element from the coordinate pass (REC): bit-identical to the in-kernel coordinates where both
    read the same silu boxes (XT, f64 accumulators: a 1024 -> 1024 layer on 2048 rows), and within the
    bar against the reference on ragged shapes the pass allows (row counts not a multiple of 1024,
    input widths not a multiple of 8)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = (
        "import sys, numpy as np, torch; sys.path[:0] = [%r, %r]\n"
        "import paper_2601_03332_b200 as lk\n"
        "a = lk.compile_layer(lk.gen_layer(5, 1024, 1024, 8), lk.QuantConfig(64),"
        " lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX))\n"
        "X = torch.from_numpy(np.random.default_rng(3).uniform(-1.3, 1.3, (2048, 1024)).astype(np.float32)).cuda()\n"
        "Y, st = lk.lut_layer_forward_batch(a, X)\n"
        "np.save(%r + '/y.npy', Y.cpu().numpy()); np.save(%r + '/s.npy', np.array([st.n_oob_inputs, st.n_oob_samples]))\n"
        # an fp32-accumulating layer (C3 layer 0, 4 j-blocks): the pass takes the walk's own MUFU silu
        "b = lk.compile_layer(lk.recipe_layer(3, 0), lk.QuantConfig(64), lk.OobConfig())\n"
        "Y2, _ = lk.lut_layer_forward_batch(b, torch.from_numpy(lk.recipe_inputs(3, 0, 3000)).cuda())\n"
        "np.save(%r + '/y2.npy', Y2.cpu().numpy())\n"
    ) % (os.path.dirname(here), here, str(tmp_path), str(tmp_path), str(tmp_path))
    outs = {}
    for rec in ("1", "0"):
        subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LKG_REC=rec), check=True)
        outs[rec] = (np.load(tmp_path / "y.npy"), np.load(tmp_path / "s.npy"), np.load(tmp_path / "y2.npy"))
    assert np.array_equal(outs["1"][0], outs["0"][0]) and np.array_equal(outs["1"][1], outs["0"][1])
    assert np.array_equal(outs["1"][2], outs["0"][2])
    # ragged shapes through the pass, against the reference
    for d, m, rows, contract in ((300, 64, 777, (0, 0)), (60, 128, 1999, (1, 1)), (64, 64, 2501, (0, 1))):
        so = oracle.gen_layer(17 + d, d, m, 8)
        for scheme in (0, 1):
            art = oracle.compile_layer(so, 64, scheme, 1, 0, *contract)
            X = np.random.default_rng(d + m).uniform(-1.4, 1.4, (rows, d)).astype(np.float32)
            _layer_parity(lk, oracle, art, X, f"REC d{d} m{m} rows{rows} scheme{scheme}")
