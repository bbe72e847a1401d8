"""C-ABI checks that need no GPU: the library loads, exports every symbol the public
header declares (and the ctypes binding covers them), host-only entry points (synthetic
config recipes) agree with the oracle, host-side validation mirrors the reference error
taxonomy, and GPU calls fail loudly (no CPU fallback) on a machine without a GPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(lkg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(lk):
    from paper_2601_03332_b200 import _capi
    lib = _capi.lib()
    declared = _declared("lutkan_b200.h")
    assert len(declared) >= 25
    nm = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (lkg_\w+)", nm))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert getattr(lib, s) is not None
        assert s in _capi.SIGNATURES, f"ctypes binding lacks {s}"


def test_library_is_sm100a(lk):
    from paper_2601_03332_b200 import _capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_recipes_match_oracle(lk, oracle):
    for cfg in (1, 2, 3):
        dims, G, lo, hi = lk.recipe_dims(cfg)
        for layer in range(len(dims) - 1):
            s, o = lk.recipe_layer(cfg, layer), oracle.recipe_layer(cfg, layer)
            assert np.array_equal(s.coeffs, o.coeffs) and np.array_equal(s.base_scale, o.base_scale)
            assert np.array_equal(s.grid.breakpoints, o.breakpoints)
        assert np.array_equal(lk.recipe_inputs(cfg, 3, 40), oracle.recipe_inputs(cfg, 3, 40))
    # column shards are the matching slices of the full spec
    full = lk.recipe_layer(3, 0)
    part = lk.recipe_layer(3, 0, 10, 20)
    assert np.array_equal(part.coeffs, full.coeffs.reshape(64, 64, -1)[:, 10:20].reshape(640, -1))
    assert lk.recipe_dims(4)[0] == [1024, 1024, 1024, 10] and lk.recipe_dims(5)[0] == [4096, 4096, 4096]


def test_recipe_errors(lk):
    with pytest.raises(lk.ConfigError):
        lk.recipe_dims(9)
    with pytest.raises(lk.DimensionError):
        lk.recipe_layer(1, 5)


def test_enum_parsing_and_host_validation(lk):
    assert lk.parse_enum("boundary_mode", "half_open") == lk.BoundaryMode.HalfOpen
    with pytest.raises(lk.ConfigError):
        lk.parse_enum("oob_policy", "wrap")
    with pytest.raises(lk.ConfigError):
        lk.QuantConfig(1).validate()
    with pytest.raises(lk.ConfigError):
        lk.QuantConfig(64, lk.Scheme.Symmetric, lk.Dtype.Uint8).validate()
    a = lk.LutLayerArtifact(1, 1, 4, lk.ValueRepr.Phi, lk.Scheme.Asymmetric, lk.Dtype.Uint8, knots=np.array([0, 1, 2], np.float32),
                            q_table=np.zeros(7, np.uint8), scale=np.ones(2, np.float32), y_min=np.zeros(2, np.float32))
    with pytest.raises(lk.DimensionError):
        a._desc()
    st = lk.OobStats(3, 2, 6, 3)
    st.merge(lk.OobStats(3, 2, 6, 3))
    assert (st.n_samples, st.n_oob_inputs, st.oob_any_frac()) == (6, 6, pytest.approx(2 / 3))


def test_gpu_calls_fail_loudly_without_gpu(lk):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(lk.CudaError):
        lk.Engine(0)


def test_gen_layer_and_inputs_match_reference(port, ref):
    """gen_layer / gen_sanity_layer / gen_inputs (model_gen.cpp:7-45): the product's host
    generator equals the reference's bit for bit (and the C port)."""
    import paper_2601_03332_b200 as lk
    for seed, d, m, K, deg in ((0, 10, 8, 8, 3), (7, 3, 5, 4, 2), (123, 1, 1, 1, 0)):
        g = lk.gen_layer(seed, d, m, K, deg)
        for o in (port, ref):
            s = o.gen_layer(seed, d, m, K, deg)
            assert np.array_equal(g.grid.breakpoints, s.breakpoints)
            assert np.array_equal(g.coeffs.ravel(), np.asarray(s.coeffs).ravel())
            for a, b in ((g.base_scale, s.base_scale), (g.spline_scale, s.spline_scale), (g.out_scale, s.out_scale)):
                assert np.array_equal(a, b)
    for clip in (False, True):
        X = lk.gen_inputs(5, 100, 7, -1.2, 1.1, clip)
        for o in (port, ref):
            assert np.array_equal(X, o.gen_inputs(5, 100, 7, -1.2, 1.1, clip))
    assert lk.gen_sanity_layer(3).coeffs.shape == (80, 11)
    with pytest.raises(lk.ConfigError):
        lk.gen_inputs(1, 2, 2, 1.0, 1.0, True)
    with pytest.raises(lk.ConfigError):
        lk.gen_layer(1, 2, 2, 0, 3)


def _build_c_demo(out):
    """tests/cpp/c_abi_demo.c: plain C11 against include/lutkan_b200.h + liblutkan_b200.so."""
    lib_dir = os.path.join(ROOT, "paper_2601_03332_b200")
    cmd = ["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "c_abi_demo.c"), "-o", str(out), "-L", lib_dir, "-llutkan_b200",
           f"-Wl,-rpath,{lib_dir}", "-lm"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_c_abi_compiles_from_plain_c(tmp_path):
    """The boundary is a C ABI: a C11 program using it compiles warning-free and links."""
    _build_c_demo(tmp_path / "c_abi_demo")
    assert (tmp_path / "c_abi_demo").exists()


@pytest.mark.gpu
def test_c_abi_demo_runs_on_gpu(tmp_path):
    """Compile, forward, save, reload, forward again, from C: identical outputs."""
    exe = tmp_path / "c_abi_demo"
    _build_c_demo(exe)
    r = subprocess.run([str(exe), str(tmp_path / "demo.lut")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert "reload identical 1" in r.stdout
