"""The `.lut` artifact container (reference artifact_io.cpp:168-300,
detail/zip.cpp, docs/artifact_format.md) through the C-ABI (csrc/artifact_io.cpp).

CPU tests pin the writer and the reader's validation to reference-written fixtures
(tests/golden/make_artifacts.py) and, where oracle/_ref is built, to the live reference:
  * lkg_artifact_save_desc writes byte-identical files,
  * lkg_artifact_check returns, for every malformed archive, the reference's error class,
  * ZIP64 (extension) and stored archives are valid ZIPs (Python's zipfile reads them).
GPU tests load archives straight into device layers and compare forwards and re-saved bytes."""
import filecmp
import json
import os
import subprocess
import sys
import zipfile

import numpy as np
import pytest

from helpers import assert_close, stats_list, to_product_artifact

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "artifacts")
REC = json.load(open(os.path.join(GOLD, "artifacts.json")))


@pytest.fixture(scope="module")
def lk():
    import paper_2601_03332_b200 as m
    return m


def _compile(oracle, a):
    return oracle.compile_layer(oracle.recipe_layer(a["cfg"], a["layer"]), a["L"], a["scheme"], a["value_repr"],
                                a["param_dtype"], a["boundary_mode"], a["oob_policy"])


@pytest.mark.parametrize("arch", REC["archives"], ids=[a["file"] for a in REC["archives"]])
def test_save_bytes_equal_reference(lk, port, arch, tmp_path):
    """save_artifact of the same artifact: our file == the reference's file, byte for byte."""
    art = to_product_artifact(lk, _compile(port, arch))  # port compile == reference compile (test_oracle)
    out = tmp_path / "o.lut"
    lk.save_artifact(art, out)
    assert filecmp.cmp(out, os.path.join(GOLD, arch["file"]), shallow=False)
    lk.check_artifact(os.path.join(GOLD, arch["file"]))


@pytest.mark.parametrize("case", REC["corrupt"], ids=[c["file"] for c in REC["corrupt"]])
def test_check_matches_reference_error_class(lk, case):
    """Every malformed archive raises the reference's error class (IoError family, then
    finalize's ConfigError / NonFiniteError); reordered entries and unknown base kinds load."""
    from paper_2601_03332_b200._capi import lib
    st = lib().lkg_artifact_check(os.fsencode(os.path.join(GOLD, case["file"])))
    assert st == case["status"], (case, lib().lkg_last_error())


def test_check_error_types(lk):
    for name, exc in (("truncated", lk.CorruptArchiveError), ("crc_mismatch", lk.CorruptBlobError),
                      ("missing_L", lk.MissingKeyError), ("shape_mismatch", lk.ShapeError),
                      ("version", lk.VersionError), ("enum_scheme", lk.EnumError),
                      ("knots_unsorted", lk.ConfigError), ("knots_nan", lk.NonFiniteError)):
        with pytest.raises(exc):
            lk.check_artifact(os.path.join(GOLD, "corrupt", name + ".lut"))
    with pytest.raises(lk.IoError):
        lk.check_artifact(os.path.join(GOLD, "corrupt", "no_such_file.lut"))
    assert issubclass(lk.CorruptBlobError, lk.IoError) and issubclass(lk.IoError, lk.Error)


def test_live_reference_statuses(lk, ref, tmp_path):
    """With oracle/_ref built: the live reference agrees with the fixtures and reads our files."""
    for c in REC["corrupt"]:
        assert ref.artifact_load_status(os.path.join(GOLD, c["file"])) == c["status"], c
    for a in REC["archives"]:
        art = _compile(ref, a)
        ours = tmp_path / "ours.lut"
        lk.save_artifact(to_product_artifact(lk, art), ours, store=True)  # stored entries
        assert ref.artifact_load_status(ours, tmp_path / "re.lut") == 0
        assert filecmp.cmp(tmp_path / "re.lut", os.path.join(GOLD, a["file"]), shallow=False)


def test_zip64_and_stored_are_valid_zips(lk, port, tmp_path):
    """ZIP64 records (forced for a small layer by the LKG_ZIP64_FORCE test hook) and stored
    entries: Python's zipfile reads both and every CRC checks; our reader accepts both."""
    arch = REC["archives"][0]
    a = _compile(port, arch)
    z64, st = tmp_path / "z64.lut", tmp_path / "stored.lut"
    code = ("import sys; sys.path[:0] = [%r, %r]\n"
            "import paper_2601_03332_b200 as lk\nfrom oracle.pyoracle import Oracle\nfrom helpers import to_product_artifact\n"
            "o = Oracle('port')\n"
            "a = o.compile_layer(o.recipe_layer(%d, %d), %d, %d, %d, %d, %d, %d)\n"
            "lk.save_artifact(to_product_artifact(lk, a), %r)\n") % (
        os.path.dirname(HERE), HERE, arch["cfg"], arch["layer"], arch["L"], arch["scheme"], arch["value_repr"],
        arch["param_dtype"], arch["boundary_mode"], arch["oob_policy"], str(z64))
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LKG_ZIP64_FORCE="1"), check=True)
    lk.save_artifact(to_product_artifact(lk, a), st, store=True)
    for path in (z64, st):
        with zipfile.ZipFile(path) as z:
            assert z.testzip() is None
            assert [i.filename for i in z.infolist()][:2] == ["manifest.json", "knots.bin"]
            assert np.array_equal(np.frombuffer(z.read("q_table.bin"), np.uint8), a.q)
        lk.check_artifact(path)
    with zipfile.ZipFile(z64) as z:
        assert z.read("manifest.json") == zipfile.ZipFile(os.path.join(GOLD, arch["file"])).read("manifest.json")


# ------------------------------------------------------------------ GPU: straight to device memory
@pytest.mark.gpu
@pytest.mark.parametrize("arch", REC["archives"], ids=[a["file"] for a in REC["archives"]])
def test_load_to_device_forward_and_resave(lk, oracle, arch, tmp_path):
    """load_artifact into a device layer: its forward equals the reference forward of the same
    artifact, its host view equals the compiled arrays, and saving it again reproduces the file."""
    a_o = _compile(oracle, arch)
    dev = lk.load_artifact(os.path.join(GOLD, arch["file"]))
    assert np.array_equal(dev.q_table, a_o.q) and np.array_equal(dev.scale.view(np.uint32), a_o.scale.view(np.uint32))
    d = dev.in_dim
    X = np.random.default_rng(3).uniform(-1.4, 1.4, (3000, d)).astype(np.float32)
    Y, st = lk.lut_layer_forward_batch(dev, X)
    Yo, sto = oracle.lut_forward(a_o, X.astype(np.float64))
    assert_close(Y, Yo, arch["file"])
    assert stats_list(st) == [int(v) for v in sto]
    lk.save_artifact(dev, tmp_path / "re.lut")
    assert filecmp.cmp(tmp_path / "re.lut", os.path.join(GOLD, arch["file"]), shallow=False)


@pytest.mark.gpu
def test_compiled_device_artifact_saves_reference_bytes(lk, tmp_path, monkeypatch):
    """A GPU-compiled layer (including a tiles-only one, whose q_table is rebuilt from the tiles)
    saves the reference's bytes; loading a stored / ZIP64 archive gives the same device layer."""
    arch = REC["archives"][3]
    spec = lk.recipe_layer(arch["cfg"], arch["layer"])
    qc = lk.QuantConfig(arch["L"], lk.Scheme(arch["scheme"]), lk.Dtype(arch["scheme"]), lk.ValueRepr(arch["value_repr"]),
                        lk.Interp.Linear, lk.ParamDtype(arch["param_dtype"]))
    oob = lk.OobConfig(lk.BoundaryMode(arch["boundary_mode"]), lk.OobPolicy(arch["oob_policy"]))
    g = lk.compile_layer(spec, qc, oob)
    lk.save_artifact(g, tmp_path / "g.lut")
    assert filecmp.cmp(tmp_path / "g.lut", os.path.join(GOLD, arch["file"]), shallow=False)
    monkeypatch.setenv("LKG_TILE_ONLY_BYTES", "0")
    g2 = lk.compile_layer(spec, qc, oob)
    lk.save_artifact(g2, tmp_path / "g2.lut", store=True)
    X = np.random.default_rng(4).uniform(-1.4, 1.4, (2000, spec.in_dim)).astype(np.float32)
    Y0, _ = lk.lut_layer_forward_batch(g, X)
    Y1, _ = lk.lut_layer_forward_batch(lk.load_artifact(tmp_path / "g2.lut"), X)
    assert np.array_equal(Y0, Y1)


@pytest.mark.gpu
def test_load_errors_gpu(lk):
    for name, exc in (("payload_flip", lk.CorruptBlobError), ("dtype_mismatch", lk.ShapeError),
                      ("knots_nan", lk.NonFiniteError)):
        with pytest.raises(exc):
            lk.load_artifact(os.path.join(GOLD, "corrupt", name + ".lut"))


def _synthetic(lk, d=32, m=1024, K=8, L=80, seed=0):
    rng = np.random.default_rng(seed)
    E = d * m
    q = (np.cumsum(rng.integers(-3, 4, (E * K, L)), axis=1) % 255).astype(np.uint8).ravel()
    return lk.LutLayerArtifact(
        d, m, L, lk.ValueRepr.SplineComponent, lk.Scheme.Asymmetric, lk.Dtype.Uint8, lk.ParamDtype.F32,
        lk.OobConfig(), "silu", knots=np.linspace(-1, 1, K + 1).astype(np.float32), q_table=q,
        scale=rng.uniform(0, 1e-2, E * K).astype(np.float32), y_min=rng.normal(0, 1, E * K).astype(np.float32),
        edge_base_scale=np.ones(E, np.float32), edge_spline_scale=np.ones(E, np.float32),
        edge_out_scale=np.ones(E, np.float32))


def test_parallel_inflate_archive(lk, tmp_path):
    """Mode 2 (parallel=True): independently deflated segments forming one valid deflate stream
    plus a segment index; zipfile reads it, our reader inflates segments on all threads, a
    corrupted segment is a CorruptBlobError, and the same artifact in the reference format
    carries identical entry payloads."""
    a = _synthetic(lk)
    par, ref_fmt = tmp_path / "par.lut", tmp_path / "ref.lut"
    lk.save_artifact(a, par, parallel=True)
    lk.save_artifact(a, ref_fmt)
    with zipfile.ZipFile(par) as zp, zipfile.ZipFile(ref_fmt) as zr:
        assert zp.testzip() is None
        for n in zr.namelist():
            assert zp.read(n) == zr.read(n), n
    lk.check_artifact(par)
    raw = bytearray(open(par, "rb").read())
    raw[len(raw) // 2] ^= 0x55
    bad = tmp_path / "bad.lut"
    bad.write_bytes(bytes(raw))
    with pytest.raises(lk.CorruptBlobError):
        lk.check_artifact(bad)


def test_parallel_archive_read_by_reference(lk, ref, tmp_path):
    a = _synthetic(lk, d=16, m=512)
    lk.save_artifact(a, tmp_path / "par.lut", parallel=True)
    lk.save_artifact(a, tmp_path / "ref.lut")
    assert ref.artifact_load_status(tmp_path / "par.lut", tmp_path / "re.lut") == 0
    assert filecmp.cmp(tmp_path / "re.lut", tmp_path / "ref.lut", shallow=False)
