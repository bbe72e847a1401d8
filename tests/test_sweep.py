"""Sweep driver (paper_2601_03332_b200/sweep.py) against the reference's own
run_sweep / collect_results output (tests/golden/sweep/, written by tests/golden/make_sweep.py
from oracle/_ref/sweep_ref = the reference's sweep.cpp compiled in place).

CPU: the nlohmann dump(2) printer on every golden file, cell config.json, manifest text, report
readers and their error classes, sweep-config parsing, and collect_results over the reference's
own per-seed reports (byte-identical CSVs). GPU: run_sweep on the same configurations — artifact
bytes, config.json and manifest.json identical, eval reports equal (counts exact, floats within
1e-9 relative), CSVs equal — and the honest bench (bench reports readable, speed CSV filled)."""
import glob
import hashlib
import json
import os
import shutil

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sweep")
NAMES = sorted(os.listdir(GOLD)) if os.path.isdir(GOLD) else []


@pytest.fixture(scope="module")
def sw():
    from paper_2601_03332_b200 import sweep
    return sweep


def _golden_files(kind):
    return sorted(glob.glob(os.path.join(GOLD, "*", "cells", "*", "*", kind)))


def test_golden_present():
    assert NAMES == ["grid", "phi_f16"]
    assert len(_golden_files("report.json")) == 16 * 2 + 2


@pytest.mark.parametrize("kind", ["report.json", "config.json", "manifest.json"])
def test_nlohmann_dump_matches_reference_files(sw, kind):
    """Every JSON file the reference wrote re-prints byte for byte (sorted keys, 2-space indent,
    shortest round-trip doubles, uint64 seeds)."""
    files = _golden_files(kind)
    assert files
    for p in files:
        raw = open(p, "rb").read().decode()
        assert sw.dumps(json.loads(raw)) == raw, p


def test_number_format_edge_cases(sw):
    # nlohmann: fixed notation for decimal exponents in (-4, 15], else d[.ddd]e+XX
    cases = [(0.0, "0.0"), (-0.0, "-0.0"), (1.0, "1.0"), (0.1, "0.1"), (1e-4, "0.0001"), (1e-5, "1e-05"),
             (123.5, "123.5"), (1e15, "1e+15"), (1234567890123456.0, "1.234567890123456e+15"),
             (999999999999999.0, "999999999999999.0"), (1.5e300, "1.5e+300"), (2.5e-300, "2.5e-300"),
             (float("nan"), "null"), (float("inf"), "null")]
    for v, s in cases:
        assert sw._num(v) == s, (v, sw._num(v), s)


@pytest.mark.parametrize("name", NAMES)
def test_cell_config_json_matches_reference(sw, name):
    cfg = sw.load_sweep_config(os.path.join(GOLD, name, "config.json"))
    n = 0
    for p in glob.glob(os.path.join(GOLD, name, "cells", "*", "*", "config.json")):
        j = json.loads(open(p).read())
        lk_enum = __import__("paper_2601_03332_b200").parse_enum
        got = sw.cell_config_json(cfg, j["L"], lk_enum("scheme", j["scheme"]),
                                  lk_enum("boundary_mode", j["boundary_mode"]), lk_enum("oob_policy", j["oob_policy"]),
                                  j["seed"])
        assert got == open(p).read(), p
        assert os.path.basename(os.path.dirname(os.path.dirname(p))) == sw.cell_dir_name(
            j["L"], lk_enum("scheme", j["scheme"]), lk_enum("boundary_mode", j["boundary_mode"]),
            lk_enum("oob_policy", j["oob_policy"]))
        n += 1
    assert n == len(cfg.Ls) * len(cfg.schemes) * len(cfg.boundary_modes) * len(cfg.oob_policies) * len(cfg.seeds)


def test_manifest_text_matches_reference(lk, sw):
    """artifact_manifest_json (host, metadata only) == the manifest.json the reference wrote."""
    for p in _golden_files("manifest.json"):
        m = json.loads(open(p).read())
        a = lk.LutLayerArtifact(m["in_dim"], m["out_dim"], m["L"], lk.parse_enum("value_repr", m["value_repr"]),
                                lk.parse_enum("scheme", m["scheme"]), lk.parse_enum("dtype", m["dtype"]),
                                lk.parse_enum("param_dtype", m["param_dtype"]),
                                lk.OobConfig(lk.parse_enum("boundary_mode", m["boundary_mode"]),
                                             lk.parse_enum("oob_policy", m["oob_policy"])), m.get("base_kind", ""))
        a.knots = np.zeros(m["segments"] + 1, np.float32)
        assert lk.artifact_manifest_json(a) == open(p).read(), p


@pytest.mark.parametrize("name", NAMES)
def test_collect_results_matches_reference_csvs(sw, name, tmp_path):
    """collect_results over the reference's own cell reports writes the reference's CSV bytes."""
    root = tmp_path / "root"
    shutil.copytree(os.path.join(GOLD, name, "cells"), root)
    sw.collect_results(root, tmp_path / "csv")
    for p in sorted(glob.glob(os.path.join(GOLD, name, "csv", "*.csv"))):
        assert (tmp_path / "csv" / os.path.basename(p)).read_bytes() == open(p, "rb").read(), p
    # a rerun rewrites identical bytes; failed / partial cells are ignored
    bad = root / "L16_symmetric_closed_clip_x" / "seed9"
    if name == "grid":
        bad.mkdir()
        (bad / "config.json").write_text((root / "L16_symmetric_closed_clip_x" / "seed0" / "config.json").read_text())
        (bad / "report.json").write_text(sw.dumps({"kind": "error", "message": "x", "seed": 9}))
        (root / "stray.txt").write_text("not a cell")
    sw.collect_results(root, tmp_path / "csv2")
    for p in sorted(glob.glob(os.path.join(GOLD, name, "csv", "*.csv"))):
        assert (tmp_path / "csv2" / os.path.basename(p)).read_bytes() == open(p, "rb").read(), p


def test_report_round_trip_and_errors(lk, sw, tmp_path):
    p = _golden_files("report.json")[0]
    r = sw.load_eval_report(p)
    assert r.n_samples == 512 and r.quant.samples_per_segment in (16, 64) and r.mae_oob is None
    assert sw.eval_report_json(r) == open(p).read()
    assert sw.read_report_kind(p) == "eval"
    b = sw.BenchReport(r.quant, r.oob, lk.Tier.Optimized, "steady", 3, 1024, 50, 200, 4, 1, 1.0, 0.1, 1.0, 0.5, 0.05,
                       0.5, 1.0 / 1024, 0.5 / 1024, 2.0, 2.0, r.memory)
    sw.save_bench_report(b, tmp_path / "b.json")
    assert sw.load_bench_report(tmp_path / "b.json") == b
    assert sw.read_report_kind(tmp_path / "b.json") == "bench"
    (tmp_path / "bad.json").write_text("[1, 2]")
    with pytest.raises(lk.CorruptBlobError):
        sw.load_eval_report(tmp_path / "bad.json")
    with pytest.raises(lk.CorruptBlobError):
        sw.read_report_kind(tmp_path / "bad.json")
    with pytest.raises(lk.ShapeError):
        sw.load_eval_report(tmp_path / "b.json")
    j = json.loads(open(p).read())
    del j["metrics"]["mae_inrange"]
    (tmp_path / "miss.json").write_text(json.dumps(j))
    with pytest.raises(lk.MissingKeyError):
        sw.load_eval_report(tmp_path / "miss.json")
    j = json.loads(open(p).read())
    j["quant"]["scheme"] = "ternary"
    (tmp_path / "enum.json").write_text(json.dumps(j))
    with pytest.raises(lk.ConfigError):
        sw.load_eval_report(tmp_path / "enum.json")
    with pytest.raises(lk.IoError):
        sw.read_report_kind(tmp_path / "absent.json")


def test_parse_sweep_config(lk, sw):
    d = sw.parse_sweep_config("{}")
    assert d == sw.SweepConfig() and d.Ls == [16, 32, 64, 128] and d.seeds == [0, 1, 2, 3, 4]
    assert (d.n_samples, d.in_dim, d.out_dim, d.segments, d.degree, d.bench_batch) == (4096, 10, 8, 8, 3, 1024)
    c = sw.parse_sweep_config(json.dumps({"Ls": [8], "schemes": ["asymmetric"], "value_repr": "phi",
                                          "param_dtype": "f16", "with_speed": False, "seeds": [7]}))
    assert c.Ls == [8] and c.schemes == [lk.Scheme.Asymmetric] and c.value_repr == lk.ValueRepr.Phi
    assert c.param_dtype == lk.ParamDtype.F16 and not c.with_speed and c.seeds == [7]
    for bad in ["[]", "not json", '{"Lz": [16]}', '{"Ls": []}', '{"seeds": []}', '{"schemes": ["odd"]}',
                '{"Ls": "16"}', '{"with_speed": 1}', '{"n_samples": -1}', '{"boundary_modes": []}']:
        with pytest.raises(lk.ConfigError):
            sw.parse_sweep_config(bad)
    with pytest.raises(lk.IoError):
        sw.load_sweep_config("/nonexistent/sweep.json")


# ------------------------------------------------------------------ GPU
def _close(a, b, rel=1e-9):
    return abs(a - b) <= rel * max(abs(a), abs(b)) + 1e-300


def _csv_rows(path):
    return [line.split(",") for line in open(path).read().splitlines()]


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_sweep_matches_reference(lk, sw, name, tmp_path):
    cfg = sw.load_sweep_config(os.path.join(GOLD, name, "config.json"))
    s = sw.run_sweep(cfg, tmp_path / "root")
    assert (s.n_total, s.n_run, s.n_failed, s.n_skipped) == (len(_golden_cells(name)),) * 2 + (0, 0)
    digests = json.load(open(os.path.join(GOLD, name, "digests.json")))
    for rel in _golden_cells(name):
        ours, gold = tmp_path / "root" / rel, os.path.join(GOLD, name, "cells", rel)
        assert hashlib.sha256((ours / "artifact.lut").read_bytes()).hexdigest() == digests[rel], rel
        for fn in ("config.json", "manifest.json"):
            assert (ours / fn).read_bytes() == open(os.path.join(gold, fn), "rb").read(), (rel, fn)
        a, b = json.loads((ours / "report.json").read_text()), json.loads(open(os.path.join(gold, "report.json")).read())
        for k in ("kind", "seed", "n_samples", "quant", "oob", "memory"):
            assert a[k] == b[k], (rel, k)
        assert a["metrics"].keys() == b["metrics"].keys()
        for k, v in b["metrics"].items():
            if k.startswith("n_"):
                assert a["metrics"][k] == v, (rel, k)
            else:
                assert _close(a["metrics"][k], v), (rel, k, a["metrics"][k], v)
        assert not (ours / "bench_optimized.json").exists()  # with_speed false
    # rerun: every cell skipped
    assert sw.run_sweep(cfg, tmp_path / "root").n_skipped == s.n_total
    sw.collect_results(tmp_path / "root", tmp_path / "csv")
    for p in sorted(glob.glob(os.path.join(GOLD, name, "csv", "*.csv"))):
        got, want = _csv_rows(tmp_path / "csv" / os.path.basename(p)), _csv_rows(p)
        assert len(got) == len(want)
        for rg, rw in zip(got, want):
            assert len(rg) == len(rw)
            for x, y in zip(rg, rw):
                assert x == y or _close(float(x), float(y), 1e-8), (p, x, y)


def _golden_cells(name):
    return sorted(os.path.relpath(d, os.path.join(GOLD, name, "cells"))
                  for d in glob.glob(os.path.join(GOLD, name, "cells", "*", "*")))


@pytest.mark.gpu
def test_gpu_sweep_with_speed_and_failures(lk, sw, tmp_path):
    """with_speed: the same-backend honest bench (spline kernel vs LUT kernel) per cell, readable
    bench reports, speed_optimized.csv filled; a failing cell (L=1) writes an error report and the
    sweep moves on; cold_start bench."""
    cfg = sw.parse_sweep_config(json.dumps({"Ls": [1, 32], "schemes": ["symmetric"], "boundary_modes": ["closed"],
                                            "oob_policies": ["clip_x"], "seeds": [5], "n_samples": 256,
                                            "bench_batch": 4096, "bench_warmup_iters": 2, "bench_timed_iters": 5}))
    s = sw.run_sweep(cfg, tmp_path / "root")
    assert (s.n_total, s.n_run, s.n_failed) == (2, 1, 1)
    err = json.loads((tmp_path / "root" / "L1_symmetric_closed_clip_x" / "seed5" / "report.json").read_text())
    assert err["kind"] == "error" and err["cell"]["L"] == 1
    d = tmp_path / "root" / "L32_symmetric_closed_clip_x" / "seed5"
    b = sw.load_bench_report(d / "bench_optimized.json")
    assert b.batch == 4096 and b.timed_iters == 5 and b.lut_ms_mean > 0 and b.spline_ms_mean > 0
    assert b.speedup == pytest.approx(b.spline_ms_mean / b.lut_ms_mean)
    sw.collect_results(tmp_path / "root", tmp_path / "csv")
    rows = _csv_rows(tmp_path / "csv" / "speed_optimized.csv")
    assert len(rows) == 2 and rows[1][:5] == ["32", "symmetric", "closed", "clip_x", "1"]
    assert float(rows[1][5]) == pytest.approx(b.speedup, rel=1e-11)
    assert _csv_rows(tmp_path / "csv" / "speed_scalar.csv")[1][4] == "0"
    layer = lk.gen_layer(5, 10, 8, 8, 3)
    X = lk.gen_inputs(5 ^ sw.INPUT_SEED_SALT, 2048, 10, -1.0, 1.0, True)
    cold = sw.run_honest_bench(layer, d / "artifact.lut", X, sw.BenchOptions(1, 3, mode="cold_start"))
    assert cold.mode == "cold_start" and cold.lut_ms_mean > 0
    with pytest.raises(lk.ConfigError):
        sw.run_honest_bench(layer, d / "artifact.lut", X, sw.BenchOptions(threads=2))
    with pytest.raises(lk.DimensionError):
        sw.run_honest_bench(layer, d / "artifact.lut", X[:, :4])


def test_reference_collect_reads_gpu_sweep_files(sw, tmp_path):
    """The REFERENCE's run_sweep + collect_results (oracle/_ref/sweep_ref) over a cell written by
    the GPU sweep (tests/golden/sweep_gpu: configs[2]-shaped L=64 cell from tools/sweeps/c3_grid.json,
    eval + honest-bench reports): it skips the complete cell, reads our report files, and its CSVs
    equal ours byte for byte."""
    import subprocess
    binp = os.path.join(os.path.dirname(GOLD), "..", "..", "oracle", "_ref", "sweep_ref")
    if not os.path.exists(binp):
        pytest.skip("oracle/_ref/sweep_ref not built (make -C oracle ref sweep; needs /root/reference)")
    root = tmp_path / "root"
    shutil.copytree(os.path.join(os.path.dirname(GOLD), "sweep_gpu"), root)
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"Ls": [64], "schemes": ["symmetric"], "boundary_modes": ["half_open"],
                               "oob_policies": ["clip_x"], "seeds": [2], "in_dim": 64, "out_dim": 64}))
    out = subprocess.run([binp, str(cfg), str(root), str(tmp_path / "ref_csv")], check=True, capture_output=True,
                         text=True).stdout
    assert json.loads(out) == {"n_total": 1, "n_run": 0, "n_skipped": 1, "n_failed": 0}
    sw.collect_results(root, tmp_path / "our_csv")
    for fn in ("accuracy", "oob_matrix", "memory", "speed_scalar", "speed_optimized"):
        assert (tmp_path / "our_csv" / f"{fn}.csv").read_bytes() == (tmp_path / "ref_csv" / f"{fn}.csv").read_bytes()
    assert _csv_rows(tmp_path / "our_csv" / "speed_optimized.csv")[1][4] == "1"
