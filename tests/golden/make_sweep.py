"""Generate the sweep-driver golden fixtures from the REFERENCE itself.

Run in the build container, where /root/reference exists:
    make -C oracle ref sweep && python tests/golden/make_sweep.py
It runs oracle/_ref/sweep_ref (the reference's run_sweep + collect_results, sweep.cpp, compiled
in place) on the small sweep configurations in CONFIGS and commits, under tests/golden/sweep/<name>/:
  * config.json (the sweep config given to the reference),
  * cells/<cell>/seed<N>/{config.json, manifest.json, report.json} exactly as the reference wrote them,
  * digests.json: SHA-256 of every artifact.lut the reference wrote,
  * csv/*.csv: the reference's collect_results tables.
tests/test_sweep.py checks the GPU sweep driver (paper_2601_03332_b200/sweep.py) against them.
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
BIN = os.path.join(ROOT, "oracle", "_ref", "sweep_ref")
OUT = os.path.join(HERE, "sweep")

CONFIGS = {
    # the reference's default grid axes (L x scheme x boundary x policy), 2 seeds, small layers
    "grid": {"Ls": [16, 64], "seeds": [0, 1], "n_samples": 512, "in_dim": 10, "out_dim": 8, "segments": 8,
             "with_speed": False},
    # phi tables with f16 parameters on an odd shape
    "phi_f16": {"Ls": [32], "schemes": ["asymmetric", "symmetric"], "boundary_modes": ["closed"],
                "oob_policies": ["zero_spline"], "seeds": [3], "n_samples": 300, "value_repr": "phi",
                "param_dtype": "f16", "in_dim": 4, "out_dim": 3, "segments": 5, "with_speed": False},
}


def main() -> None:
    if not os.path.exists(BIN):
        sys.exit("build the reference sweep first: make -C oracle ref sweep")
    shutil.rmtree(OUT, ignore_errors=True)
    for name, cfg in CONFIGS.items():
        with tempfile.TemporaryDirectory() as tmp:
            cpath, root, csv = (os.path.join(tmp, "config.json"), os.path.join(tmp, "root"),
                                os.path.join(tmp, "csv"))
            with open(cpath, "w") as f:
                json.dump(cfg, f, indent=2)
            subprocess.run([BIN, cpath, root, csv], check=True, capture_output=True)
            dst = os.path.join(OUT, name)
            os.makedirs(dst)
            shutil.copy(cpath, os.path.join(dst, "config.json"))
            shutil.copytree(csv, os.path.join(dst, "csv"))
            digests = {}
            for cell in sorted(os.listdir(root)):
                for seed in sorted(os.listdir(os.path.join(root, cell))):
                    src = os.path.join(root, cell, seed)
                    d = os.path.join(dst, "cells", cell, seed)
                    os.makedirs(d)
                    for fn in ("config.json", "manifest.json", "report.json"):
                        shutil.copy(os.path.join(src, fn), os.path.join(d, fn))
                    with open(os.path.join(src, "artifact.lut"), "rb") as f:
                        digests[f"{cell}/{seed}"] = hashlib.sha256(f.read()).hexdigest()
            with open(os.path.join(dst, "digests.json"), "w") as f:
                json.dump(digests, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
