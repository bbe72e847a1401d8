"""Cold-start artifact loading (the paper's steady vs cold-start comparison):
wall time from a `.lut` file on disk to a device layer ready for the forward kernels
(lkg_artifact_load: parse, inflate, CRC, upload, tile build), against the reference's
load_artifact to host memory (oracle/_ref, artifact_io.cpp:221-300).

Usage: python tools/bench_io.py [cfg] [layer] [L] [reps]   (default: C4 layer 0, L=64)
Prints one JSON line per archive kind (deflate as the reference writes it, stored)."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 0
L = int(sys.argv[3]) if len(sys.argv) > 3 else 64
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
o = Oracle("auto")
eng = lk.default_engine()
spec = lk.recipe_layer(cfg, layer)
g = lk.compile_layer(spec, lk.QuantConfig(L), lk.OobConfig(), engine=eng)
tmp = tempfile.mkdtemp(dir="/tmp")
for mode in ("deflate", "stored", "parallel"):
    store, par = mode == "stored", mode == "parallel"
    path = os.path.join(tmp, f"a_{mode}.lut")
    t0 = time.perf_counter()
    lk.save_artifact(g, path, store=store, parallel=par)
    save_s = time.perf_counter() - t0
    size = os.path.getsize(path)
    ours = []
    for _ in range(reps):
        t0 = time.perf_counter()
        a = lk.load_artifact(path, engine=eng)
        eng.synchronize()
        ours.append(time.perf_counter() - t0)
        del a
    ref = None
    if o.kind == "reference":
        ts = []
        for _ in range(max(1, reps - 1)):
            t0 = time.perf_counter()
            assert o.artifact_load_status(path) == 0
            ts.append(time.perf_counter() - t0)
        ref = min(ts)
    table = spec.in_dim * spec.out_dim * spec.grid.K * L
    print(json.dumps({"metric": "artifact cold-start load, file -> ready", "cfg": cfg, "layer": layer, "L": L,
                      "archive": {"deflate": "deflate (reference format)", "stored": "stored", "parallel": "parallel-inflate deflate"}[mode], "file_bytes": size,
                      "q_table_bytes": table, "save_s": save_s,
                      "ours_to_device_s": min(ours), "ours_GBps_of_table": table / min(ours) / 1e9,
                      "reference_to_host_s": ref, "speedup": (ref / min(ours)) if ref else None}))
    os.remove(path)
torch.cuda.synchronize()
