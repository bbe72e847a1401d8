"""Per-rank cost of the sharded configurations, measured on ONE GPU (only one is available to this
run): rank 0's share of an N-way split is timed alone, N = 1, 2, 4, 8.

  c4 (configs[3], batch sharded, LUT replicated, no collective): the chain forward on rank 0's rows
      of sharding.batch_bounds — the ranks are independent, so t(1) / (N * t(N)) is the strong-scaling
      efficiency every rank would see, up to host/power effects one GPU cannot show.
  c5 (configs[4], output columns sharded): rank 0's column shard of both layers (compiled on the GPU
      from its own edges) on the full 16,384-row batch; layer 1 reads a synthetic full-width hidden
      batch. The NCCL all-gather between the layers is NOT in this figure (it needs the peers): its
      payload per rank is reported so the reader can set it against the compute time.

Usage: python tools/shard_proxy.py [c4|c5] [iters]      (prints one JSON line)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402
from bench import WORKLOADS  # noqa: E402
from paper_2601_03332_b200._capi import lib  # noqa: E402
from paper_2601_03332_b200.sharding import batch_bounds, column_bounds  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg, rows, L, scheme, bm, op = WORKLOADS[wl]
dims, _, _, _ = lk.recipe_dims(cfg)
nl = len(dims) - 1
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
eng = lk.Engine(0, s.cuda_stream)
qc = lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme))
oob = lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op))


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


out = {"workload": wl, "dims": dims, "rows": rows, "iters": iters, "gpu": torch.cuda.get_device_name(0), "ranks": {}}
if wl == "c4":
    chain = [lk.compile_layer(lk.recipe_layer(cfg, l), qc, oob, engine=eng) for l in range(nl)]
    dev = [a.device(eng) for a in chain]
    hs = (C.c_void_p * nl)(*[d.handle for d in dev])
    X = torch.from_numpy(lk.recipe_inputs(cfg, 0, rows)).cuda()
    Y = torch.empty((rows, dims[-1]), device="cuda")
    ee_row = sum(dims[l] * dims[l + 1] for l in range(nl))
    for n in (1, 2, 4, 8):
        r0, r1 = batch_bounds(rows, n, 0)
        nr = r1 - r0
        ms = timed(lambda: lk.lutkan.check(lib().lkg_model_forward(eng.handle, hs, nl, C.c_void_p(X.data_ptr()), nr,
                                                                   C.c_void_p(Y.data_ptr()), None)))
        eng.collect(nl)
        out["ranks"][n] = {"rows_per_rank": nr, "ms_per_step": ms, "edge_evals_per_s_per_rank": nr * ee_row / ms * 1e3}
    t1 = out["ranks"][1]["ms_per_step"]
    for n in (2, 4, 8):
        out["ranks"][n]["strong_scaling_efficiency_proxy"] = t1 / (n * out["ranks"][n]["ms_per_step"])
    out["note"] = "batch shards are independent (no collective): per-rank time of rank 0's rows on one B200"
else:
    X = torch.from_numpy(lk.recipe_inputs(cfg, 0, rows)).cuda()
    for n in (8, 4, 2):
        per_layer = []
        for l in range(nl):
            c0, c1 = column_bounds(dims[l + 1], n, 0)
            a = lk.compile_layer(lk.recipe_layer(cfg, l, c0, c1), qc, oob, engine=eng)
            d = a.device(eng)
            Xin = X if l == 0 else torch.empty((rows, dims[l]), device="cuda").uniform_(-2.2, 2.2)
            Yl = torch.empty((rows, c1 - c0), device="cuda")
            ms = timed(lambda: lk.lutkan.check(lib().lkg_layer_forward(eng.handle, d.handle, C.c_void_p(Xin.data_ptr()),
                                                                       rows, C.c_void_p(Yl.data_ptr()), None)))
            eng.collect(1)
            per_layer.append(ms)
            del a, d
            eng.trim()
        ee = rows * sum(dims[l] * (dims[l + 1] // n) for l in range(nl))
        out["ranks"][n] = {"columns_per_rank": dims[1] // n, "ms_per_layer": per_layer, "ms_per_step_compute": sum(per_layer),
                           "edge_evals_per_s_per_rank": ee / sum(per_layer) * 1e3,
                           "all_gather_payload_bytes_per_rank_per_boundary": rows * (dims[1] // n) * 4}
    out["note"] = ("column shards: rank 0's compute only; the all-gather of the hidden activations between the layers "
                   "(payload above, chunk-pipelined behind the compute in lkg_model_forward_sharded) needs the peers")
print(json.dumps(out))
