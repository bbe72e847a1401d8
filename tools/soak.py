"""Repeat-launch soak: every main kernel variant launched many times on the same inputs, the output
bits and OobStats of every launch compared with the first (a shared-memory / TMEM / mbarrier race in
the barrier-free stage release, the x boxes, the input split or the fused chain would make results
launch-dependent). L2 is disturbed between launches.  Usage: python tools/soak.py [repeats]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_03332_b200 as lk  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
eng = lk.Engine(0)
junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def soak(tag, fn, n=N):
    ref = None
    for it in range(n):
        junk.random_(0, 255) if it % 8 == 0 else None
        out = fn()
        sig = tuple(o.clone() if torch.is_tensor(o) else o for o in out)
        if ref is None:
            ref = sig
            continue
        for a, b in zip(ref, sig):
            ok = torch.equal(a, b) if torch.is_tensor(a) else a == b
            if not ok:
                print(f"{tag}: MISMATCH at launch {it}", flush=True)
                sys.exit(1)
    print(f"{tag}: {n} launches bit-identical", flush=True)


def layer_case(tag, spec, X, L=64, scheme=0, bm=1, op=0, n=N):
    a = lk.compile_layer(spec, lk.QuantConfig(L, lk.Scheme(scheme), lk.Dtype(scheme)),
                         lk.OobConfig(lk.BoundaryMode(bm), lk.OobPolicy(op)), engine=eng)

    def fn():
        Y, st = lk.lut_layer_forward_batch(a, X, engine=eng)
        return Y, (st.n_oob_samples, st.n_oob_inputs)
    soak(tag, fn, n)


X2 = torch.from_numpy(lk.recipe_inputs(2, 0, 1_000_000)).cuda()
layer_case("C2 layer 0, 1M rows (BAL, XB=2, IDP)", lk.recipe_layer(2, 0), X2, n=max(20, N // 4))
layer_case("C2 layer 0, 4096 rows (R=1, 4 stages)", lk.recipe_layer(2, 0), X2[:4096].contiguous())
layer_case("C2a layer 0, 100k rows (asym)", lk.recipe_layer(2, 0), X2[:100_000].contiguous(), scheme=1)
X3 = torch.from_numpy(lk.recipe_inputs(3, 0, 262_144)).cuda()
layer_case("C3 layer 0 (REC walk, 4 j-blocks)", lk.recipe_layer(3, 0), X3, bm=0, n=max(20, N // 2))
layer_case("C3 layer 0 L=128 asym zero_spline (codes in global, lines)", lk.recipe_layer(3, 0), X3[:50_000].contiguous(),
           L=128, scheme=1, op=1)
X4 = torch.empty((4096, 1024), device="cuda").uniform_(-1.2, 1.2)
layer_case("1024->1024, 4096 rows (REC, TMEM f64)", lk.gen_layer(5, 1024, 1024, 8), X4, bm=0, n=max(20, N // 2))
layer_case("1024->512, 2048 rows (input split, reduce kernel)", lk.gen_layer(6, 1024, 512, 8), X4[:2048].contiguous(), bm=0)
X5 = torch.from_numpy(lk.recipe_inputs(5, 0, 2048)).cuda()
layer_case("C5 shard 4096->256 (pair entries, GC, asym, zero_spline)", lk.recipe_layer(5, 0, 0, 256), X5, L=128, scheme=1,
           op=1, n=max(10, N // 8))
ch = lk.compile_model([lk.recipe_layer(1, l) for l in range(2)], lk.QuantConfig(64),
                      lk.OobConfig(lk.BoundaryMode.HalfOpen, lk.OobPolicy.ClipX), engine=eng)
X1 = torch.from_numpy(lk.recipe_inputs(1, 0, 65_536)).cuda()


def chain_fn():
    r = lk.lut_model_forward_batch(ch, X1, engine=eng)
    return (r.Y,) + tuple((s.n_oob_samples, s.n_oob_inputs) for s in r.per_layer)


soak("C1 fused chain, 65536 rows", chain_fn)
print("soak ok", flush=True)
