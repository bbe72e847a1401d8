import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2601_03332_b200 as lk
spec = lk.recipe_layer(2, 0)
a = lk.compile_layer(spec, lk.QuantConfig(64), lk.OobConfig())
for rows in (4096, 65536, 250000):
    X = lk.recipe_inputs(2, 0, rows)
    t = time.time()
    Yd, sd = lk.lut_layer_forward_batch(a, torch.from_numpy(X).cuda())
    Yd = Yd.cpu().numpy()
    print(rows, "dev", time.time() - t, sd.n_oob_inputs, flush=True)
    Yh, sh = lk.lut_layer_forward_batch(a, X)
    print(rows, "host", sh.n_oob_inputs, flush=True)
    bad = np.argwhere(np.any(Yh != Yd, axis=1))[:, 0]
    print(rows, "rows differing", len(bad), bad[:10], bad[-10:] if len(bad) else "", flush=True)
