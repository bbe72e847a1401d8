import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_03332_b200 as lk
from paper_2601_03332_b200._capi import lib
rows = int(sys.argv[1])
eng = lk.Engine(0)
chain = [lk.compile_layer(lk.recipe_layer(2, l), lk.QuantConfig(64), lk.OobConfig(), engine=eng) for l in range(2)]
dev = [a.device(eng) for a in chain]
hs = (C.c_void_p * 2)(*[d.handle for d in dev])
X = torch.from_numpy(lk.recipe_inputs(2, 0, rows)).cuda()
Y = torch.empty((rows, 2), device="cuda")
for _ in range(5):
    lib().lkg_model_forward(eng.handle, hs, 2, C.c_void_p(X.data_ptr()), rows, C.c_void_p(Y.data_ptr()), None)
eng.synchronize()
