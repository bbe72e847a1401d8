import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2601_03332_b200 as lk
from paper_2601_03332_b200._capi import lib
eng = lk.Engine(0)
a = lk.compile_layer(lk.recipe_layer(2, 0), lk.QuantConfig(64), lk.OobConfig(), engine=eng)
dl = a.device(eng)
X = torch.from_numpy(lk.recipe_inputs(2, 0, 100000)).cuda()
Y = torch.empty((100000, 16), device="cuda")
st = lib().lkg_layer_forward(eng.handle, dl.handle, C.c_void_p(X.data_ptr()), 100000, C.c_void_p(Y.data_ptr()), None)
print("status", st, lib().lkg_last_error())
eng.synchronize()
