"""Fixed costs around one pass (handle create / push / finish / close) at
config 2 — the part of an end-to-end call that is not the pass kernel.
    python tools/overhead_probe.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P
from paper_1704_07669_b200 import _lib
from paper_1704_07669_b200.synth import config_matrix

a = config_matrix("cfg2", device=torch.device("cuda:0"))
om = P.gaussian_matrix(10000, 60, seed=1)
m, n, l = a.shape[0], 10000, 60
g = torch.empty((m, l), dtype=torch.float64, device="cuda")
hh = torch.empty((n, l), dtype=torch.float64, device="cuda")
cs = torch.empty((n,), dtype=torch.float64, device="cuda")
for rep in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk = P.GpuSketch(n, om, np.float32, rows_hint=m)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sk.push(a, 0, final=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rows = ctypes.c_int64(0)
    rc = sk.lib.spca_sketch_finish(sk.h, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(hh.data_ptr()),
                                   ctypes.c_void_p(cs.data_ptr()), ctypes.byref(rows), _lib.MEM_DEVICE)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    sk.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} push {1e3*(t2-t1):.2f} finish(C) {1e3*(t3-t2):.2f} close {1e3*(t4-t3):.2f} ms")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = P.sketch_pass(P.DeviceRowStream(a), om, keep_on_device=True)
    torch.cuda.synchronize()
    print("sketch_pass (device result) ms", round(1e3 * (time.perf_counter() - t0), 2))
