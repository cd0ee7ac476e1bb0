"""Where the end-to-end single_pass_pca seconds go at a config (Omega draw,
pass, blocked QB, small SVD, U/S/V to host).  python tools/pca_probe.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1704_07669_b200 as P
from paper_1704_07669_b200.algorithms import finish_svd
from paper_1704_07669_b200.device import host_copy
from paper_1704_07669_b200.linalg import STREAM_SKETCH
from paper_1704_07669_b200.synth import config_matrix, config_shape

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cs = config_shape(cfg_name)
a = config_matrix(cfg_name, device=torch.device("cuda:0"))
cfg = P.PcaConfig(k=cs["k"], oversample=cs["l"] - cs["k"], seed=1)
for rep in range(3):
    T = {}
    torch.cuda.synchronize()
    t = time.perf_counter()

    def lap(name):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[name] = round(1e3 * (now - t), 2)
        t = now

    om = P.gaussian_matrix_device(a.shape[1], cfg.l, cfg.seed, stream=STREAM_SKETCH)
    lap("omega")
    st = P.sketch_pass(P.DeviceRowStream(a), om, keep_on_device=True)
    lap("pass")
    f = P.blocked_qb(st.g, st.h, st.omega, cfg.block_size, repair_seed=cfg.seed)
    lap("qb")
    u, s, v = finish_svd(f, cfg.k)
    lap("svd")
    u, s, v = host_copy(u), host_copy(s), host_copy(v)
    lap("to_host")
    print(rep, T, "total", round(sum(T.values()), 2))
