"""Disk streaming through FileRowStream (SURVEY §8 f, rank 2): GB/s of A
read from a matrix file (page cache warm: the file was just written) through
the page-locked read pipeline, H2D and the pass, vs the same rows handed
over from pinned memory. Prints one JSON line.
    python tools/file_bench.py [config] [rows] [dir]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P
from paper_1704_07669_b200.synth import config_matrix, config_shape

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else None
where = sys.argv[3] if len(sys.argv) > 3 else "/tmp"
cs = config_shape(cfg)
a = config_matrix(cfg, device=torch.device("cuda:0"), rows=rows)
m, n = a.shape
om = P.gaussian_matrix(n, cs["l"], seed=1)
path = os.path.join(where, f"spca_file_bench_{os.getpid()}.spca")
host = a.cpu().numpy()
t0 = time.perf_counter()
P.matfile.write_matrix(path, host, dtype="float32")
write_s = time.perf_counter() - t0
try:
    res = {}
    for threads in (1, 4, 8, 12, 16):
        times, read_s = [], []
        for rep in range(3):
            fs = P.FileRowStream(path, read_threads=threads)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st = P.sketch_pass(fs, om)
            times.append(time.perf_counter() - t0)
            read_s.append(fs.read_seconds)
        t = float(np.median(times))
        res[threads] = {"gbs": m * n * 4 / t / 1e9, "s": t, "read_s_sum": float(np.median(read_s))}
    # reference point: the same rows from pinned host memory
    pin = torch.from_numpy(host).pin_memory()
    times = []
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st2 = P.sketch_pass(P.PinnedRowStream(pin), om)
        times.append(time.perf_counter() - t0)
    same = bool(np.array_equal(st.g, st2.g) and np.array_equal(st.h, st2.h))
    best = max(res, key=lambda k: res[k]["gbs"])
    print(json.dumps({"metric": "file-stream sketch GB/s of A", "config": cfg, "m": m, "n": n, "l": cs["l"],
                      "file_bytes": os.path.getsize(path), "write_s": write_s,
                      "by_read_threads": res, "best": res[best]["gbs"], "best_threads": best,
                      "pinned_gbs": m * n * 4 / float(np.median(times)) / 1e9,
                      "bitwise_equal_to_pinned": same,
                      "cpu_cores": os.cpu_count(), "page_cache": "warm (file just written)"}))
finally:
    os.unlink(path)
