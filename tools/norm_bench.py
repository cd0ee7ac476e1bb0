"""Normalized-row pass (SURVEY §8 f, rank 3): the pass over
NormalizedRowStream(DeviceRowStream(A)) (normalisation fused into the pass
kernel) vs the plain pass, both timed with CUDA events on the kernel, and the
standalone normalisation kernel against the HBM roofline (read + write of A).
    python tools/norm_bench.py [config] [rows]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P
from paper_1704_07669_b200.sketch import normalize_rows_device
from paper_1704_07669_b200.synth import config_matrix, config_shape

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else None
cs = config_shape(cfg)
a = config_matrix(cfg, device=torch.device("cuda:0"), rows=rows)
m, n = a.shape
om = P.gaussian_matrix(n, cs["l"], seed=1)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


t_plain = timed(lambda: P.sketch_pass(P.DeviceRowStream(a), om, keep_on_device=True))
t_norm = timed(lambda: P.sketch_pass(P.NormalizedRowStream(P.DeviceRowStream(a)), om, keep_on_device=True))


def kernel_ms(normalize, reps=5):
    sk = P.GpuSketch(n, om, np.float32, rows_hint=m, normalize=normalize)
    sk.enable_timing(True)
    for _ in range(2):
        sk.reset()
        sk.push(a, 0, final=True)
        sk.finish()
    sk.enable_timing(False)
    sk.enable_timing(True)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        sk.reset()
        sk.push(a, 0, final=True)
    ev1.record()
    torch.cuda.synchronize()
    sk.close()
    return ev0.elapsed_time(ev1) / reps


pass_plain_ms, pass_norm_ms = kernel_ms(False), kernel_ms(True)
out = torch.empty_like(a)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
normalize_rows_device(a, out)
ev0.record()
for _ in range(5):
    normalize_rows_device(a, out)
ev1.record()
torch.cuda.synchronize()
k_ms = ev0.elapsed_time(ev1) / 5
peaks = {}
try:
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
except Exception:
    pass
hbm = next((v for k, v in peaks.items() if "hbm" in k.lower() and isinstance(v, (int, float))), 6564.0)
bytes_k = 2 * m * n * 4
print(json.dumps({"metric": "normalized sketch-pass GB/s of A", "config": cfg, "m": m, "n": n,
                  "pass_ms_plain": pass_plain_ms, "pass_ms_normalized_fused": pass_norm_ms,
                  "normalized_pass_gbs": m * n * 4 / pass_norm_ms / 1e6,
                  "plain_gbs": m * n * 4 / t_plain / 1e9, "normalized_gbs": m * n * 4 / t_norm / 1e9,
                  "normalize_kernel_ms": k_ms, "normalize_kernel_gbs": bytes_k / k_ms / 1e6,
                  "normalize_kernel_hbm_frac": bytes_k / k_ms / 1e6 / hbm, "hbm_peak_gbs": hbm,
                  "note": "kernel bytes = read + write of A; pass wall times include Omega upload and finish"}))
