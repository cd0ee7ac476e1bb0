"""Golden fixtures for SURVEY.md §8(f) rank 4 — the two-pass yardstick
``basic_rand_svd`` (algorithms.py:207-263) and the two-sketch one-pass
baseline ``legacy_single_pass`` (algorithms.py:312-392) — made by the REAL
reference (run once in the build container; outputs committed):

    python tests/golden/make_golden_alg.py     -> tests/golden/golden_alg.npz

Inputs are small and stored with the outputs: the reference's synth matrix
for fp64 cases, the BASELINE low-rank + noise construction (fp32, widened to
fp64 as FileRowStream does) for fp32 cases, plain and centered, and one
ill-conditioned co-sketch system (legacy's ConditioningWarning)."""
import os
import sys
import warnings

import numpy as np
from threadpoolctl import threadpool_limits

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import streampca as sp  # noqa: E402  (the reference)
from streampca.algorithms import basic_rand_svd, legacy_single_pass  # noqa: E402

from oracle import gaussian, reference_synth_matrix, synth_lowrank_plus_noise  # noqa: E402

CASES = {
    # name: (matrix builder, k, oversample, block_size, seed, center, block_rows)
    "f64": (lambda: reference_synth_matrix(400, 150, 10.0 ** (-np.arange(150) / 37.0), seed=21),
            12, 8, 5, 3, False, 64),
    "f64c": (lambda: reference_synth_matrix(300, 90, 0.9 ** np.arange(90), seed=22) + 2.5,
             10, 10, 10, 4, True, 50),
    "f32": (lambda: synth_lowrank_plus_noise(800, 300, 60, "inv", 1e-3, seed=23).astype(np.float64),
            20, 10, 10, 1, False, 256),
    "f32c": (lambda: (synth_lowrank_plus_noise(700, 240, 40, "exp30", 1e-3, seed=24) + 0.75)
             .astype(np.float32).astype(np.float64), 15, 15, 10, 2, True, 200),
}

out = {}
with threadpool_limits(limits=1):
    for name, (build, k, p, b, seed, center, br) in CASES.items():
        a = build()
        # fp32 cases hold fp32 values exactly: store them as float32
        out[f"{name}_a"] = a.astype(np.float32) if name.startswith("f32") else a
        out[f"{name}_cfg"] = np.array([k, p, b, seed, int(center), br])
        cfg = sp.PcaConfig(k=k, oversample=p, block_size=b, seed=seed, center=center)
        r = basic_rand_svd(a, cfg, block_rows=br)
        out[f"{name}_basic_u"], out[f"{name}_basic_s"], out[f"{name}_basic_v"] = r.u, r.s, r.v
        out[f"{name}_basic_meta"] = np.array([r.passes, r.retained_floats])
        if center:
            out[f"{name}_basic_mean"] = r.mean
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            r = legacy_single_pass(a, cfg, block_rows=br)
        out[f"{name}_legacy_u"], out[f"{name}_legacy_s"], out[f"{name}_legacy_v"] = r.u, r.s, r.v
        out[f"{name}_legacy_meta"] = np.array([r.passes, r.retained_floats, len(r.warnings)])
        if center:
            out[f"{name}_legacy_mean"] = r.mean
    # the conditioning warning (algorithms.py:366-372): full-rank data (so Q,
    # Qt and the condition number are determined, not rounding noise) and a
    # threshold the co-sketch system's condition number exceeds
    a = gaussian(200, 60, seed=31) * np.exp(-np.arange(60) / 6.0)
    out["ill_a"] = a
    cfg = sp.PcaConfig(k=5, oversample=15, block_size=5, seed=7)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        r = legacy_single_pass(a, cfg, block_rows=40, cond_warn=2.0)
    out["ill_legacy_s"] = r.s
    out["ill_legacy_nwarn"] = np.array([len(r.warnings), len(w)])
    out["ill_legacy_msg"] = np.array(r.warnings[0] if r.warnings else "")

np.savez_compressed(os.path.join(HERE, "golden_alg.npz"), **out)
print("wrote", len(out), "arrays:", sorted(out))
