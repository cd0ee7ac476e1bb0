"""Golden fixtures for the §8 (f) widening rows, made by the REAL reference
(run once in the build container; outputs committed):

    python tests/golden/make_golden_f.py     -> tests/golden/golden_f.npz

Cases: normalize_rows on a matrix with constant / zero / ordinary rows
(sketch.py:142-153); single_pass_pca over NormalizedRowStream
(sketch.py:156-182); the SinglePassPCA estimator (estimator.py:36-111) fit /
transform / inverse_transform with centering, with normalisation and at
power 1. Inputs come from oracle.gaussian (Philox) seeds and are stored too
(they are small)."""
import os
import sys

import numpy as np
from threadpoolctl import threadpool_limits

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import streampca as sp  # noqa: E402  (the reference)
from streampca.estimator import SinglePassPCA  # noqa: E402
from streampca.sketch import NormalizedRowStream, normalize_rows  # noqa: E402
from streampca.streams import ArrayRowStream  # noqa: E402

from oracle import gaussian, synth_lowrank_plus_noise  # noqa: E402

out = {}
with threadpool_limits(limits=1):
    # normalize_rows: ordinary, constant, zero, tiny-scale and large-offset rows
    x = gaussian(9, 13, seed=41) * 3.0
    x[2] = 7.5
    x[4] = 0.0
    x[6] *= 1e-12
    x[7] += 1e6
    out["norm_in"] = x
    out["norm_out"] = normalize_rows(x)

    # single_pass_pca over a normalized stream
    a = synth_lowrank_plus_noise(400, 120, 15, "inv", 1e-3, 5)
    out["ns_a"] = a
    cfg = sp.PcaConfig(k=8, oversample=6, block_size=7, seed=2)
    r = sp.single_pass_pca(NormalizedRowStream(ArrayRowStream(a)), cfg, block_rows=64)
    out["ns_u"], out["ns_s"], out["ns_v"] = r.u, r.s, r.v
    # the same on the fp32-rounded matrix widened to fp64 (what FileRowStream feeds it)
    a32 = a.astype(np.float32).astype(np.float64)
    r = sp.single_pass_pca(NormalizedRowStream(ArrayRowStream(a32)), cfg, block_rows=64)
    out["ns32_u"], out["ns32_s"], out["ns32_v"] = r.u, r.s, r.v

    # estimator: default (center), normalize, power 1
    x2 = gaussian(37, 120, seed=43)
    z = gaussian(5, 8, seed=44)
    out["est_x2"], out["est_z"] = x2, z
    for tag, kw in (("c", {}), ("n", {"normalize": True}), ("p", {"power": 1}),
                    ("nc", {"center": False})):
        est = SinglePassPCA(n_components=8, oversample=6, block_size=7, seed=3, **kw).fit(a)
        out[f"est_{tag}_components"] = est.components_
        out[f"est_{tag}_sv"] = est.singular_values_
        out[f"est_{tag}_ev"] = est.explained_variance_
        out[f"est_{tag}_mean"] = est.mean_
        out[f"est_{tag}_meta"] = np.array([est.n_samples_, est.n_passes_, est.retained_floats_])
        out[f"est_{tag}_t"] = est.transform(x2)
        out[f"est_{tag}_it"] = est.inverse_transform(z)
np.savez_compressed(os.path.join(HERE, "golden_f.npz"), **out)
print("wrote", len(out), "arrays")
