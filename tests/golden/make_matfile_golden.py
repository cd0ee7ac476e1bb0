"""Golden matrix files written by the reference's own writers (run once, in
the container that has /root/reference; the outputs are committed):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_matfile_golden.py

Writes tests/golden/matfile/: inputs.npz (the arrays), ref_f64.spca,
ref_f32.spca, ref_f32.raw (streampca.matfile.write_matrix) and sigma.csv
(write_sigma_csv)."""
import os

import numpy as np
from streampca import matfile

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "matfile")
os.makedirs(out, exist_ok=True)
rng = np.random.default_rng(20240611)
a64 = rng.standard_normal((7, 5))
a32 = rng.standard_normal((6, 4)) * 3.0
sig = np.array([3.0, 1.5, 1e-13, 0.12345678901234567, 2.0 ** -1074, 1e300])
np.savez(os.path.join(out, "inputs.npz"), a64=a64, a32=a32, sig=sig)
matfile.write_matrix(os.path.join(out, "ref_f64.spca"), a64, dtype="float64", header=True)
matfile.write_matrix(os.path.join(out, "ref_f32.spca"), a32, dtype="float32", header=True)
matfile.write_matrix(os.path.join(out, "ref_f32.raw"), a32, dtype="float32", header=False)
matfile.write_sigma_csv(os.path.join(out, "sigma.csv"), sig)
print("wrote", sorted(os.listdir(out)))
