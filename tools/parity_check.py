"""Print S / subspace-angle errors of the GPU path vs the oracle for fp32 constructions."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_1704_07669_b200 as P
cases = [("f32 golden 4000x1500 k50", (4000, 1500, 200, "inv", 1e-3, 11), 50, 10),
         ("cfg3-like 8000x2048 exp30", (8000, 2048, 300, "exp30", 1e-3, 3), 100, 20),
         ("cfg5-like 3000x8000 pow15", (3000, 8000, 500, "pow15", 1e-3, 5), 200, 50),
         ("cfg2-like 40000x10000 inv", (40000, 10000, 200, "inv", 1e-3, 2), 50, 10)]
for name, gen, k, p in cases:
    a = O.synth_lowrank_plus_noise(*gen[:5], seed=gen[5])
    u0, s0, v0, *_ = O.oracle_single_pass(a, k=k, oversample=p, seed=1, block_rows=4096)
    for prec in ("simt", "tc"):
        try:
            r = P.single_pass_pca(a, P.PcaConfig(k=k, oversample=p, seed=1), precision=prec)
        except P.ConfigError as exc:
            print(f"{name:28s} {prec:5s} skipped: {exc}")
            continue
        print(f"{name:28s} {prec:5s} S rel {np.max(np.abs(r.s-s0)/s0):.2e}  angU {O.subspace_angle(r.u,u0):.2e}  "
              f"angV {O.subspace_angle(r.v,v0):.2e}", flush=True)
