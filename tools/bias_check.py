"""Tensor-core accumulation bias probe: relative error and signed bias of G/H
vs the fp64 oracle for several chunk sizes (accumulation lengths)."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import oracle as O
    import paper_1704_07669_b200 as P
    a = O.synth_lowrank_plus_noise(20000, 10000, 200, "inv", 1e-3, seed=2)
    om = O.gaussian(10000, 60, 1)
    ref = O.oracle_sketch(O.row_blocks(a, 4096), om.astype(np.float32).astype(np.float64))
    out = {}
    for prec in ("simt", "tc"):
        st = P.sketch_pass(P.ArrayRowStream(a), om, precision=prec)
        for key, x, r in (("G", st.g, ref.g), ("H", st.h, ref.h)):
            d = x - r
            out[f"{prec}_{key}_rel"] = float(np.linalg.norm(d) / np.linalg.norm(r))
            out[f"{prec}_{key}_bias"] = float(np.sum(d * r) / np.sum(r * r))
    print(json.dumps(out))
else:
    for mb in ("4", "48", "640"):
        env = dict(os.environ, SPCA_TC_CHUNK_MB=mb)
        res = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print("chunk MB", mb, res.stdout.strip() or res.stderr[-500:])
