import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_1704_07669_b200 as P
for (m, n, l) in [(32, 128, 60), (128, 128, 60), (256, 256, 60)]:
    a = O.gaussian(m, n, seed=1).astype(np.float32)
    om = O.gaussian(n, l, seed=2)
    st = P.sketch_pass(P.ArrayRowStream(a), om, precision="tc")
    href = a.astype(np.float64).T @ st.g
    h = st.h
    print(m, n, l, "||H||", np.linalg.norm(h), "||Href||", np.linalg.norm(href),
          "cos", float(np.sum(h * href) / (np.linalg.norm(h) * np.linalg.norm(href) + 1e-300)))
    np.set_printoptions(precision=3, linewidth=200, suppress=True)
    print("H[:4,:6]\n", h[:4, :6], "\nHref[:4,:6]\n", href[:4, :6])
    nz = np.argwhere(np.abs(h) > 1e-6)
    print("nonzero count", len(nz), nz[:10].tolist())
    # try to explain H as a permutation: for a few H entries find matching Href
    if len(nz):
        i, j = nz[0]
        match = np.argwhere(np.isclose(href, h[i, j], rtol=1e-3))
        print("H[%d,%d]=%g matches Href at" % (i, j, h[i, j]), match[:5].tolist())
