"""CPU oracle for the single-pass PCA sketch path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithm of the reference
package ``streampca`` (``/root/reference/pkg/src/streampca``) for the one
hot path this repository accelerates: the streaming sketch pass
(``sketch.py:52-116``), the post-hoc centering (``sketch.py:119-139``), the
blocked QB post-pass (``qb.py:59-171``), the dense kernels it uses
(``linalg.py:39-169``) and the ``single_pass_pca`` driver
(``algorithms.py:144-204``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import it, and only as the checker or the timed CPU
baseline. The product package (``paper_1704_07669_b200``) never imports it:
the product path is CUDA behind ``libspca.so`` and fails loudly without it.

Parity is pinned: ``tests/golden/make_golden.py`` imports the real
reference in the build container and stores its outputs as fixtures;
``tests/test_oracle_golden.py`` checks this restatement against them.
"""

from .spca_oracle import *  # noqa: F401,F403
