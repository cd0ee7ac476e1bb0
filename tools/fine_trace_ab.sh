#!/bin/bash
# per-K-block timeline (fine-trace build) of the config-2 pass: defaults, and the
# skeleton (no loads, no MMAs, no epilogue) whose 1.0 ms floor is being explained
SPCA_BUILD_FINE_TRACE=1 python -m paper_1704_07669_b200.build --force > /dev/null
for d in 0 18446 18434 18432; do
  echo "=== SPCA_TC_DEBUG=$d"
  SPCA_TC_TRACE=1 SPCA_TC_DEBUG=$d timeout 120 python tools/trace_fused.py 2>&1 | grep -v "^  [GH] units" | tail -14
done
