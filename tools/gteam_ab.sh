#!/bin/bash
# G slice reductions on a reduction team (config 2), same box: team of one warp, two warps, off
for cfg in "SPCA_BUILD_GTEAM=1" "SPCA_BUILD_GTEAM=2" "SPCA_BUILD_GTEAM=0"; do
  env $cfg python -m paper_1704_07669_b200.build --force > /dev/null || { echo "build failed: $cfg"; continue; }
  echo "--- build: $cfg"
  bash tools/knobs.sh "X=1" "X=2" "SPCA_TC_LAGF=1.25"
  if [ "$cfg" != "SPCA_BUILD_GTEAM=0" ]; then timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2; fi
done
