#!/bin/bash
# G slice reduction with ten loads in flight (SPCA_GRED_WIDE), same box
for cfg in "SPCA_BUILD_GWIDE=1" "SPCA_BUILD_GWIDE=0" "SPCA_BUILD_GWIDE=1"; do
  env $cfg python -m paper_1704_07669_b200.build --force > /dev/null || { echo "build failed: $cfg"; continue; }
  echo "--- build: $cfg"
  bash tools/knobs.sh "X=1" "X=2"
  BENCH_ARGS="--config cfg5" bash tools/knobs.sh "X=1"
done
